# Round-end evidence on one B200: GPU suite, smoke, the default bench line
# (C2 headline + C1 / C3 / C4 sub-records), the reference arm, and the C2
# ncu launch list + one full capture of the CTA-pair kernel.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_gputest.log 2>&1; tail -2 gpurun_out/final_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_c2_launches.csv \
    python bench.py --no-sub --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/final_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2w -s 3 -c 1 -o gpurun_out/final_c2 \
    python bench.py --no-sub --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/final_ncu_full.log 2>&1; echo "ncu full rc=$?"
