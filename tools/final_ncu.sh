# ncu launch lists + one full capture per sub-config (C1 / C3 / C4) of the final build
set -u
mkdir -p gpurun_out
for cfg in C1 C3 C4; do
  case $cfg in C1) k=gemm_splitk;; C3) k=conv3x3_tc;; C4) k=dwconv_tc64;; esac
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_${cfg}_launches.csv \
      python bench.py --config $cfg --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/final_ncu_${cfg}_l.log 2>&1; echo "$cfg launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/final_$cfg \
      python bench.py --config $cfg --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/final_ncu_${cfg}_f.log 2>&1; echo "$cfg full rc=$?"
done
