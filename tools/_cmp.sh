timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_gemm.py tests/test_sparse_pipeline.py > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for c in ${CFGS:-default}; do
  echo "== cfg=$c"
  for i in 1 2; do Q8G_SK_CFG=$c timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python3 -c "import json,sys; d=json.loads(open(\"gpurun_out/b.json\").readline()); print(round(d[\"value\"],1), round(d[\"ms_per_step\"]*1e3,2), d[\"clocks\"][\"sm_mhz\"], d[\"roofline\"][\"frac\"])"; done
  Q8G_SK_CFG=$c Q8G_TC_TRACE=1 timeout 120 python tools/tc_trace.py --m 128 --requant --steady 31 2>&1 | head -17 | tail -16
done
