run() { python bench.py --config C1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step']*1e3,3), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step']*1e3,1))"; }
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_sparse_pipeline.py tests/test_cpp_api.py -x -q 2>&1 | tail -2
for i in 1 2 3; do Q8G_SK_GRP=0 run kmajor; run grp; done
Q8G_TC_TRACE=1 timeout 120 python tools/tc_trace.py --m 128 --requant --steady 31 2>&1 | head -17 | tail -16
Q8G_SK_GRP=0 Q8G_TC_TRACE=1 timeout 120 python tools/tc_trace.py --m 128 --requant --steady 31 2>&1 | head -17 | tail -16
