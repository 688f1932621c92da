mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_baseline_parity.py -q > gpurun_out/g_fp32_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k pr1_64 > gpurun_out/g_pr1.log 2>&1
timeout 600 python bench.py --precision fp32 --cpu-sample 0 > gpurun_out/g_bench_fp32.log 2>&1
export DD_PROBE_BATCHES=0
timeout 900 python scripts/probe_spec.py 3 2048 > gpurun_out/g_2048_fp64.log 2>&1
