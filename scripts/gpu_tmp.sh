mkdir -p gpurun_out
DD_PROBE_BATCHES=0 DD_MS_PRECISION=fp32 timeout 300 python scripts/probe_spec.py 2 99999 > gpurun_out/t_fp32.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_baseline_parity.py -q --timeout 300 -rxX > gpurun_out/t_tests.log 2>&1
