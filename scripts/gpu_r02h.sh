mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32.py -q > gpurun_out/h_fp32_tests.log 2>&1
