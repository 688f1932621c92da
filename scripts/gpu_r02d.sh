mkdir -p gpurun_out
export DD_PROBE_BATCHES=1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "golden or sinkhorn or sweep" > gpurun_out/d_tests.log 2>&1
timeout 300 python scripts/probe_spec.py 2 1024 > gpurun_out/d_spec_nt512.log 2>&1
DD_LIB_PATH=$PWD/build_nt256/libdomdec_b200.so timeout 300 python scripts/probe_spec.py 2 1024 > gpurun_out/d_spec_nt256.log 2>&1
DD_LIB_PATH=$PWD/build_nt256/libdomdec_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/d_tests_nt256.log 2>&1
timeout 300 python scripts/probe_spec.py 1 256 > gpurun_out/d_spec256.log 2>&1
