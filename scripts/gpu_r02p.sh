mkdir -p gpurun_out
export DD_PROBE_BATCHES=1
timeout 300 python scripts/probe_spec.py 2 1024 > gpurun_out/p_spec_split.log 2>&1
DD_NO_SPLIT=1 timeout 300 python scripts/probe_spec.py 2 1024 > gpurun_out/p_spec_nosplit.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q --timeout 300 > gpurun_out/p_tests.log 2>&1
