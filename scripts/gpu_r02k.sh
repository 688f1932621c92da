mkdir -p gpurun_out
export DD_PROBE_BATCHES=1
DD_NO_CLUSTER_CAPPED=1 timeout 120 python scripts/probe_spec.py 2 512 > gpurun_out/k_spec_nocc.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -k "default" > gpurun_out/k_parity_default.log 2>&1
DD_NO_CLUSTER_CAPPED=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -k "default" > gpurun_out/k_parity_nocc.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -k "cluster2" > gpurun_out/k_parity_c2.log 2>&1
