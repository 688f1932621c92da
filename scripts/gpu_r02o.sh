mkdir -p gpurun_out
export DD_PROBE_BATCHES=0
timeout 300 python scripts/probe_spec.py 2 512 > gpurun_out/o_spec_default.log 2>&1
DD_CLUSTER_CAPPED=1 timeout 300 python scripts/probe_spec.py 2 512 > gpurun_out/o_spec_cc.log 2>&1
DD_CLUSTER_CAPPED=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "default" > gpurun_out/o_parity_cc.log 2>&1
