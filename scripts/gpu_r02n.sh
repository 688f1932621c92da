mkdir -p gpurun_out
timeout 600 python scripts/probe_cluster_long.py > gpurun_out/n_cluster_long.log 2>&1
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -k ms256 --timeout 600 > gpurun_out/n_ms256.log 2>&1
