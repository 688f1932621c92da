mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/t_smi.log 2>&1
DD_PROBE_BATCHES=0 DD_MS_PRECISION=fp32 timeout 300 python scripts/probe_spec.py 2 99999 > gpurun_out/t_fp32.log 2>&1
DD_PROBE_BATCHES=0 timeout 300 python scripts/probe_spec.py 2 99999 > gpurun_out/t_fp64.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rxX > gpurun_out/t_tests.log 2>&1
