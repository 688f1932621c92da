mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1
DD_PROBE_BATCHES=0 DD_MS_PRECISION=fp32 timeout 300 python scripts/probe_spec.py 2 99999 > gpurun_out/s_fp32.log 2>&1
