mkdir -p gpurun_out
export DD_LIB_PATH=$PWD/build_nt1024/libdomdec_b200.so
DD_PROBE_BATCHES=0 timeout 400 python scripts/probe_spec.py 2 99999 > gpurun_out/ms1024_nt1024.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 400 -k "default" > gpurun_out/p_nt1024.log 2>&1
