mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_volume.py tests/test_gpu_kernels.py -q -x --timeout 400 -k "not split and not cluster4" > gpurun_out/p_tests.log 2>&1
for v in default nsingle; do
  if [ $v = default ]; then unset DD_LIB_PATH; else export DD_LIB_PATH=$PWD/build_$v/libdomdec_b200.so; fi
  DD_PROBE_BATCHES=0 timeout 300 python scripts/probe_spec.py 2 99999 > gpurun_out/ms1024_$v.log 2>&1
  timeout 300 python scripts/probe_vol.py 128 > gpurun_out/vol128_$v.log 2>&1
done
