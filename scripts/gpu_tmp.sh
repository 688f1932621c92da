mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_volume.py -q --timeout 300 > gpurun_out/v_tests.log 2>&1
for v in default mb3 mb1; do
  if [ $v = default ]; then unset DD_LIB_PATH; else export DD_LIB_PATH=$PWD/build_$v/libdomdec_b200.so; fi
  timeout 300 python scripts/probe_vol.py 128 > gpurun_out/vol128_$v.log 2>&1
done
unset DD_LIB_PATH
timeout 600 python bench.py --config vol_128 --steps 2 --warmup 3 > gpurun_out/bench_vol128.log 2>&1
