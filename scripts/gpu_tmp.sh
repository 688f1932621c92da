mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_volume.py tests/test_gpu_sharded.py tests/test_gpu_volume_sharded.py tests/test_gpu_fp32.py -q --timeout 600 -x > gpurun_out/p_sp.log 2>&1
timeout 600 python bench.py --cpu-sample 0 > gpurun_out/bench_sp.log 2>&1
timeout 600 python bench.py --config vol_128 --cpu-sample 0 > gpurun_out/bench_vol_sp.log 2>&1
