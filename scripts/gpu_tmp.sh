mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_volume.py -q --timeout 300 -x -k "grid_lse3 or global_sinkhorn3" > gpurun_out/v_a.log 2>&1
timeout 900 python -m pytest tests/test_gpu_volume.py -q --timeout 300 -k "not vol32 and not multiscale" > gpurun_out/v_b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_volume.py -q --timeout 500 -k "multiscale" > gpurun_out/v_c.log 2>&1
