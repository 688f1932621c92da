mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/i_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/i_bench.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/i_ncu_list.log 2>&1
