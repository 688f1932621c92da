set -x
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/f2_tests.log 2>&1; tail -2 gpurun_out/f2_tests.log
DD_FORCE_CLUSTER=4 timeout 200 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f2_smoke.log 2>&1; tail -1 gpurun_out/f2_smoke.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/f2_smi.txt
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/f2_bench.log 2>&1; tail -1 gpurun_out/f2_bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/f2_bench_ref.log 2>&1; tail -1 gpurun_out/f2_bench_ref.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_solve_kernel --launch-skip 40 -c 1 -o gpurun_out/f2_prof_cell python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/f2_ncu_full.log 2>&1; tail -2 gpurun_out/f2_ncu_full.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/f2_ncu_list.log 2>&1; tail -1 gpurun_out/f2_ncu_list.log | cut -c1-200
