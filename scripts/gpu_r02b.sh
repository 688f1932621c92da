mkdir -p gpurun_out
./scripts/micro/fp64_peak > gpurun_out/b_fp64_peak.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/b_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/b_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cell_solve_kernel --launch-skip 12 -c 1 -o gpurun_out/b_cell1024 python scripts/probe_spec.py 2 99999 > gpurun_out/b_ncu_full.log 2>&1
