set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
./scripts/micro/fp64_peak > gpurun_out/a_fp64_peak.json 2>&1
timeout 600 python scripts/make_cell_sample.py > gpurun_out/a_sample.log 2>&1
cp tests/golden/ms1024_cells.npz gpurun_out/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/a_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/a_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/a_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_launches.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/a_ncu_list.log 2>&1
