mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/l_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/l_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/l_bench_ref.log 2>&1
