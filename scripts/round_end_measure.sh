#!/bin/bash
# Round-2 end-of-round measurement on one B200 (writes gpurun_out/final_*):
# GPU test suite, the bench line (ms_1024), the CPU reference arm, ms_256, the fp32
# mode and configs[4] vol_128 as extra bench lines.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rxX > gpurun_out/final_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/final_bench_ref.log 2>&1
timeout 600 python bench.py --config vol_128 --cpu-sample 0 > gpurun_out/final_bench_vol128.log 2>&1
timeout 600 python bench.py --config ms_256 --cpu-sample 0 > gpurun_out/final_bench_ms256.log 2>&1
timeout 600 python bench.py --precision fp32 --cpu-sample 0 --steps 1 > gpurun_out/final_bench_fp32.log 2>&1
timeout 600 python bench.py --config vol_128 --precision fp32 --cpu-sample 0 > gpurun_out/final_bench_vol128_fp32.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
