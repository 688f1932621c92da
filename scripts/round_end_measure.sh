#!/bin/bash
# Round-2 end-of-round measurement on one B200 (writes gpurun_out/final_*):
# GPU test suite, the bench line (ms_1024), the CPU reference arm, ms_256 and the
# fp32 mode as extra bench lines, and configs[3] ms_2048 on one GPU.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/final_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/final_bench_ref.log 2>&1
timeout 600 python bench.py --config ms_256 --cpu-sample 0 > gpurun_out/final_bench_ms256.log 2>&1
timeout 600 python bench.py --precision fp32 --cpu-sample 0 --steps 1 > gpurun_out/final_bench_fp32.log 2>&1
DD_PROBE_BATCHES=0 timeout 900 python scripts/probe_spec.py 3 2048 > gpurun_out/final_2048.log 2>&1
