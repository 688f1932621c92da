#!/bin/bash
# bench ms_256 + first two 1024^2 iterations for each library build variant
for v in default build_occ2 build_pair; do
  if [ "$v" = default ]; then export DD_LIB_PATH=""; else export DD_LIB_PATH="$PWD/$v/libdomdec_b200.so"; fi
  echo "== $v" >> gpurun_out/variants.log
  timeout 150 python bench.py --steps 2 --warmup 3 --cpu-sample 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms256', d['value'])" >> gpurun_out/variants.log 2>&1
  timeout 420 python scripts/probe_level.py 2 1024 1 2>/dev/null | grep -E "stage\] N=(512|1024)|launch" | cut -c1-110 >> gpurun_out/variants.log 2>&1
done
