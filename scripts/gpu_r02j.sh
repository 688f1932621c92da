mkdir -p gpurun_out
timeout 300 python scripts/dump_ms256_switch.py > gpurun_out/j_dump.log 2>&1
cp tests/golden/ms256_switch_duals.npz gpurun_out/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/j_bench.log 2>&1
timeout 600 python bench.py > gpurun_out/j_bench2.log 2>&1
export DD_PROBE_BATCHES=1
timeout 300 python scripts/probe_spec.py 2 512 > gpurun_out/j_spec.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/j_tests.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches.csv -k 'regex:^(?!axpb_kernel|terms_kernel|sk_check_kernel|newton_global_kernel|row_lse_tab_kernel).*' python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/j_ncu_list.log 2>&1
