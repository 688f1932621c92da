mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cell_solve_kernel --launch-skip 12 -c 1 -o gpurun_out/m_cell1024 python scripts/probe_spec.py 2 99999 > gpurun_out/m_ncu_full.log 2>&1
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches.csv -k 'regex:^(?!axpb_kernel|terms_kernel|sk_check_kernel|newton_global_kernel|row_lse_tab_kernel).*' python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/m_ncu_list.log 2>&1
