mkdir -p gpurun_out
for n in 64 128 256 512 1024; do timeout 120 python scripts/probe_sinkhorn.py 2 $n 200 >> gpurun_out/e_sk.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_sk_launches.csv --launch-skip 300 --launch-count 60 python scripts/probe_sinkhorn.py 2 64 100 > gpurun_out/e_ncu.log 2>&1
timeout 300 python scripts/probe_spec.py 2 99999 > gpurun_out/e_spec.log 2>&1
