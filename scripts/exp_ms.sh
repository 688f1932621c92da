export DD_PROBE_BATCHES=0
timeout 300 python scripts/probe_spec.py 1 256 > gpurun_out/e2_256a.log 2>&1
DD_MS_SWITCH_DELTA=5e-6 timeout 300 python scripts/probe_spec.py 1 256 > gpurun_out/e2_256b.log 2>&1
DD_MS_PROTOCOL=ladder timeout 300 python scripts/probe_spec.py 1 256 > gpurun_out/e2_256c.log 2>&1
timeout 600 python scripts/probe_spec.py 2 512 > gpurun_out/e2_1024a.log 2>&1
DD_MS_SWITCH=9 timeout 600 python scripts/probe_spec.py 2 512 > gpurun_out/e2_1024b.log 2>&1
DD_MS_SWITCH_DELTA=5e-6 timeout 600 python scripts/probe_spec.py 2 512 > gpurun_out/e2_1024c.log 2>&1
DD_MS_GDELTA=5e-7 DD_MS_SWITCH_DELTA=5e-7 timeout 600 python scripts/probe_spec.py 2 512 > gpurun_out/e2_1024d.log 2>&1
