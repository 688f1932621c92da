# parity (default, forced clusters, forced global workspace), smoke, bench line, capped-cell phases
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/f3_tests.log 2>&1; tail -1 gpurun_out/f3_tests.log
DD_FORCE_CLUSTER=2 timeout 200 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
DD_FORCE_CLUSTER=4 timeout 200 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
DD_FORCE_GLOBAL_WS=1 timeout 200 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/f3_bench.log 2>&1; tail -1 gpurun_out/f3_bench.log | cut -c1-160
DD_DBG_LIB=$PWD/build_dbg/libdomdec_b200.so timeout 400 python scripts/probe_phase_level.py 256 1 2>&1 | grep cycles
DD_DBG_LIB=$PWD/build_dbg/libdomdec_b200.so timeout 400 python scripts/probe_phase_level.py 1024 2 2>&1 | grep cycles
