mkdir -p gpurun_out
export DD_PROBE_BATCHES=1
timeout 300 python scripts/probe_spec.py 2 1024 > gpurun_out/c_spec_occ1.log 2>&1
DD_LIB_PATH=$PWD/build_occ2/libdomdec_b200.so timeout 300 python scripts/probe_spec.py 2 1024 > gpurun_out/c_spec_occ2.log 2>&1
timeout 600 python bench.py > gpurun_out/c_bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 > gpurun_out/c_bench_ref.log 2>&1
