mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/f_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/f_bench.log 2>&1
DD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 1 --cpu-sample 0 > gpurun_out/f_bench2.log 2>&1
