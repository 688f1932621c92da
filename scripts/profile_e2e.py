"""Host-side profile of the e2e path of bench.py (ms_1024): where the non-device time goes."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import bench

prob, cfg, eps_start = bench.problem(sys.argv[1] if len(sys.argv) > 1 else "ms_1024", 0)
bench.run_solve(prob, cfg, eps_start, None)   # warm-up
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
st, rep = bench.run_solve(prob, cfg, eps_start, None)
d2h = bench.fetch_result(st)
torch.cuda.synchronize()
pr.disable()
print("e2e wall", time.perf_counter() - t0, "d2h bytes", d2h)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
