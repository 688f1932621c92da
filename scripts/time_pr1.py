"""GPU time of configs[0] (pr1_64: 64^2, 30 domdec sweeps, cell tolerance 1e-7, reference
warm start) -- the one BASELINE config the reference itself was run on in full here
(tests/golden/pr1_64.npz: 4106 s of reference CPU, one core).  Same inputs, same protocol."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import torch

from _engine_run import run_device
from _golden import load

g = load("pr1_64")
run_device(g)                      # warm-up
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob, dec, st, rep = run_device(g)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"pr1_64 GPU solve: {np.median(ts):.3f} s (median of 3; runs {['%.3f' % t for t in ts]}), "
      f"iterations {rep.iterations} (reference {int(g['iterations'])}), total "
      f"{rep.final_score['total']!r} (reference {float(g['score'][-1])!r}); reference CPU "
      f"{float(g['ref_seconds']):.0f} s")
