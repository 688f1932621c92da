"""Probe: device global Sinkhorn on one pyramid level of a BASELINE config (timing)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
from paper_2410_08859_b200.multiscale import coarsen
from paper_2410_08859_b200.sinkhorn import DeviceProblem, SolverConfig, sinkhorn_solve, mass_balanced_start

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 500
mu, nu, dx, org, cfg = config_problem_arrays(idx, seed=0)
N = mu.shape[0]
while mu.shape[0] > n:
    mu, nu = coarsen(mu), coarsen(nu)
h = 1.0 / n
g = Grid(mu.shape, h, (0.5 * h, 0.5 * h))
eps = cfg["eps_start_h2"] * dx * dx
prob = TransportProblem(GridMeasure(g, mu), GridMeasure(g, nu), DivergenceSpec(cfg["lam"]), eps)
dp = DeviceProblem(prob)
a0, b0 = mass_balanced_start(dp)
for trace in (False, True):
    sinkhorn_solve(dp, a0, b0, SolverConfig(delta=1e-30, max_iters=20), collect_trace=trace)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = sinkhorn_solve(dp, a0, b0, SolverConfig(delta=1e-30, max_iters=iters), collect_trace=trace)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"n={n} {'host loop' if trace else 'device loop'}: {iters} iterations {t*1e3:.1f} ms = {t/iters*1e6:.1f} us/iteration", flush=True)
