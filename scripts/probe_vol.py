"""Probe: configs[4] (3D) SPEC multiscale on the three-axis path, per-stage and per-batch stats.

usage: probe_vol.py [N] [max_domdec_iters]
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.engine import EngineConfig
from paper_2410_08859_b200.multiscale import multiscale_solve
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.volume as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
mu, nu, dx, org, cfg = config_problem_arrays(4, seed=0, n=n)
h2 = dx * dx
prob = TransportProblem(GridMeasure(Grid(mu.shape, dx, org), mu),
                        GridMeasure(Grid(nu.shape, dx, org), nu), DivergenceSpec(cfg["lam"]),
                        cfg["eps_final_h2"] * h2)
orig = V._Batch3.solve


def solve(self):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    orig(self)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    c1, c2 = self.stats()
    it = c1[:, 2]
    print(f"    batch cells={self.n} t={t:.3f}s ny mean={self.ny.mean():.0f} max={self.ny.max()} "
          f"iters mean={it.mean():.0f} p50={np.median(it):.0f} max={it.max():.0f} "
          f"capped={(it >= self.cfg.max_iters).sum()} nonconv={(c1[:, 3] == 0).sum()} "
          f"fallback_sweeps={int(c2[:, 3].sum())} newton/node-iter="
          f"{c2[:, 4].sum() / max((c2[:, 2] * self.ny).sum(), 1):.2f} "
          f"cycles/iter(longest)={c2[np.argmax(it), 5] / max(it.max(), 1):.0f}", flush=True)


V._Batch3.solve = solve


def progress(N, eps, r):
    d = r.diagnostics
    print(f"  [stage] N={N} eps/h2={eps / (1.0 / N) ** 2:.1f} solver={d.get('solver', 'domdec')} "
          f"iters={r.iterations} conv={r.converged} t={r.timings['total']:.2f}s "
          f"cell_it={d.get('cell_iterations', 0)} nonconv={d.get('nonconverged_cells', 0)}",
          flush=True)
    for row in r.trace:
        print(f"      k={row.k} {row.label} {row.action} total={row.total:.10e} gap={row.gap:.3e} "
              f"wall={row.wall_time:.2f}", flush=True)


torch.cuda.synchronize()
t0 = time.perf_counter()
st, rep = multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2,
                           config=EngineConfig(delta=2e-5, max_iters=maxit), progress=progress)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(f"TOTAL {t:.2f}s converged={rep.converged} timings={rep.timings} final={rep.final_score} "
      f"rel_gap={rep.rel_pd_gap:.3e} sparsity={st.sparsity()}", flush=True)
