"""Probe: SPEC multiscale protocol on a BASELINE config, per-stage and per-batch stats.

usage: probe_spec.py CONFIG_IDX [min_level_for_batch_log] [max_domdec_iters]
env: DD_MS_SWITCH (switch layer), DD_MS_SWITCH_DELTA, DD_MS_GDELTA, DD_MS_PROTOCOL
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
import paper_2410_08859_b200.multiscale as M

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lvl = int(sys.argv[2]) if len(sys.argv) > 2 else 512
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
kw = {}
if os.environ.get("DD_MS_SWITCH"):
    kw["switch"] = int(os.environ["DD_MS_SWITCH"])
if os.environ.get("DD_MS_SWITCH_DELTA"):
    kw["switch_delta"] = float(os.environ["DD_MS_SWITCH_DELTA"])
if os.environ.get("DD_MS_GDELTA"):
    kw["global_delta"] = float(os.environ["DD_MS_GDELTA"])
if os.environ.get("DD_MS_PROTOCOL"):
    kw["protocol"] = os.environ["DD_MS_PROTOCOL"]
prec = os.environ.get("DD_MS_PRECISION", "fp64")
print("options", kw, "precision", prec, flush=True)
mu, nu, dx, org, cfg = config_problem_arrays(idx, seed=0)
h2 = dx * dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]),
                        cfg["eps_final_h2"] * h2)
orig_solve = E._Batch.solve


def solve(self):
    N = self.st.dp.geom.nx0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    orig_solve(self)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    if N >= lvl and os.environ.get("DD_PROBE_BATCHES", "1") == "1":
        c1, c2 = self.stats()
        ny = (self.ybox[:, 1] * self.ybox[:, 3]).astype(float)
        it = c1[:, 2]
        print(f"    batch N={N} cells={self.n} t={t:.2f}s ny mean={ny.mean():.0f} p99={np.percentile(ny, 99):.0f} "
              f"max={ny.max():.0f} iters mean={it.mean():.0f} p50={np.median(it):.0f} p99={np.percentile(it, 99):.0f} "
              f"capped={(it >= 9999).sum()} nonconv={(c1[:, 3] == 0).sum()}", flush=True)


E._Batch.solve = solve


def prog(n, e, r):
    if prec == "fp32":
        import ctypes
        from paper_2410_08859_b200 import _lib
        buf = (ctypes.c_ulonglong * 4)()
        _lib.load().dd_sweep_fallbacks(buf)
        print(f"  fp32 sweeps: X {buf[0]}/{buf[2]} fell back, Y {buf[1]}/{buf[3]} fell back", flush=True)
    d = r.diagnostics
    print(f"  [stage] N={n} eps/h2={e / h2:.1f} solver={d.get('solver', 'domdec')} iters={r.iterations} "
          f"conv={r.converged} t={r.timings['total']:.2f}s gap={d.get('gap', r.rel_pd_gap):.3e} "
          f"cell_it={d.get('cell_iterations')} nonconv={d.get('nonconverged_cells')} fb={d.get('safe_fallbacks')}",
          flush=True)
    for row in r.trace[:6] + r.trace[-2:] if len(r.trace) > 8 else r.trace:
        print(f"      k={row.k} {row.label} {row.action} total={row.total:.10e} gap={row.gap:.3e} wall={row.wall_time:.2f}",
              flush=True)


torch.cuda.synchronize()
t0 = time.perf_counter()
st, rep = M.multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2,
                             config=E.EngineConfig(max_iters=maxit,
                                                   cell=E.CellSolverConfig(precision=prec)),
                             progress=prog,
                             **kw)
torch.cuda.synchronize()
print(f"TOTAL {time.perf_counter() - t0:.2f}s converged={rep.converged} timings={rep.timings} "
      f"final={rep.final_score} rel_gap={rep.rel_pd_gap:.3e} sparsity={st.sparsity()}", flush=True)
