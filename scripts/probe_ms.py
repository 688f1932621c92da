"""Probe: one multiscale solve of a BASELINE config on cuda:0, per-stage timings."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem, _lib
from paper_2410_08859_b200.problems import config_problem_arrays
from paper_2410_08859_b200.multiscale import multiscale_solve
from paper_2410_08859_b200.engine import EngineConfig, StrategyConfig

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
every = int(sys.argv[3]) if len(sys.argv) > 3 else 1
maxit = int(sys.argv[4]) if len(sys.argv) > 4 else 2000
mu, nu, dx, org, cfg = config_problem_arrays(idx, seed=0, n=n)
N = mu.shape[0]
h2 = dx * dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), cfg["eps_final_h2"] * h2)
tr = _lib.Tracer()
_lib.set_tracer(tr)
torch.cuda.synchronize()
t0 = time.perf_counter()
st, rep = multiscale_solve(prob, cfg["cell"], cfg["coarsest"], (cfg["eps_start_h2"] or 2.0) * h2,
                           config=EngineConfig(gap_check_every=every, max_iters=maxit),
                           progress=lambda n, e, r: print(f"  [stage] level {n} eps/h2={e/h2:.1f} iters={r.iterations} gap={r.rel_pd_gap:.2e} t={r.timings['total']:.2f}s solve={r.timings['solve']:.2f} score={r.timings['score']:.2f} cell_it={r.diagnostics['cell_iterations']} nonconv={r.diagnostics['nonconverged_cells']} fb={r.diagnostics['safe_fallbacks']}", flush=True))
torch.cuda.synchronize()
T = time.perf_counter() - t0
print(f"config {idx} N={N} total {T:.3f}s converged={rep.converged} iters={rep.total_iterations}", flush=True)
print("timings", {k: round(v, 3) for k, v in rep.timings.items()})
for lvn, eps, r in rep.stages:
    print(f"  level {lvn:5d} eps/h2={eps/h2:8.2f} iters={r.iterations:3d} conv={r.converged} gap={r.rel_pd_gap:.2e} "
          f"t={r.timings['total']:.3f} solve={r.timings['solve']:.3f} score={r.timings['score']:.3f} "
          f"commit={r.timings['commit']:.3f} cell_it={r.diagnostics['cell_iterations']} nonconv={r.diagnostics['nonconverged_cells']}", flush=True)
tm = tr.times_ms()
for k, v in tm.items():
    print(f"{k}: n={len(v)} total={sum(v):.1f}ms mean={np.mean(v):.3f}ms max={max(v):.3f}")
print("launches", tr.launches(), "calls", tr.calls)
print("final", rep.final_score, "sparsity", st.sparsity())
