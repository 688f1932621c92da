"""Probe: per-cell cost profile of the cell-solve launches in a multiscale run."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
from paper_2410_08859_b200.multiscale import multiscale_solve

idx = int(sys.argv[1]); n = int(sys.argv[2]); maxit = int(sys.argv[3]); stop_level = int(sys.argv[4])
mu, nu, dx, org, cfg = config_problem_arrays(idx, seed=0, n=n)
h2 = dx * dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), 2 * h2)
rows = []
orig = E._Batch.solve
def solve(self):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    orig(self)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    c1, c2 = self.stats()
    N = self.st.dp.geom.nx0
    for k in range(self.n):
        rows.append((N, t, int(self.ybox[k, 1]), int(self.ybox[k, 3]), int(c1[k, 2]), c2[k, 2], c2[k, 3], bool(self.batch.smem_mode)))
E._Batch.solve = solve
class Stop(Exception): pass
def prog(nl, e, r):
    print(f"[stage] {nl} eps/h2={e/h2:.1f} iters={r.iterations} t={r.timings['total']:.2f}", flush=True)
    if nl >= stop_level: raise Stop()
try:
    multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2, config=E.EngineConfig(max_iters=maxit), progress=prog)
except Stop:
    pass
R = np.array([(r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]) for r in rows])
for N in np.unique(R[:, 0]):
    S = R[R[:, 0] == N]
    ny = S[:, 2] * S[:, 3]
    it = S[:, 4]
    cyc = S[:, 5]
    print(f"N={int(N)} cells={len(S)} ny mean={ny.mean():.0f} max={ny.max():.0f} iters mean={it.mean():.1f} max={it.max():.0f} "
          f"cyc/iter median={np.median(cyc/np.maximum(it,1)):.0f} newton/node/iter median={np.median(S[:,6]/np.maximum(it*ny,1)):.2f} smem_frac={S[:,7].mean():.2f}")
    top = np.argsort(-cyc)[:8]
    for t in top:
        print(f"   slow: ny={int(S[t,2])}x{int(S[t,3])} iters={int(S[t,4])} cycles={S[t,5]:.3g} cyc/iter={S[t,5]/max(S[t,4],1):.0f} newton/node/iter={S[t,6]/max(S[t,4]*S[t,2]*S[t,3],1):.2f} smem={bool(S[t,7])}")
