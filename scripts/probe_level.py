"""Per-launch profile of the first domdec iterations at a given multiscale level."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
import paper_2410_08859_b200.multiscale as M
idx, level, iters_at_level = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
final_stages = int(sys.argv[4]) if len(sys.argv) > 4 else 1
mu, nu, dx, org, cfg = config_problem_arrays(idx, seed=0)
h2 = dx*dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), 2*h2)
orig_solve = E._Batch.solve
def solve(self):
    N = self.st.dp.geom.nx0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    orig_solve(self)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    if N >= level:
        c1, c2 = self.stats()
        ny = (self.ybox[:,1]*self.ybox[:,3]).astype(float)
        it = c1[:,2]
        top = np.argsort(-c2[:,2])[:3]
        print(f"  launch N={N} cells={self.n} t={t:.2f}s ny mean={ny.mean():.0f} p99={np.percentile(ny,99):.0f} max={ny.max():.0f} "
              f"iters mean={it.mean():.0f} p99={np.percentile(it,99):.0f} max={it.max():.0f} capped={(it>=9999).sum()} smem={self.batch.smem_mode}/{self.batch.smem_bytes} "
              f"slowest: " + "; ".join(f"ny={int(ny[k])} it={int(it[k])} cyc/it={c2[k,2]/max(it[k],1):.0f} nwt/node/it={c2[k,3]/max(it[k]*ny[k],1):.1f}" for k in top), flush=True)
E._Batch.solve = solve
orig_dd = M.domdec_solve
def dd(problem, dec, strategy, config, state=None, evaluator=None):
    N = problem.mu.grid.dims[0]
    cfg2 = E.EngineConfig(max_iters=iters_at_level) if N >= level else config
    st, r = orig_dd(problem, dec, strategy, cfg2, state=state, evaluator=evaluator)
    print(f"[stage] N={N} eps/h2={problem.eps/h2:.1f} iters={r.iterations} t={r.timings['total']:.2f}", flush=True)
    if N >= level:
        raise SystemExit(0)
    return st, r
M.domdec_solve = dd
M.multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"]*h2, final_stages=final_stages)
