import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem, _lib
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.multiscale as M
import paper_2410_08859_b200.engine as E

mu, nu, dx, org, cfg = config_problem_arrays(2, seed=0)
h2 = dx * dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), 2 * h2)
orig = E.domdec_solve
def dd(problem, dec, strategy, config, state=None, evaluator=None):
    N = problem.mu.grid.dims[0]
    st, r = orig(problem, dec, strategy, E.EngineConfig(max_iters=4), state=state, evaluator=evaluator)
    a, b, d = evaluator._best
    print(f"N={N} eps/h2={problem.eps/h2:.1f} gaps={[row.gap for row in r.trace]} totals={[row.total for row in r.trace]}", flush=True)
    print("   best D", d, "nan a", int(torch.isnan(a).sum()), "nan b", int(torch.isnan(b).sum()), "inf b", int(torch.isinf(b).sum()),
          "b range", float(b.min()), float(b.max()), flush=True)
    sb = st.energy(); print("   energy", sb, flush=True)
    xm = st.x_marg_d; print("   nan xmarg", int(torch.isnan(xm).sum()), "nan yval", int(torch.isnan(st.yval).sum()), "nan tr", int(torch.isnan(st.transport_d).sum()), int(torch.isnan(st.kl_d).sum()))
    for lab, store in st.stores.items():
        print("   store", lab, "nan alpha", int(torch.isnan(store.alpha).sum()), "nan beta", int(torch.isnan(store.beta).sum()), "inf beta", int(torch.isinf(store.beta).sum()))
    return st, r
M.domdec_solve = dd
st, rep = M.multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2)
