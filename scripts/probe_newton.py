import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2410_08859_b200 import _lib
_lib.LIB_PATH = os.environ.get("DD_DBG_LIB", os.path.join(os.getcwd(), "build_dbg", "libdomdec_b200.so"))
_lib.load(_lib.LIB_PATH)
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
from paper_2410_08859_b200.multiscale import multiscale_solve
idx, stop = int(sys.argv[1]), int(sys.argv[2])
mu, nu, dx, org, cfg = config_problem_arrays(idx, seed=0)
h2 = dx*dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), 2*h2)
rows = []
orig = E._Batch.solve
def solve(self):
    orig(self)
    c1, c2 = self.stats()
    for k in range(self.n):
        ny = self.ybox[k,1]*self.ybox[k,3]; it = max(c1[k,2], 1)
        rows.append((self.st.dp.geom.nx0, ny, c1[k,2], c2[k,3]/it/ny, c1[k,4]/it/ny, c1[k,5]/it/ny, c1[k,6], c1[k,7]/it/ny))
E._Batch.solve = solve
class Stop(Exception): pass
def prog(nl, e, r):
    if nl >= stop: raise Stop()
try:
    multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"]*h2, progress=prog)
except Stop: pass
R = np.array(rows)
for N in np.unique(R[:,0]):
    S = R[R[:,0]==N]
    w = S[:,2]*S[:,1]
    print(f"N={int(N)} evals/node/iter={np.average(S[:,3],weights=w):.2f} clips/node/iter={np.average(S[:,4],weights=w):.4f} bisect/node/iter={np.average(S[:,5],weights=w):.4f} maxevals={S[:,6].max():.0f} frac_nodes>=6={np.average(S[:,7],weights=w):.4f}")
