import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import _lib
_lib.LIB_PATH = os.path.join(os.getcwd(), "build_dbg", "libdomdec_b200.so")
_lib.load(_lib.LIB_PATH)
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
from paper_2410_08859_b200.multiscale import multiscale_solve
idx = int(sys.argv[1])
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
        it = max(c1[k, 2], 1)
        rows.append((self.st.dp.geom.nx0, self.ybox[k, 1]*self.ybox[k, 3], c1[k, 2], c1[k, 4]/it, c1[k, 5]/it, c1[k, 6]/it, c1[k, 7]/it, c2[k, 3]/it/max(self.ybox[k,1]*self.ybox[k,3],1)))
E._Batch.solve = solve
multiscale_solve(prob, cfg["cell"], cfg["coarsest"], (cfg["eps_start_h2"] or 2)*h2)
R = np.array(rows)
for N in np.unique(R[:, 0]):
    S = R[(R[:, 0] == N) & (R[:, 2] > 20)]
    if not len(S): continue
    print(f"N={int(N)} cells={len(S)} ny med={np.median(S[:,1]):.0f} cycles/iter med: lse_x={np.median(S[:,3]):.0f} gap={np.median(S[:,4]):.0f} lse_y={np.median(S[:,5]):.0f} newton={np.median(S[:,6]):.0f} newton_evals/node={np.median(S[:,7]):.2f}")
