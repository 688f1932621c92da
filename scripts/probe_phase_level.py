"""Phase cycles per Sinkhorn iteration of capped cells in the first batch at a level (DD_PHASE_TIMING build)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2410_08859_b200 import _lib
_lib.load(os.environ.get("DD_DBG_LIB", os.path.join(os.getcwd(), "build_dbg", "libdomdec_b200.so")))
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
import paper_2410_08859_b200.multiscale as M
level = int(sys.argv[1])
mu, nu, dx, org, cfg = config_problem_arrays(int(sys.argv[2]) if len(sys.argv) > 2 else 2, seed=0)
h2 = dx * dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), 2 * h2)
orig = E._Batch.solve
def solve(self):
    orig(self)
    if self.st.dp.geom.nx0 >= level:
        c1, c2 = self.stats()
        ny = (self.ybox[:, 1] * self.ybox[:, 3]).astype(float)
        it = np.maximum(c1[:, 2], 1)
        clu = np.zeros(self.n, bool)
        for _, sel, _ in self.clu_groups:
            clu[sel] = True
        for name, sel in (("smem capped", (c1[:, 2] >= 9999) & ~clu & self.owned), ("all smem", ~clu)):
            if not sel.any():
                continue
            ph = c1[sel, 4:8] / it[sel, None]
            fbx = np.floor(c2[sel, 1] / 1e6) / it[sel]
            fby = (c2[sel, 1] % 1e6) / it[sel]
            print(f"{name}: n={sel.sum()} ny med={np.median(ny[sel]):.0f} ny0 med={np.median(self.ybox[sel,1]):.0f} ny1 med={np.median(self.ybox[sel,3]):.0f} cycles/iter med: lse_x={np.median(ph[:,0]):.0f} gap={np.median(ph[:,1]):.0f} lse_y={np.median(ph[:,2]):.0f} newton={np.median(ph[:,3]):.0f} "
                  f"fallback frac x={np.median(fbx):.2f} y={np.median(fby):.2f} fallback cyc/iter={np.median(c2[sel,0]/it[sel]):.0f}", flush=True)
        raise SystemExit(0)
E._Batch.solve = solve
M.multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2)
