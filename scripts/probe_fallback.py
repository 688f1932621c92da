import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem, _lib
_lib.LIB_PATH = os.path.join(os.getcwd(), "build_dbg", "libdomdec_b200.so")
h = _lib.load(_lib.LIB_PATH)
h.dd_debug_fallbacks.argtypes = [ctypes.c_void_p]
from paper_2410_08859_b200.problems import config_problem_arrays
import paper_2410_08859_b200.engine as E
from paper_2410_08859_b200.multiscale import multiscale_solve
mu, nu, dx, org, cfg = config_problem_arrays(2, seed=0)
h2 = dx * dx
grid = Grid(mu.shape, dx, org)
prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu), DivergenceSpec(cfg["lam"]), 2 * h2)
buf = (ctypes.c_ulonglong * 2)()
last = [0, 0]
class Stop(Exception): pass
def prog(nl, e, r):
    h.dd_debug_fallbacks(ctypes.addressof(buf))
    fb, out = buf[0] - last[0], buf[1] - last[1]
    last[0], last[1] = buf[0], buf[1]
    print(f"[stage] {nl} eps/h2={e/h2:.1f} t={r.timings['total']:.2f} fallbacks={fb} outputs={out} frac={fb/max(out,1):.4f}", flush=True)
    if nl >= 256: raise Stop()
try:
    multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2, progress=prog)
except Stop:
    pass
