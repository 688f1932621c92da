"""Dump the SPEC multiscale handoff of configs[1] (ms_256) at its switch layer (run on a GPU).

For N = 256 the switch layer is the finest one: layers 32^2..128^2 are solved by
global Sinkhorn at delta/4 on the device, and their duals, prolonged to 256^2,
warm-start the switch layer's warm_start_plan.  This script records those
prolonged duals (tests/golden/ms256_switch_duals.npz); scripts/make_golden.py
``ms256`` then runs the REFERENCE's warm_start_plan (its global Sinkhorn started
from these duals) and domdec_solve on them, and tests/test_gpu_baseline_parity.py
compares the GPU's whole ms_256 multiscale solve with that reference output.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    import paper_2410_08859_b200.engine as E
    import paper_2410_08859_b200.multiscale as M
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.problems import config_problem_arrays

    mu, nu, dx, org, cfg = config_problem_arrays(1, seed=0)
    h2 = dx * dx
    grid = Grid(mu.shape, dx, org)
    prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu),
                            DivergenceSpec(cfg["lam"]), 2 * h2)
    got = {}
    orig = M.warm_start_plan

    def hook(problem, dec, delta=1e-3, max_iters=20_000, trunc_threshold=1e-15, dp=None,
             alpha0=None, beta0=None):
        got.update(alpha0=alpha0.cpu().numpy().reshape(mu.shape),
                   beta0=beta0.cpu().numpy().reshape(nu.shape), delta=delta, max_iters=max_iters,
                   eps=problem.eps)
        return orig(problem, dec, delta=delta, max_iters=max_iters,
                    trunc_threshold=trunc_threshold, dp=dp, alpha0=alpha0, beta0=beta0)

    M.warm_start_plan = hook
    try:
        st, rep = M.multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2)
    finally:
        M.warm_start_plan = orig
    out = os.path.join(ROOT, "tests", "golden", "ms256_switch_duals.npz")
    np.savez_compressed(out, mu=mu, nu=nu, dx=dx, origin=np.array(org), lam=cfg["lam"],
                        s=cfg["cell"], eps=got["eps"], warm_delta=got["delta"],
                        warm_max_iters=got["max_iters"], alpha0=got["alpha0"],
                        beta0=got["beta0"], gpu_total=rep.final_score["total"],
                        gpu_iterations=rep.stages[-1][2].iterations)
    print("wrote", out, os.path.getsize(out), "GPU final total", rep.final_score["total"],
          "stage", rep.stages[-1][0], rep.stages[-1][2].iterations)


if __name__ == "__main__":
    main()
