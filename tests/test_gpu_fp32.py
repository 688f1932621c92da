"""fp32 mode (north_star: "in the fp32 mode, within 1e-4 relative").

The cell sweeps run in fp32 (tables, shifted weights, contractions; fp64
potentials, Newton Y-step, gap test and epilogue) and the results are compared
with the reference's fp64 outputs (golden fixtures) at 1e-4 relative: the
primal-dual objective, the basic-cell marginals (max-abs error / max-abs of the
reference array) and the stored cell duals.  Iteration counts may differ by the
borderline stopping decisions fp32 rounding can flip, so they are not compared.
"""

import numpy as np
import pytest

from _golden import dense, load, ref_duals, ref_marginals, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-4
CASES = ["toy1d_staggered", "toy1d_safe", "toy1d_swift", "mix16_staggered", "mix16_warm",
         "mix32_staggered", "mix16_zeros", "pr1_64"]


@pytest.mark.parametrize("name", CASES)
def test_fp32_mode_within_1e4_of_reference(name):
    from _engine_run import box4, problem_from_golden
    import warnings
    from paper_2410_08859_b200.decomposition import make_decomposition
    from paper_2410_08859_b200.engine import (CellSolverConfig, EngineConfig, StrategyConfig,
                                              domdec_solve, warm_start_plan)
    from _golden import cell_cap

    g = load(name)
    prob = problem_from_golden(g)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(prob.mu, int(g["s"]))
    cfg = EngineConfig(delta=float(g["delta"]), max_iters=int(g["max_iters"]),
                       cell=CellSolverConfig(max_iters=cell_cap(g), precision="fp32"),
                       cell_delta_factor=float(g["cell_delta_factor"]) if "cell_delta_factor" in g
                       else 0.25)
    state = warm_start_plan(prob, dec, delta=1e-3) if bool(g["warm"]) else None
    st, rep = domdec_solve(prob, dec, StrategyConfig(kind=str(g["strategy"])), cfg, state=state)
    got = rep.final_score["total"]
    assert abs(got - float(g["score"][-1])) <= TOL * abs(float(g["score"][-1]))
    shape = prob.nu.mass.reshape(1, -1).shape if prob.nu.grid.ndim == 1 else prob.nu.mass.shape
    nu_i = st.nu_i
    mine = np.zeros(shape)
    ref = np.zeros(shape)
    worst = 0.0
    for i, (box, vals) in enumerate(ref_marginals(g)):
        b = box4(nu_i[i].box)
        m = dense(b, nu_i[i].values.reshape(b[1], b[3]) if b[1] else np.zeros((0, 0)), shape)
        r = dense(box, vals, shape)
        worst = max(worst, rel_err(m, r))
        mine += m
        ref += r
    assert worst < TOL, worst
    assert rel_err(mine, ref) < TOL
    duals = st.duals
    for key, (a, bb, b) in ref_duals(g).items():
        d = duals[key]
        assert rel_err(d.alpha, a) < TOL, key
