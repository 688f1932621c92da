"""Parity of the three-axis path (volume.py, csrc/vol.cu) with the reference.

* 3D fixtures produced by the reference itself with its two 2D-only guards lifted
  (scripts/make_golden.py ``vol3``: Grid accepts three axes; the separable sweep
  reduces one more axis in its own pattern): every basic-cell marginal and cell
  dual within 1e-9, objectives within 1e-10, iterations and actions exact.
* The same path on the 1D/2D reference fixtures, embedded as (1, n0, n1) /
  (1, 1, n): identical tolerances -- the embedding is exact, so this pins every
  kernel of the three-axis path against the reference's own outputs.
* The full-grid three-axis sweep against the oracle's GridKernel3 (1e-12) and the
  global Sinkhorn's iteration count against the oracle's.
"""

import warnings

import numpy as np
import pytest

from _golden import load, rel_err

pytestmark = pytest.mark.gpu

MARG_TOL = 1e-9
DUAL_TOL = 1e-9
OBJ_TOL = 1e-10
# opt strategy: the blend weights come from the reference's cyclic coordinate descent,
# which stops once no weight moves by more than opt_tol = 1e-9 (engine.py:557-588).  The
# two sides' g/h sums differ in the last ulp, so a sweep can stop one step apart and the
# weights agree only to ~opt_tol; a blended marginal (and the duals stored with it) moves
# linearly with that.  The objective is stationary in theta at the optimum, so it stays
# at OBJ_TOL.
OPT_STATE_TOL = 5e-9

VOL_CASES = ["vol8_staggered", "vol8_safe", "vol8_fast_warm", "vol16_warm", "vol16_cold",
             "vol32_warm", "vol8_swift", "vol8_sequential", "vol16_swift_warm", "vol8_opt",
             "vol16_opt_warm"]
EMBEDDED_CASES = ["toy1d_staggered", "toy1d_safe", "toy1d_fast", "toy1d_swift", "toy1d_sequential",
                  "toy1d_cellcap_swift", "toy1d_opt", "mix16_zeros_warm_opt", "mix16_staggered", "mix16_warm", "mix32_staggered",
                  "mix16_cellcap", "mix16_zeros", "pr1_64"]


def _box6(b):
    b = [int(x) for x in b]
    if len(b) == 2:
        b = [0, 1] + b
    if len(b) == 4:
        b = [0, 1] + b
    if any(b[2 * a + 1] == 0 for a in range(3)):
        return (0,) * 6
    return tuple(b)


def _dense(b6, vals, shape3):
    out = np.zeros(shape3)
    if b6[1] and b6[3] and b6[5]:
        out[b6[0]:b6[0] + b6[1], b6[2]:b6[2] + b6[3], b6[4]:b6[4] + b6[5]] = \
            np.asarray(vals).reshape(b6[1], b6[3], b6[5])
    return out


def _run(g):
    from _engine_run import problem_from_golden
    from _golden import cell_cap
    from paper_2410_08859_b200.decomposition import make_decomposition
    from paper_2410_08859_b200.engine import CellSolverConfig, EngineConfig, StrategyConfig
    from paper_2410_08859_b200.volume import domdec_solve3, warm_start_plan3

    prob = problem_from_golden(g)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(prob.mu, int(g["s"]))
    cfg = EngineConfig(delta=float(g["delta"]), max_iters=int(g["max_iters"]),
                       cell=CellSolverConfig(max_iters=cell_cap(g)),
                       cell_delta_factor=float(g["cell_delta_factor"]) if "cell_delta_factor" in g
                       else 0.25)
    state = warm_start_plan3(prob, dec, delta=1e-3) if bool(g["warm"]) else None
    st, rep = domdec_solve3(prob, dec, StrategyConfig(kind=str(g["strategy"])), cfg, state=state)
    return prob, st, rep


def _check(g, prob, st, rep):
    tol = OPT_STATE_TOL if str(g["strategy"]) == "opt" else MARG_TOL
    assert rep.iterations == int(g["iterations"])
    assert [r.action for r in rep.trace] == [str(a) for a in g["trace_action"]]
    np.testing.assert_allclose([r.total for r in rep.trace], g["trace_total"], rtol=OBJ_TOL)
    sc = rep.final_score
    got = np.array([sc["transport"], sc["entropy"], sc["d1"], sc["d2"], sc["total"]])
    np.testing.assert_allclose(got[-1], g["score"][-1], rtol=OBJ_TOL)
    np.testing.assert_allclose(got, g["score"], rtol=1e-9, atol=1e-14)
    shape3 = st.dp.shape_y
    nu_i = st.nu_i
    offs = g["nu_i_off"]
    for i, rb in enumerate(g["nu_i_box"]):
        want_b = _box6(rb)
        mine_b = _box6([c for ax in nu_i[i].box for c in ax])
        assert mine_b == want_b, f"cell {i}: box {mine_b} != reference {want_b}"
        want = _dense(want_b, g["nu_i_val"][offs[i]:offs[i + 1]], shape3)
        mine = _dense(mine_b, nu_i[i].values, shape3)
        assert rel_err(mine, want) < tol, f"cell {i}"
    duals = st.duals
    for k, key in enumerate(g["dual_keys"]):
        label, j = str(key).split(":")
        d = duals[(label, int(j))]
        a = g["dual_alpha"][g["dual_alpha_off"][k]:g["dual_alpha_off"][k + 1]]
        b = g["dual_beta"][g["dual_beta_off"][k]:g["dual_beta_off"][k + 1]]
        assert _box6([c for ax in d.beta_box for c in ax]) == _box6(g["dual_beta_box"][k])
        assert rel_err(d.alpha, a) < max(tol, DUAL_TOL), key
        assert rel_err(d.beta, b) < max(tol, DUAL_TOL), key
    np.testing.assert_allclose(st.transport, g["transport"], rtol=tol, atol=1e-18)
    np.testing.assert_allclose(st.kl, g["kl"], rtol=tol, atol=1e-15)
    assert rep.rel_pd_gap == pytest.approx(float(g["rel_pd_gap"]), rel=1e-6, abs=1e-12)


@pytest.mark.parametrize("name", VOL_CASES)
def test_volume_engine_matches_reference_3d(name):
    g = load(name)
    prob, st, rep = _run(g)
    assert prob.mu.grid.ndim == 3
    _check(g, prob, st, rep)


@pytest.mark.parametrize("name", EMBEDDED_CASES)
def test_volume_engine_matches_reference_embedded_2d(name):
    g = load(name)
    prob, st, rep = _run(g)
    _check(g, prob, st, rep)


def test_volume_public_api_dispatches_3d():
    """engine.domdec_solve on a 3D problem runs the three-axis path."""
    from _engine_run import run_device
    from paper_2410_08859_b200.volume import PlanState3

    g = load("vol8_staggered")
    prob, dec, st, rep = run_device(g)
    assert isinstance(st, PlanState3)
    _check(g, prob, st, rep)


def test_grid_lse3_matches_oracle():
    import torch

    from oracle.ref_lse import GridKernel3
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.volume import VolumeProblem

    rng = np.random.default_rng(3)
    dims = (6, 9, 7)
    dx = 1.0 / 9
    org = (0.03, 0.01, 0.05)
    eps = 2 * dx * dx
    mu = rng.uniform(0.1, 1.0, dims)
    g = Grid(dims, dx, org)
    prob = TransportProblem(GridMeasure(g, mu), GridMeasure(g, mu * 1.1), DivergenceSpec(1.0), eps)
    dp = VolumeProblem(prob)
    sw = dp.make_sweeper()
    axes = [org[a] + dx * np.arange(dims[a]) for a in range(3)]
    ker = GridKernel3(axes, axes, eps)
    v = rng.normal(0, 3, dims)
    v[0, 0, 0] = -np.inf
    v[2, :, 3] = -40.0          # rows far below the max (exercises the exact fallback)
    vt = torch.from_numpy(v.ravel().copy()).cuda()
    for to_x, want in ((1, ker.lse_x(v)), (0, ker.lse_y(v))):
        got = (sw.lse_x(vt) if to_x else sw.lse_y(vt)).cpu().numpy().reshape(dims)
        assert rel_err(got, want) < 1e-12


def test_global_sinkhorn3_matches_oracle_iterations():
    from oracle.ref_lse import GridKernel3, global_sinkhorn
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.problems import config_problem_arrays
    from paper_2410_08859_b200.sinkhorn import SolverConfig, sinkhorn_solve
    from paper_2410_08859_b200.volume import VolumeProblem

    mu, nu, dx, org, cfg = config_problem_arrays(4, seed=0, n=12)
    eps = 8 * dx * dx
    g = Grid(mu.shape, dx, org)
    prob = TransportProblem(GridMeasure(g, mu), GridMeasure(g, nu), DivergenceSpec(1.0), eps)
    res = sinkhorn_solve(VolumeProblem(prob), config=SolverConfig(delta=1e-6))
    axes = [org[a] + dx * np.arange(12) for a in range(3)]
    ref = global_sinkhorn(GridKernel3(axes, axes, eps), mu, nu, None, np.zeros(mu.shape),
                          np.zeros(mu.shape), 1.0, 1e-6)
    assert res.iterations == ref["iterations"]
    assert rel_err(res.alpha.cpu().numpy(), ref["alpha"].ravel()) < 1e-10
    assert rel_err(res.beta.cpu().numpy(), ref["beta"].ravel()) < 1e-10


def test_volume_multiscale_converges_configs4_reduced():
    """configs[4]'s generator and schedule at 32^3 (16^3 -> 32^3): SPEC multiscale
    (global Sinkhorn on 16^3, warm start + domdec at 32^3) converges."""
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.engine import EngineConfig
    from paper_2410_08859_b200.multiscale import multiscale_solve
    from paper_2410_08859_b200.problems import config_problem_arrays

    mu, nu, dx, org, cfg = config_problem_arrays(4, seed=0, n=32)
    h2 = dx * dx
    g = Grid(mu.shape, dx, org)
    prob = TransportProblem(GridMeasure(g, mu), GridMeasure(g, nu), DivergenceSpec(cfg["lam"]),
                            2 * h2)
    st, rep = multiscale_solve(prob, cfg["cell"], 16, cfg["eps_start_h2"] * h2,
                               config=EngineConfig(delta=2e-5))
    assert rep.converged
    assert np.isfinite(rep.final_score["total"])
    y = st.assemble().mass
    assert y.shape == (32, 32, 32) and abs(y.sum() - float(np.sum(nu))) < 0.2 * nu.sum()
