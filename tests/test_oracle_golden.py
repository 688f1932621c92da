"""Pin the CPU oracle against fixtures produced by running the reference itself.

The fixtures come from ``scripts/make_golden.py`` (reference package
imported from its source tree in the build container).  CPU only.
"""

import numpy as np
import pytest

from oracle import ref_lse
from oracle.ref_problem import make_ctx
from oracle.ref_sweep import CellCfg, EngCfg, StratCfg, solve, warm_state

from _golden import ENGINE_CASES, cell_cap, dense, load, ref_duals, ref_marginals, rel_err, scalar


def test_newton_grid_matches_reference():
    g = load("newton_grid")
    for k in range(g["z"].size):
        b, _ = ref_lse.newton_y(g["z"][k:k + 1], g["m"][k:k + 1], float(g["eps"][k]),
                                float(g["lam"][k]), np.zeros(1))
        assert b[0] == pytest.approx(g["beta"][k], rel=1e-13, abs=1e-300)


def test_separable_sweep_matches_reference():
    g = load("separable_sweep")
    ker = ref_lse.GridKernel([g["xa0"], g["xa1"]], [g["ya0"], g["ya1"]], float(g["eps"]))
    assert rel_err(ker.lse_x(g["v"]), g["lse_x"]) < 1e-14
    assert rel_err(ker.lse_y(g["v"]), g["lse_y"]) < 1e-14


def test_global_sinkhorn_matches_reference():
    g = load("global_sinkhorn")
    n = g["mu"].shape[0]
    ax = float(g["origin"][0]) + float(g["dx"]) * np.arange(n)
    ker = ref_lse.GridKernel([ax, ax], [ax, ax], float(g["eps"]))
    r = ref_lse.global_sinkhorn(ker, g["mu"], g["nu"], None, np.zeros((n, n)), np.zeros((n, n)),
                                float(g["lam"]), float(g["delta"]))
    assert r["iterations"] == int(g["iterations"])
    assert rel_err(r["alpha"], g["alpha"]) < 1e-12
    assert rel_err(r["beta"], g["beta"]) < 1e-12


def oracle_run(g):
    mu, nu = g["mu"], g["nu"]
    ctx = make_ctx(mu, nu, float(g["dx"]), tuple(g["origin"]), float(g["lam"]), float(g["eps"]),
                   int(g["s"]))
    st = warm_state(ctx, delta=1e-3) if bool(g["warm"]) else None
    cfg = EngCfg(delta=float(g["delta"]), max_iters=int(g["max_iters"]),
                 cell=CellCfg(max_iters=cell_cap(g)))
    return ctx, solve(ctx, st, StratCfg(kind=str(g["strategy"])), cfg)


@pytest.mark.parametrize("name", ENGINE_CASES)
def test_engine_matches_reference(name):
    g = load(name)
    ctx, (st, rep, trace) = oracle_run(g)
    assert rep["iterations"] == int(g["iterations"])
    assert bool(rep["converged"]) == bool(g["converged"])
    assert [t["action"] for t in trace] == [str(a) for a in g["trace_action"]]
    np.testing.assert_allclose([t["total"] for t in trace], g["trace_total"], rtol=1e-10)
    sc = rep["final_score"]
    got = np.array([sc["transport"], sc["entropy"], sc["d1"], sc["d2"], sc["total"]])
    np.testing.assert_allclose(got, g["score"], rtol=1e-10, atol=1e-15)
    shape = ctx.nu.shape
    for i, (box, vals) in enumerate(ref_marginals(g)):
        assert tuple(st.box[i]) == box, f"cell {i} box"
        assert rel_err(dense(st.box[i], st.vals[i], shape), dense(box, vals, shape)) < 1e-9
    duals = ref_duals(g)
    assert set(duals) == set(st.duals)
    for key, (a, bb, b) in duals.items():
        oa, ob_box, ob = st.duals[key]
        assert tuple(ob_box) == bb
        assert rel_err(oa, a) < 1e-9
        assert rel_err(ob, b) < 1e-9
    np.testing.assert_allclose(st.transport, g["transport"], rtol=1e-9, atol=1e-18)
    np.testing.assert_allclose(st.kl, g["kl"], rtol=1e-9, atol=1e-15)
    assert rep["rel_pd_gap"] == pytest.approx(scalar(g, "rel_pd_gap"), rel=1e-6, abs=1e-12)


def test_pr1_64_fixture_is_baseline_configs0():
    """The configs[0] golden fixture was produced by the reference on exactly the
    bench/problem generator's input (64^2, 3 Gaussians + 1e-4 floor, masses 1.0/1.3,
    lam = 1, eps = 2h^2, 4x4 cells, 30 sweeps)."""
    from paper_2410_08859_b200.problems import config_problem_arrays

    g = load("pr1_64")
    mu, nu, dx, org, cfg = config_problem_arrays(0, seed=0)
    assert np.array_equal(g["mu"], mu) and np.array_equal(g["nu"], nu)
    assert float(g["dx"]) == dx and float(g["lam"]) == cfg["lam"] == 1.0
    assert float(g["eps"]) == 2 * dx * dx and int(g["s"]) == cfg["cell"] == 4
    assert int(g["iterations"]) == int(g["max_iters"]) == cfg["domdec_sweeps"] == 30
    assert abs(mu.sum() - 1.0) < 1e-12 and abs(nu.sum() - 1.3) < 1e-12
