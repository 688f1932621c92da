"""Parity of the CUDA engine with the reference (golden fixtures) and the oracle.

Tolerances (BASELINE north_star, fp64): basic-cell marginals and dual
potentials within 1e-9 relative (max-abs error over the array / max-abs of
the reference array), primal-dual objective within 1e-10 relative.
"""

import numpy as np
import pytest

from _golden import ENGINE_CASES, dense, load, ref_duals, ref_marginals, rel_err

pytestmark = pytest.mark.gpu

MARG_TOL = 1e-9
DUAL_TOL = 1e-9
OBJ_TOL = 1e-10

DEVICE_CASES = ENGINE_CASES


@pytest.mark.parametrize("name", DEVICE_CASES)
def test_engine_matches_reference_golden(name):
    from _engine_run import box4, run_device

    g = load(name)
    prob, dec, st, rep = run_device(g)
    assert rep.iterations == int(g["iterations"])
    assert [r.action for r in rep.trace] == [str(a) for a in g["trace_action"]]
    np.testing.assert_allclose([r.total for r in rep.trace], g["trace_total"], rtol=OBJ_TOL)
    sc = rep.final_score
    got = np.array([sc["transport"], sc["entropy"], sc["d1"], sc["d2"], sc["total"]])
    np.testing.assert_allclose(got[-1], g["score"][-1], rtol=OBJ_TOL)
    np.testing.assert_allclose(got, g["score"], rtol=1e-9, atol=1e-14)
    shape = prob.nu.mass.reshape(1, -1).shape if prob.nu.grid.ndim == 1 else prob.nu.mass.shape
    nu_i = st.nu_i
    for i, (box, vals) in enumerate(ref_marginals(g)):
        b = box4(nu_i[i].box)
        assert b == box, f"cell {i}: box {b} != reference {box}"
        mine = dense(b, nu_i[i].values.reshape(b[1], b[3]) if b[1] else np.zeros((0, 0)), shape)
        assert rel_err(mine, dense(box, vals, shape)) < MARG_TOL, f"cell {i}"
    duals = st.duals
    for key, (a, bb, b) in ref_duals(g).items():
        d = duals[key]
        assert box4(d.beta_box) == bb
        assert rel_err(d.alpha, a) < DUAL_TOL, key
        assert rel_err(d.beta, b) < DUAL_TOL, key
    np.testing.assert_allclose(st.transport, g["transport"], rtol=1e-9, atol=1e-18)
    np.testing.assert_allclose(st.kl, g["kl"], rtol=1e-9, atol=1e-15)
    assert rep.rel_pd_gap == pytest.approx(float(g["rel_pd_gap"]), rel=1e-6, abs=1e-12)
