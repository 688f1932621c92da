"""Kernel-level parity of the CUDA library against reference-generated fixtures."""

import numpy as np
import pytest

from _golden import load, rel_err

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def test_newton_nodes_match_reference_grid():
    import torch
    from paper_2410_08859_b200 import _lib

    g = load("newton_grid")
    n = g["z"].size
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    beta0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    z, m, e, l = (_dev(g[k]) for k in ("z", "m", "eps", "lam"))  # keep alive across the launch
    _lib.check(_lib.lib().dd_newton_nodes(n, z.data_ptr(), m.data_ptr(), beta0.data_ptr(),
                                          e.data_ptr(), l.data_ptr(), 1e-12, 100, out.data_ptr(),
                                          None, _lib.stream_handle()))
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, g["beta"], rtol=1e-12, atol=1e-300)


def _bisect_root(m, z, eps, lam):
    """Bisection oracle for g(b) = log(m + exp(b/eps + z)) + b/lam = 0 (increasing in b),
    run until the bracket is two adjacent doubles."""
    ratio = eps * lam / (eps + lam)
    with np.errstate(divide="ignore"):
        lm = np.log(m)
    hi = np.minimum(-lam * lm, -ratio * z)
    hi = hi + 1e-6 * (1.0 + np.abs(hi))      # rounding margin: g(hi) >= 0 strictly
    lo = hi - lam * np.log(2.0) * 1.01 - 1.0
    g = lambda b: np.logaddexp(lm, b / eps + z) + b / lam  # noqa: E731
    assert np.all(g(lo) <= 0) and np.all(g(hi) >= 0)
    for _ in range(2200):
        mid = 0.5 * (lo + hi)
        up = g(mid) > 0
        hi = np.where(up, mid, hi)
        lo = np.where(up, lo, mid)
        if np.all(np.nextafter(lo, np.inf) >= hi):
            break
    return 0.5 * (lo + hi)


def test_newton_residual_and_bisection_agreement_random():
    """SPEC acceptance criterion 2: on a 10^4-point randomized (m, z, eps, lam)
    grid, residual |g(beta)| <= 1e-12 (scaled), agreement with an independent
    bisection oracle <= 1e-10, and the closed form at m = 0 exact."""
    import torch
    from paper_2410_08859_b200 import _lib

    rng = np.random.default_rng(3)
    n = 10_000
    m = 10.0 ** rng.uniform(-12, 6, n)
    m[::7] = 0.0
    z = rng.uniform(-700, 50, n)
    eps = 10.0 ** rng.uniform(-4, 1, n)
    lam = 10.0 ** rng.uniform(-2, 2, n)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    zd, md, ed, ld = _dev(z), _dev(m), _dev(eps), _dev(lam)
    _lib.check(_lib.lib().dd_newton_nodes(n, zd.data_ptr(), md.data_ptr(), None, ed.data_ptr(),
                                          ld.data_ptr(), 1e-12, 100, out.data_ptr(), None,
                                          _lib.stream_handle()))
    b = out.cpu().numpy()
    gen = m > 0
    res = np.logaddexp(np.log(m[gen]), b[gen] / eps[gen] + z[gen]) + b[gen] / lam[gen]
    assert np.max(np.abs(res)) <= 1e-12 * 10  # residual scale O(1) after the log
    ratio = eps * lam / (eps + lam)
    np.testing.assert_allclose(b[~gen], -ratio[~gen] * z[~gen], rtol=1e-15)
    bis = _bisect_root(m[gen], z[gen], eps[gen], lam[gen])
    err = np.abs(b[gen] - bis) / np.maximum(1.0, np.abs(bis))
    assert err.max() <= 1e-10, err.max()


def test_assemble_is_the_sequential_cell_order_sum_bitwise():
    """dd_assemble (fixed-order gather) equals the reference's assemble_y_marginal
    (measures.py:410-425: zeros, then += each cell's box in index order) bit for bit."""
    import warnings
    from _engine_run import problem_from_golden
    from paper_2410_08859_b200.decomposition import make_decomposition
    from paper_2410_08859_b200.engine import warm_start_plan

    g = load("mix32_staggered")
    prob = problem_from_golden(g)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(prob.mu, int(g["s"]))
    st = warm_start_plan(prob, dec, delta=1e-3)
    got = st.assemble_device().cpu().numpy().reshape(prob.nu.mass.shape)
    want = np.zeros(prob.nu.mass.shape)
    for m in st.nu_i:
        if m.is_empty:
            continue
        want[tuple(slice(o, o + e) for o, e in m.box)] += m.values
    assert np.array_equal(got, want)


def test_grid_sweeps_match_reference():
    import torch
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.sinkhorn import GridSweeper

    g = load("separable_sweep")
    v = g["v"]

    class DP:  # minimal device-problem stand-in for the sweeper
        pass

    dp = DP()
    dp.device = torch.device("cuda")
    n0, n1 = v.shape
    dp.geom = _lib.Geom(nx0=n0, nx1=n1, ny0=n0, ny1=n1, x_dx=float(g["xa0"][1] - g["xa0"][0]),
                        x_org0=float(g["xa0"][0]), x_org1=float(g["xa1"][0]),
                        y_dx=float(g["ya0"][1] - g["ya0"][0]), y_org0=float(g["ya0"][0]),
                        y_org1=float(g["ya1"][0]), eps=float(g["eps"]), lam=1.0, nu_total=1.0)
    dp.nx = dp.ny = v.size
    dp.empty_x = lambda: torch.empty(v.size, dtype=torch.float64, device="cuda")
    dp.empty_y = dp.empty_x
    sw = GridSweeper(dp)
    vd = _dev(v.ravel())
    lx = sw.lse_x(vd).cpu().numpy().reshape(v.shape)
    ly = sw.lse_y(vd).cpu().numpy().reshape(v.shape)
    assert rel_err(lx, g["lse_x"]) < 1e-13
    assert rel_err(ly, g["lse_y"]) < 1e-13


def test_global_sinkhorn_matches_reference():
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.sinkhorn import DeviceProblem, SolverConfig, sinkhorn_solve

    g = load("global_sinkhorn")
    n = g["mu"].shape[0]
    grid = Grid((n, n), float(g["dx"]), tuple(g["origin"]))
    prob = TransportProblem(GridMeasure(grid, g["mu"]), GridMeasure(grid, g["nu"]),
                            DivergenceSpec(float(g["lam"])), float(g["eps"]))
    dp = DeviceProblem(prob)
    r = sinkhorn_solve(dp, config=SolverConfig(delta=float(g["delta"])))
    assert r.iterations == int(g["iterations"])
    assert rel_err(r.alpha.cpu().numpy().reshape(n, n), g["alpha"]) < 1e-10
    assert rel_err(r.beta.cpu().numpy().reshape(n, n), g["beta"]) < 1e-10
    assert r.gap == pytest.approx(float(g["gap"]), rel=1e-8)


def test_cut_plan_2d_kernel_matches_embedded_three_axis_cut():
    """The 2D per-term plan cut (dd_cut_plan, every term of the full Y grid) and the
    three-axis separable cut the warm start uses on the (1, n0, n1) embedding agree:
    same boxes, marginals / X-marginals / fragments to 1e-12."""
    import warnings

    import torch
    from _engine_run import problem_from_golden
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.decomposition import make_decomposition
    from paper_2410_08859_b200.engine import PlanState, _cut_plan_embedded
    from paper_2410_08859_b200.sinkhorn import DeviceProblem, SolverConfig, sinkhorn_solve

    g = load("mix32_staggered")
    prob = problem_from_golden(g)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(prob.mu, int(g["s"]))
    dp = DeviceProblem(prob)
    res = sinkhorn_solve(dp, config=SolverConfig(delta=1e-3))
    a = PlanState(prob, dec.basic, dp, cap=1)
    tr_a = torch.zeros(a.n_basic, dtype=torch.float64, device="cuda")
    boxes = torch.zeros(a.n_basic * 4, dtype=torch.int32, device="cuda")
    L = _lib.lib()
    s = a.state_struct()
    s.yval = None
    _lib.check(L.dd_cut_plan(dp.geom, s, res.alpha.data_ptr(), res.beta.data_ptr(), 1e-15,
                             tr_a.data_ptr(), boxes.data_ptr(), _lib.stream_handle()))
    bh = boxes.view(-1, 4).cpu().numpy()
    a.ensure_cap(int((bh[:, 1].astype(np.int64) * bh[:, 3]).max(initial=1)))
    _lib.check(L.dd_cut_plan(dp.geom, a.state_struct(), res.alpha.data_ptr(), res.beta.data_ptr(),
                             1e-15, tr_a.data_ptr(), boxes.data_ptr(), _lib.stream_handle()))
    b = PlanState(prob, dec.basic, dp, cap=1)
    tr_b = torch.zeros(b.n_basic, dtype=torch.float64, device="cuda")
    _cut_plan_embedded(b, dp, res.alpha, res.beta, 1e-15, tr_b)
    assert np.array_equal(a.ybox.cpu().numpy(), b.ybox.cpu().numpy())
    for ma, mb in zip(a.nu_i, b.nu_i):
        assert ma.box == mb.box
        if not ma.is_empty:
            assert rel_err(mb.values, ma.values) < 1e-12
    assert rel_err(b.x_marg_d.cpu().numpy(), a.x_marg_d.cpu().numpy()) < 1e-12
    assert rel_err(b.transport, a.transport) < 1e-12
    assert rel_err(b.kl, a.kl) < 1e-12
