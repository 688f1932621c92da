"""Parity on states produced by the multiscale path.

The multiscale driver (not in the reference source) hands each stage a
refined, partially converged state.  Here the GPU state at the start of the
finest stage is copied into the CPU oracle (a restatement of the reference
engine), both run the same domdec stage, and their results are compared with
the BASELINE tolerances.  Also checks mass accounting of the refinement.
"""

import warnings

import numpy as np
import pytest

from _golden import rel_err

pytestmark = pytest.mark.gpu


def _oracle_state(st, ctx):
    from oracle.ref_sweep import OState

    boxes = [tuple(int(x) for x in b) for b in st.ybox.view(-1, 4).cpu().numpy()]
    vals_all = st.yval.view(st.n_basic, st.cap).cpu().numpy()
    vals = [vals_all[i, :b[1] * b[3]].reshape(b[1], b[3]).copy() for i, b in enumerate(boxes)]
    boxes = [b if b[1] and b[3] else (0, 0, 0, 0) for b in boxes]
    duals = {}
    for (label, j), d in st.duals.items():
        b = [c for ax in d.beta_box for c in ax]
        duals[(label, j)] = (d.alpha.copy(), tuple(int(x) for x in b), d.beta.copy())
    gd = None
    if st.global_duals is not None:
        gd = (st.global_duals[0].cpu().numpy().reshape(ctx.mu.shape),
              st.global_duals[1].cpu().numpy().reshape(ctx.nu.shape))
    return OState(box=boxes, vals=vals, x_marg=[x.copy() for x in st.x_marg],
                  mu_nodes=[m.copy() for m in st.mu_nodes], transport=st.transport.copy(),
                  kl=st.kl.copy(), duals=duals, truncated_mass=st.truncated_mass,
                  global_duals=gd)


def test_finest_stage_matches_oracle_from_refined_state():
    import paper_2410_08859_b200.multiscale as M
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.engine import EngineConfig, StrategyConfig, domdec_solve
    from paper_2410_08859_b200.problems import config_problem_arrays
    from oracle.ref_problem import make_ctx
    from oracle.ref_sweep import EngCfg, StratCfg, solve

    mu, nu, dx, org, cfg = config_problem_arrays(1, seed=3, n=64)
    h2 = dx * dx
    grid = Grid(mu.shape, dx, org)
    prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu),
                            DivergenceSpec(cfg["lam"]), 2 * h2)
    captured = {}
    orig = M.domdec_solve

    def hook(problem, dec, strategy, config, state=None, evaluator=None):
        if problem.mu.grid.dims[0] == 64 and "state" not in captured:
            captured["state"] = state.clone()
            captured["problem"] = problem
            captured["dec"] = dec
            raise StopIteration
        return orig(problem, dec, strategy, config, state=state, evaluator=evaluator)

    M.domdec_solve = hook
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            M.multiscale_solve(prob, 4, 16, 8 * h2, protocol="ladder")
    except StopIteration:
        pass
    finally:
        M.domdec_solve = orig
    st, fprob, dec = captured["state"], captured["problem"], captured["dec"]
    # refinement mass accounting: per-cell masses add up to the coarse plan's total
    ym = st.assemble().mass
    assert ym.sum() + st.truncated_mass == pytest.approx(float(sum(x.sum() for x in st.x_marg))
                                                        + st.truncated_mass, rel=1e-9)
    ctx = make_ctx(mu, nu, dx, org, cfg["lam"], fprob.eps, 4)
    ost = _oracle_state(st, ctx)
    iters = 3
    gst, grep = domdec_solve(fprob, dec, StrategyConfig("staggered"),
                             EngineConfig(max_iters=iters), state=st)
    ost2, orep, otrace = solve(ctx, ost, StratCfg("staggered"), EngCfg(max_iters=iters))
    assert grep.iterations == orep["iterations"]
    np.testing.assert_allclose([r.total for r in grep.trace], [t["total"] for t in otrace],
                               rtol=1e-10)
    shape = ctx.nu.shape
    nu_i = gst.nu_i
    for i in range(len(ost2.box)):
        b = ost2.box[i]
        d_o = np.zeros(shape)
        if b[1] and b[3]:
            d_o[b[0]:b[0] + b[1], b[2]:b[2] + b[3]] = ost2.vals[i]
        g = nu_i[i]
        d_g = np.zeros(shape)
        if not g.is_empty:
            (o0, e0), (o1, e1) = g.box
            d_g[o0:o0 + e0, o1:o1 + e1] = g.values
        assert rel_err(d_g, d_o) < 1e-9, i
    gd = gst.duals
    for key, (a, _, b) in ost2.duals.items():
        assert rel_err(gd[key].alpha, a) < 1e-9
        assert rel_err(gd[key].beta, b) < 1e-9
