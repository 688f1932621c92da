"""Parity at the BASELINE configurations' own scale (configs[2], 1024^2).

The SPEC multiscale driver runs ms_1024 on the GPU up to the start of the
1024^2 stage.  The first staggered batch of partition A is then solved on the
device, and a sample of its composite cells is re-solved by the CPU oracle (a
restatement of the reference cells.py) from the identical inputs: the same
plan state, the same assembled snapshot and the same warm duals.  The sample
takes the largest windows, cells that hit the iteration cap and cells that
converge.  The batch runs under every execution path: the default size rule,
the global-memory workspace, forced 4-CTA clusters, and a 48 KB per-CTA budget
under which the size rule itself sends the larger windows to 2..16-CTA
thread-block clusters (at this stage every window fits one SM's 220 KB).  To
keep the oracle within seconds the cell iteration cap is lowered to 200 on
both sides (the cap is a reference configuration parameter,
CellSolverConfig.max_iters).

Tolerances (north_star, fp64): member marginals and duals within 1e-9
relative, fragments within 1e-9, iteration counts and convergence flags equal.
"""

import time
import warnings
from types import SimpleNamespace

import numpy as np
import pytest

from _golden import rel_err

pytestmark = pytest.mark.gpu

CAP = 200


def _capture_1024_stage():
    import paper_2410_08859_b200.multiscale as M
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.problems import config_problem_arrays

    mu, nu, dx, org, cfg = config_problem_arrays(2, seed=0)
    h2 = dx * dx
    grid = Grid(mu.shape, dx, org)
    prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu),
                            DivergenceSpec(cfg["lam"]), 2 * h2)
    captured = {}
    orig = M.domdec_solve

    def hook(problem, dec, strategy, config, state=None, evaluator=None):
        if problem.mu.grid.dims[0] == 1024:
            captured.update(state=state, problem=problem, dec=dec)
            raise StopIteration
        return orig(problem, dec, strategy, config, state=state, evaluator=evaluator)

    M.domdec_solve = hook
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            M.multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2)
    except StopIteration:
        pass
    finally:
        M.domdec_solve = orig
    return captured, mu, nu, dx, org, cfg


MODES = {"default": {},
         "split": {"split_loop": True},    # 1024 cells >= 3 x 148: loop kernel + epilogue
         "global_ws": {"force_global_ws": True}, "cluster4": {"force_cluster": 4},
         # 48 KB per CTA: the size rule sends the larger windows to 2..16-CTA clusters
         "small_smem": {"smem_budget": 48 * 1024},
         # north_star fp32 mode against the fp64 oracle at 1e-4
         "fp32": {}}


@pytest.mark.parametrize("mode", sorted(MODES))
def test_1024_batch_cells_match_oracle(mode):
    import torch
    from paper_2410_08859_b200.engine import (CellSolverConfig, _Batch, _tables, set_exec_mode)
    from oracle.ref_cell import prepare, solve_batch
    from oracle.ref_problem import make_ctx
    from oracle.ref_sweep import CellCfg

    cap, mu, nu, dx, org, cfg = _capture_1024_stage()
    st, prob, dec = cap["state"], cap["problem"], cap["dec"]
    part = dec.composites[0]
    pt = _tables(part)
    ids = np.asarray(pt.batches[0])
    delta = 2e-5 * 0.25
    ccfg = CellSolverConfig(delta=delta, max_iters=CAP,
                            precision="fp32" if mode == "fp32" else "fp64")
    tol = 1e-4 if mode == "fp32" else 1e-9
    prev = set_exec_mode(**MODES[mode])
    try:
        snap = st.assemble_device()
        # host mirrors of the inputs, taken before the commit changes the state
        boxes = [tuple(int(x) for x in b) for b in st.ybox.view(-1, 4).cpu().numpy()]
        vals_all = st.yval.view(st.n_basic, st.cap).cpu().numpy()
        duals = {}
        for (label, j), d in st.duals.items():
            if label == part.label:
                b = [c for ax in d.beta_box for c in ax]
                duals[(label, j)] = (d.alpha.copy(), tuple(int(x) for x in b), d.beta.copy())
        snap_h = snap.cpu().numpy().reshape(nu.shape)
        bt = _Batch(st, pt, ids, snap, ccfg)
        bt.solve()
        c1, _ = bt.stats()
        n_clu = bt.n_clu
        bt.commit(np.ones(bt.n))
        torch.cuda.synchronize()
    finally:
        set_exec_mode(prev)
    if mode in ("small_smem", "cluster4"):
        assert n_clu > 0, "no cell of the 1024^2 batch took the cluster path"
    if mode == "split":
        assert bt.n_split > 0, "the 1024-cell batch did not take the split loop kernel"
    if mode == "small_smem":
        assert len(bt.clu_groups) >= 2, "expected several natural cluster sizes"
    iters = c1[:, 2].astype(int)
    ny = bt.ny
    # sample: the two largest windows, two capped median-size cells, two converged cells
    order = np.argsort(-ny, kind="stable")
    pick = list(order[:2])
    capped = [k for k in np.argsort(np.abs(ny - np.median(ny)), kind="stable") if iters[k] >= CAP]
    quick = [k for k in np.argsort(np.abs(ny - np.median(ny)), kind="stable")
             if 2 <= iters[k] < CAP]
    pick += [k for k in capped if k not in pick][:2] + [k for k in quick if k not in pick][:2]
    assert len(pick) >= 5
    ctx = make_ctx(mu, nu, dx, org, cfg["lam"], prob.eps, cfg["cell"])
    opart = [p for p in ctx.parts if p["label"] == part.label][0]
    vals = [vals_all[i, :b[1] * b[3]].reshape(b[1], b[3]) if b[1] and b[3] else np.zeros((0, 0))
            for i, b in enumerate(boxes)]
    ost = SimpleNamespace(box=[b if b[1] and b[3] else (0, 0, 0, 0) for b in boxes], vals=vals,
                          duals=duals)
    ocfg = CellCfg(delta=delta, max_iters=CAP)
    gd = st.duals
    nu_i = st.nu_i
    xm = st.x_marg
    t0 = time.perf_counter()
    for k in pick:
        j = int(ids[k])
        probs = prepare(ctx, opart, [j], ost, snap_h)
        sol = solve_batch(probs, ctx, ocfg)[0]
        if mode != "fp32":
            assert sol.iterations == iters[k], (j, sol.iterations, iters[k])
            assert bool(sol.converged) == bool(c1[k, 3]), j
        d = gd[(part.label, j)]
        assert rel_err(d.alpha, sol.alpha) < tol, j
        if mode != "fp32" or d.beta.shape == sol.beta.shape:
            assert rel_err(d.beta, sol.beta) < tol, j
        for q, i in enumerate(sol.members):
            ob = tuple(int(x) for x in sol.new_box[q])
            g = nu_i[i]
            if ob[1] == 0 or ob[3] == 0:
                assert g.is_empty
                continue
            gb = tuple(c for ax in g.box for c in ax)
            if mode == "fp32":
                # truncation at 1e-15 may keep or drop an edge row: compare on the union
                shp = (1, nu.shape[1]) if nu.ndim == 1 else nu.shape
                a = np.zeros(shp)
                a[gb[0]:gb[0] + gb[1], gb[2]:gb[2] + gb[3]] = g.values.reshape(gb[1], gb[3])
                o = np.zeros(shp)
                o[ob[0]:ob[0] + ob[1], ob[2]:ob[2] + ob[3]] = sol.new_vals[q]
                assert rel_err(a, o) < tol, (j, i)
                assert rel_err(xm[i], sol.x_marg[q]) < tol, (j, i)
                continue
            assert gb == ob, (j, i)
            assert rel_err(g.values, sol.new_vals[q]) < tol, (j, i)
            assert rel_err(xm[i], sol.x_marg[q]) < tol, (j, i)
        np.testing.assert_allclose(st.transport[sol.members], sol.transport, rtol=tol, atol=1e-18)
        np.testing.assert_allclose(st.kl[sol.members], sol.kl, rtol=tol, atol=1e-15)
    print(f"oracle time for {len(pick)} cells: {time.perf_counter() - t0:.1f}s; "
          f"windows {[int(ny[k]) for k in pick]}, iterations {[int(iters[k]) for k in pick]}")


def test_ms256_multiscale_matches_reference_on_its_switch_layer():
    """BASELINE configs[1] end to end: the GPU's SPEC multiscale solve of ms_256
    against the REFERENCE's warm_start_plan + domdec_solve on the 256^2 switch
    layer, started from the duals the GPU's global Sinkhorn layers hand over
    (scripts/dump_ms256_switch.py -> scripts/make_golden.py ms256).  fp64
    tolerances: marginals and duals 1e-9, objective 1e-10, iterations and
    actions exact."""
    import os
    from _golden import GOLDEN, dense, ref_duals, ref_marginals
    from _engine_run import box4
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.multiscale import multiscale_solve
    from paper_2410_08859_b200.problems import config_problem_arrays

    if not os.path.exists(os.path.join(GOLDEN, "ms256_final.npz")):
        pytest.skip("ms256_final fixture not generated")
    from _golden import load
    g = load("ms256_final")
    mu, nu, dx, org, cfg = config_problem_arrays(1, seed=0)
    assert np.array_equal(mu, g["mu"]) and np.array_equal(nu, g["nu"])
    h2 = dx * dx
    prob = TransportProblem(GridMeasure(Grid(mu.shape, dx, org), mu),
                            GridMeasure(Grid(mu.shape, dx, org), nu),
                            DivergenceSpec(cfg["lam"]), 2 * h2)
    st, rep = multiscale_solve(prob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2)
    r = rep.stages[-1][2]
    assert r.iterations == int(g["iterations"])
    assert [t.action for t in r.trace] == [str(a) for a in g["trace_action"]]
    np.testing.assert_allclose([t.total for t in r.trace], g["trace_total"], rtol=1e-10)
    shape = mu.shape
    nu_i = st.nu_i
    for i, (box, vals) in enumerate(ref_marginals(g)):
        b = box4(nu_i[i].box)
        assert b == box, i
        mine = dense(b, nu_i[i].values.reshape(b[1], b[3]) if b[1] else np.zeros((0, 0)), shape)
        assert rel_err(mine, dense(box, vals, shape)) < 1e-9, i
    duals = st.duals
    for key, (a, bb, b) in ref_duals(g).items():
        assert rel_err(duals[key].alpha, a) < 1e-9, key
        assert rel_err(duals[key].beta, b) < 1e-9, key
    np.testing.assert_allclose(rep.final_score["total"], g["score"][-1], rtol=1e-10)
