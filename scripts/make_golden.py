"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python scripts/make_golden.py

Writes tests/golden/<case>.npz.  Each fixture stores the inputs (mu, nu,
grid spacing/origin, lam, eps, cell size, strategy, engine tolerances,
iteration cap) and the reference's outputs after ``domdec_solve``:

* per-basic-cell Y-marginals (boxes + concatenated values),
* per-cell transport / KL fragments and the x-marginals,
* the final score breakdown, the relative PD gap and the trace totals/gaps,
* the stored cell duals of both partitions (alpha, beta box, beta).

Plus kernel-level fixtures: a Newton Y-step grid, a separable full-grid
sweep pair and one global Sinkhorn solve.
"""

from __future__ import annotations

import os
import sys
import warnings
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def _import_ref():
    sys.path.insert(0, str(REF))
    import domdec.engine as eng  # noqa: F401
    import domdec.measures as meas  # noqa: F401
    import domdec.sinkhorn as sk  # noqa: F401
    return eng, meas, sk


def _mixture(grid_dims, dx, origin, rng, n_bumps, floor_rel=1e-8):
    axes = [origin[a] + dx * np.arange(grid_dims[a], dtype=np.float64) for a in range(len(grid_dims))]
    dens = np.zeros(grid_dims)
    for _ in range(n_bumps):
        c = rng.uniform(0.15, 0.85, size=len(grid_dims))
        sig = rng.uniform(0.04, 0.15)
        w = rng.uniform(0.5, 1.5)
        q = np.zeros(grid_dims)
        for a, xs in enumerate(axes):
            shape = [1] * len(grid_dims)
            shape[a] = xs.size
            q = q + ((xs - c[a]) ** 2).reshape(shape)
        dens += w * np.exp(-q / (2.0 * sig * sig))
    dens = np.maximum(dens, floor_rel * dens.mean())
    return dens / dens.sum()


CASES = [
    # name, dims, s, lam, eps (None -> 2 dx^2), strategy, delta, max_iters, warm, nu_scale
    dict(name="toy1d_staggered", dims=(32,), s=1, lam=1.0, strategy="staggered", delta=1e-6,
         max_iters=40, warm=False, seed=0, uniform=True),
    dict(name="toy1d_safe", dims=(16,), s=2, lam=0.5, strategy="safe", delta=1e-6,
         max_iters=12, warm=False, seed=0, uniform=False),
    dict(name="toy1d_swift", dims=(16,), s=2, lam=1.0, strategy="swift", delta=1e-6,
         max_iters=12, warm=False, seed=1, uniform=False),
    dict(name="toy1d_opt", dims=(16,), s=1, lam=1.0, strategy="opt", delta=1e-6,
         max_iters=8, warm=False, seed=2, uniform=False),
    dict(name="toy1d_sequential", dims=(16,), s=2, lam=1.0, strategy="sequential", delta=1e-6,
         max_iters=10, warm=False, seed=3, uniform=False),
    dict(name="toy1d_fast", dims=(16,), s=1, lam=1.0, strategy="fast", delta=1e-6,
         max_iters=10, warm=False, seed=4, uniform=False),
    dict(name="mix16_staggered", dims=(16, 16), s=4, lam=1.0, strategy="staggered", delta=1e-5,
         max_iters=12, warm=False, seed=5, uniform=False),
    dict(name="mix16_warm", dims=(16, 16), s=2, lam=1.0, strategy="staggered", delta=1e-6,
         max_iters=10, warm=True, seed=6, uniform=False, nu_scale=1.3),
    dict(name="mix32_staggered", dims=(32, 32), s=4, lam=0.5, strategy="staggered", delta=1e-6,
         max_iters=6, warm=True, seed=7, uniform=False, nu_scale=0.8),
    # cell iteration cap hit on every solve (non-converged cells, final recompute path)
    dict(name="mix16_cellcap", dims=(16, 16), s=4, lam=1.0, strategy="staggered", delta=1e-7,
         max_iters=4, warm=False, seed=8, uniform=False, nu_scale=1.2, cell_max_iters=7),
    dict(name="toy1d_cellcap_swift", dims=(16,), s=2, lam=2.0, strategy="swift", delta=1e-8,
         max_iters=5, warm=False, seed=9, uniform=False, cell_max_iters=3),
    # zero-mass mu regions: dropped basic cells, padded composites, zero nodes inside cells
    dict(name="mix16_zeros", dims=(16, 16), s=2, lam=1.0, strategy="staggered", delta=1e-6,
         max_iters=8, warm=False, seed=10, uniform=False, zero_mu=True),
    dict(name="mix16_zeros_warm_opt", dims=(16, 16), s=4, lam=0.7, strategy="opt", delta=1e-6,
         max_iters=4, warm=True, seed=11, uniform=False, zero_mu=True, nu_scale=1.1),
]

# BASELINE.json configs[0] (the PR1 correctness model) on its own generator
# (paper_2410_08859_b200.problems.config_problem_arrays(0, seed=0): 64^2, 3
# Gaussians + 1e-4 floor, masses 1.0 / 1.3), lam = 1, eps = 2h^2, 4x4 basic
# cells, staggered, warm start (reference warm_start_plan, delta 1e-3), exactly
# 30 domdec sweeps (global delta 1e-12 never stops early) with the cell
# Sinkhorn tolerance 1e-7 (cell_delta_factor 1e5).  Slow: ~1 h of reference CPU.
BASELINE_CASES = [
    dict(name="pr1_64", baseline=0, s=4, lam=1.0, strategy="staggered", delta=1e-12,
         cell_delta_factor=1e5, max_iters=30, warm=True, seed=0),
]


# Three-axis cases (BASELINE configs[4] generator at reduced sizes).  The reference is
# dimension-generic except for two guards, lifted here and nowhere else:
#   * measures.Grid.__post_init__ rejects more than 2 axes (measures.py:76-77);
#   * sinkhorn.SeparableKernel._sweep reduces at most 2 axes (sinkhorn.py:159-175) --
#     extended by one axis in its own pattern (last axis first, one _lse per axis).
# Everything else (partitions, cells, engine) runs unmodified.
VOL_CASES = [
    dict(name="vol8_staggered", n=8, s=2, lam=1.0, strategy="staggered", delta=1e-5,
         max_iters=6, warm=False, seed=0),
    dict(name="vol8_safe", n=8, s=2, lam=0.7, strategy="safe", delta=1e-5, max_iters=4,
         warm=False, seed=1),
    dict(name="vol8_fast_warm", n=8, s=2, lam=1.0, strategy="fast", delta=1e-5, max_iters=4,
         warm=True, seed=2),
    dict(name="vol16_warm", n=16, s=4, lam=1.0, strategy="staggered", delta=2e-5, max_iters=4,
         warm=True, seed=3),
    dict(name="vol16_cold", n=16, s=4, lam=1.0, strategy="staggered", delta=1e-5, max_iters=6,
         warm=False, seed=4),
    dict(name="vol32_warm", n=32, s=4, lam=1.0, strategy="staggered", delta=2e-5, max_iters=4,
         warm=True, seed=5),
    dict(name="vol8_swift", n=8, s=2, lam=0.8, strategy="swift", delta=1e-5, max_iters=4,
         warm=False, seed=6),
    dict(name="vol8_sequential", n=8, s=2, lam=1.0, strategy="sequential", delta=1e-5,
         max_iters=4, warm=False, seed=7),
    dict(name="vol16_swift_warm", n=16, s=4, lam=1.0, strategy="swift", delta=2e-5,
         max_iters=3, warm=True, seed=8),
    dict(name="vol8_opt", n=8, s=2, lam=0.8, strategy="opt", delta=1e-5, max_iters=4,
         warm=False, seed=9),
    dict(name="vol16_opt_warm", n=16, s=4, lam=1.0, strategy="opt", delta=2e-5, max_iters=2,
         warm=True, seed=10),
]


def lift_3d_guards(meas, sk):
    grid_init = meas.Grid.__post_init__

    def post_init(self):
        if len(self.dims) == 3:
            object.__setattr__(self, "dims", tuple(int(n) for n in self.dims))
            object.__setattr__(self, "origin", tuple(float(o) for o in self.origin))
            object.__setattr__(self, "dx", float(self.dx))
            return
        grid_init(self)

    meas.Grid.__post_init__ = post_init
    sweep2 = sk.SeparableKernel._sweep

    def sweep(self, v, to_x):
        tables = self._neg_sq if to_x else [t.T for t in self._neg_sq]
        if len(tables) != 3:
            return sweep2(self, v, to_x)
        t0, t1, t2 = tables
        v = np.asarray(v, dtype=np.float64)
        a = sk._lse(v[:, :, None, :] + t2[None, None, :, :], axis=3)       # (m0, m1, n2)
        b = sk._lse(a[:, None, :, :] + t1[None, :, :, None], axis=2)       # (m0, n1, n2)
        return sk._lse(b[None, :, :, :] + t0[:, :, None, None], axis=1)    # (n0, n1, n2)

    sk.SeparableKernel._sweep = sweep


def run_vol_case(eng, meas, c):
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2410_08859_b200.problems import config_problem_arrays
    mu, nu, dx, origin, _ = config_problem_arrays(4, seed=c["seed"], n=c["n"])
    eps = 2.0 * dx * dx
    grid = meas.Grid(mu.shape, dx=dx, origin=origin)
    prob = meas.TransportProblem(
        mu=meas.GridMeasure(grid, mu), nu=meas.GridMeasure(grid, nu),
        div=meas.DivergenceSpec(lam=c["lam"]), eps=eps)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = eng.make_decomposition(prob.mu, c["s"])
    cfg = eng.EngineConfig(delta=c["delta"], max_iters=c["max_iters"])
    state = eng.warm_start_plan(prob, dec, delta=1e-3) if c["warm"] else None
    st, rep = eng.domdec_solve(prob, dec, eng.StrategyConfig(kind=c["strategy"]), cfg, state=state)
    out = dict(mu=mu, nu=nu, dx=dx, origin=np.array(origin), lam=c["lam"], eps=eps, s=c["s"],
               cell_max_iters=10_000, strategy=c["strategy"], delta=c["delta"],
               max_iters=c["max_iters"], warm=c["warm"], cell_delta_factor=0.25)
    return _outputs(st, rep, out)


def run_case(eng, meas, c):
    if "baseline" in c:
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from paper_2410_08859_b200.problems import config_problem_arrays
        mu, nu, dx, origin, _ = config_problem_arrays(c["baseline"], seed=c["seed"])
        dims = mu.shape
    else:
        dims = c["dims"]
        n = dims[0] if len(dims) == 1 else dims[0]
        dx = 1.0 / n
        origin = tuple(0.5 * dx for _ in dims)
        rng = np.random.default_rng(c["seed"])
    if "baseline" in c:
        pass
    elif c.get("uniform"):
        origin = tuple(0.0 for _ in dims)
        mu = np.full(dims, 1.0 / np.prod(dims))
        nu = np.full(dims, 1.0 / np.prod(dims))
    else:
        mu = _mixture(dims, dx, origin, rng, 3)
        nu = _mixture(dims, dx, origin, rng, 3) * c.get("nu_scale", 1.0)
        if c.get("zero_mu"):
            mu[4:8, 8:12] = 0.0            # a whole block (dropped basic cells)
            mu[rng.uniform(size=dims) < 0.05] = 0.0   # scattered zero nodes
            mu = mu / mu.sum()
    eps = 2.0 * dx * dx
    grid = meas.Grid(dims, dx=dx, origin=origin)
    prob = meas.TransportProblem(
        mu=meas.GridMeasure(grid, mu), nu=meas.GridMeasure(grid, nu),
        div=meas.DivergenceSpec(lam=c["lam"]), eps=eps)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = eng.make_decomposition(prob.mu, c["s"])
    cell = eng.CellSolverConfig(max_iters=c.get("cell_max_iters", 10_000))
    cfg = eng.EngineConfig(delta=c["delta"], max_iters=c["max_iters"], cell=cell,
                           cell_delta_factor=c.get("cell_delta_factor", 0.25))
    state = eng.warm_start_plan(prob, dec, delta=1e-3) if c["warm"] else None
    st, rep = eng.domdec_solve(prob, dec, eng.StrategyConfig(kind=c["strategy"]), cfg, state=state)
    out = dict(mu=mu, nu=nu, dx=dx, origin=np.array(origin), lam=c["lam"], eps=eps, s=c["s"],
               cell_max_iters=c.get("cell_max_iters", 10_000),
               strategy=c["strategy"], delta=c["delta"], max_iters=c["max_iters"],
               warm=c["warm"], cell_delta_factor=c.get("cell_delta_factor", 0.25))
    return _outputs(st, rep, out)


def _outputs(st, rep, out):
    """Reference state + report -> fixture arrays (shared by every case)."""
    boxes, vals, offs = [], [], [0]
    for m in st.nu_i:
        b = [x for ax in m.box for x in ax]
        if len(b) == 2:
            b = [0, 1 if m.values.size else 0] + b
        boxes.append(b)
        vals.append(m.values.ravel())
        offs.append(offs[-1] + m.values.size)
    out["nu_i_box"] = np.array(boxes, dtype=np.int64)
    out["nu_i_off"] = np.array(offs, dtype=np.int64)
    out["nu_i_val"] = np.concatenate(vals) if vals else np.zeros(0)
    xo = [0]
    for x in st.x_marg:
        xo.append(xo[-1] + x.size)
    out["x_marg_off"] = np.array(xo, dtype=np.int64)
    out["x_marg_val"] = np.concatenate(st.x_marg)
    out["transport"] = st.transport
    out["kl"] = st.kl
    out["truncated_mass"] = st.truncated_mass
    sb = rep.final_score
    out["score"] = np.array([sb["transport"], sb["entropy"], sb["d1"], sb["d2"], sb["total"]])
    out["rel_pd_gap"] = rep.rel_pd_gap
    out["converged"] = rep.converged
    out["iterations"] = rep.iterations
    out["trace_total"] = np.array([r.total for r in rep.trace])
    out["trace_gap"] = np.array([r.gap for r in rep.trace])
    out["trace_action"] = np.array([r.action for r in rep.trace])
    out["trace_xerr"] = np.array([r.x_err for r in rep.trace])
    out["trace_yerr"] = np.array([r.y_err for r in rep.trace])
    keys = sorted(st.duals)
    out["dual_keys"] = np.array([f"{l}:{j}" for l, j in keys])
    ao, bo, abox = [0], [0], []
    av, bv = [], []
    for k in keys:
        d = st.duals[k]
        av.append(d.alpha.ravel())
        bv.append(d.beta.ravel())
        ao.append(ao[-1] + d.alpha.size)
        bo.append(bo[-1] + d.beta.size)
        b = [x for ax in d.beta_box for x in ax]
        if len(b) == 2:
            b = [0, 1] + b
        abox.append(b)
    out["dual_alpha"] = np.concatenate(av)
    out["dual_alpha_off"] = np.array(ao)
    out["dual_beta"] = np.concatenate(bv)
    out["dual_beta_off"] = np.array(bo)
    out["dual_beta_box"] = np.array(abox, dtype=np.int64)
    out["diag_safe_fallbacks"] = rep.diagnostics["safe_fallbacks"]
    return out


def run_ms256(eng, meas):
    """configs[1] (ms_256) finest stage from the GPU's SPEC handoff.

    tests/golden/ms256_switch_duals.npz (scripts/dump_ms256_switch.py, GPU) holds
    the duals the device's global Sinkhorn layers 32^2..128^2 prolong to 256^2.
    The reference's own warm_start_plan (its global Sinkhorn started from those
    duals instead of zeros, same delta/4 tolerance, then its plan cut) and
    domdec_solve (staggered, delta 2e-5) produce the fixture.
    """
    d = {k: v for k, v in np.load(OUT / "ms256_switch_duals.npz").items()}
    mu, nu = d["mu"], d["nu"]
    dx = float(d["dx"])
    origin = tuple(float(o) for o in d["origin"])
    grid = meas.Grid(mu.shape, dx=dx, origin=origin)
    prob = meas.TransportProblem(mu=meas.GridMeasure(grid, mu), nu=meas.GridMeasure(grid, nu),
                                 div=meas.DivergenceSpec(lam=float(d["lam"])), eps=float(d["eps"]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = eng.make_decomposition(prob.mu, int(d["s"]))
    orig = eng.sinkhorn_solve

    def started(kernel, mu_, nu_, m, a0, b0, div, config):
        return orig(kernel, mu_, nu_, m, d["alpha0"].copy(), d["beta0"].copy(), div, config)

    eng.sinkhorn_solve = started
    try:
        ws = eng.warm_start_plan(prob, dec, delta=float(d["warm_delta"]),
                                 max_iters=int(d["warm_max_iters"]))
    finally:
        eng.sinkhorn_solve = orig
    st, rep = eng.domdec_solve(prob, dec, eng.StrategyConfig(kind="staggered"),
                               eng.EngineConfig(delta=2e-5), state=ws)
    out = dict(mu=mu, nu=nu, dx=dx, origin=np.array(origin), lam=float(d["lam"]), eps=prob.eps,
               s=int(d["s"]), cell_max_iters=10_000, strategy="staggered", delta=2e-5,
               max_iters=2000, warm=True, cell_delta_factor=0.25)
    return _outputs(st, rep, out)


def kernel_fixtures(sk, meas):
    rng = np.random.default_rng(11)
    # Newton Y-step on a grid including the degenerate extremes
    m = np.array([0.0, 1e-12, 1e-6, 1.0, 1e6, 0.0, 3.0, 0.5] * 4)
    z = np.array([-700.0, 0.0, 50.0, -np.inf, 0.0, -np.inf, 2.0, -3.0] * 4)
    z = z + rng.normal(0, 1e-3, z.size) * np.isfinite(z)
    eps = np.repeat([1e-3, 1.0, 0.3, 5.0], 8)
    lam = np.repeat([1.0, 1.0, 100.0, 0.01], 8)
    beta = np.empty_like(z)
    for k in range(z.size):
        b, _ = sk.y_halfstep_newton(z[k:k + 1], m[k:k + 1], float(eps[k]),
                                    meas.DivergenceSpec(lam=float(lam[k])), np.zeros(1))
        beta[k] = b[0]
    np.savez(OUT / "newton_grid.npz", m=m, z=z, eps=eps, lam=lam, beta=beta)
    # separable sweeps on a rectangular grid pair
    n0, n1 = 12, 20
    dx = 1.0 / 20
    xa = [0.03 + dx * np.arange(n0), 0.01 + dx * np.arange(n1)]
    ya = [0.02 + dx * np.arange(n0), 0.04 + dx * np.arange(n1)]
    ker = sk.SeparableKernel(xa, ya, 2 * dx * dx)
    v = rng.normal(0, 3, (n0, n1))
    v[0, 0] = -np.inf
    np.savez(OUT / "separable_sweep.npz", xa0=xa[0], xa1=xa[1], ya0=ya[0], ya1=ya[1],
             eps=2 * dx * dx, v=v, lse_x=ker.lse_x(v), lse_y=ker.lse_y(v))
    # one global Sinkhorn solve (zero background) on a 24x24 mixture
    n = 24
    dx = 1.0 / n
    org = (0.5 * dx, 0.5 * dx)
    mu = _mixture((n, n), dx, org, rng, 3)
    nu = _mixture((n, n), dx, org, rng, 3) * 1.2
    axes = [org[0] + dx * np.arange(n)] * 2
    ker = sk.SeparableKernel(axes, axes, 2 * dx * dx)
    res = sk.sinkhorn_solve(ker, mu, nu, None, np.zeros((n, n)), np.zeros((n, n)),
                            meas.DivergenceSpec(lam=0.7), sk.SolverConfig(delta=1e-7))
    np.savez(OUT / "global_sinkhorn.npz", mu=mu, nu=nu, dx=dx, origin=np.array(org), lam=0.7,
             eps=2 * dx * dx, delta=1e-7, alpha=res.alpha, beta=res.beta, gap=res.gap,
             iterations=res.iterations, x_marginal=res.x_marginal)


def main():
    eng, meas, sk = _import_ref()
    OUT.mkdir(parents=True, exist_ok=True)
    only = set(sys.argv[1:])
    if not only or only & {"kernels"}:
        kernel_fixtures(sk, meas)
    if only & {c["name"] for c in VOL_CASES} or "vol3" in only:
        import time as _t
        lift_3d_guards(meas, sk)
        for c in VOL_CASES:
            if "vol3" not in only and c["name"] not in only:
                continue
            t0 = _t.perf_counter()
            out = run_vol_case(eng, meas, c)
            out["ref_seconds"] = _t.perf_counter() - t0
            np.savez_compressed(OUT / f"{c['name']}.npz", **out)
            print(c["name"], "iters", out["iterations"], "total", out["score"][-1], "seconds",
                  round(out["ref_seconds"], 1), "actions", list(out["trace_action"]), flush=True)
        return
    if "ms256" in only:
        import time as _t
        t0 = _t.perf_counter()
        out = run_ms256(eng, meas)
        out["ref_seconds"] = _t.perf_counter() - t0
        np.savez_compressed(OUT / "ms256_final.npz", **out)
        print("ms256 iters", out["iterations"], "total", out["score"][-1], "seconds",
              out["ref_seconds"])
    for c in CASES + BASELINE_CASES:
        if not only and c in BASELINE_CASES:
            continue   # slow: generate explicitly by name
        if only and c["name"] not in only:
            continue
        import time as _t
        t0 = _t.perf_counter()
        out = run_case(eng, meas, c)
        out["ref_seconds"] = _t.perf_counter() - t0
        np.savez_compressed(OUT / f"{c['name']}.npz", **out)
        print(c["name"], "iters", out["iterations"], "total", out["score"][-1],
              "size", os.path.getsize(OUT / f"{c['name']}.npz"))


if __name__ == "__main__":
    main()
