"""Coarse-to-fine driver: grid pyramid, epsilon ladder, plan refinement, domdec per stage.

The reference package's SPEC names this layer (``multiscale``: build_pyramid,
eps_schedule, refine_plan, multiscale_solve) but its source tree does not
implement it, so this module follows the SPEC text and the BASELINE.json
configurations (eps annealed from ``eps_start`` to ``eps_final`` by halving,
grids refined x2 per level from ``n_coarsest`` up to the problem grid):

* ``build_pyramid`` sums 2^d children per coarse node (mass preserving);
* ``eps_schedule`` halves eps from start to final and runs each value on the
  coarsest level whose spacing satisfies h^2 <= eps (the last value always
  on the finest level);
* (spec) the coarsest global Sinkhorn starts from the mass-balanced constant
  duals (``sinkhorn.mass_balanced_start``);
* the coarsest level starts from ``warm_start_plan`` (global device Sinkhorn
  plus plan cut); every later level starts from ``refine_plan`` — each coarse
  basic-cell Y-marginal mass split over its 2^d child cells by fine mu mass,
  duals prolonged bilinearly
  (``dd_prolong``; piecewise-constant potentials would put an
  O(|grad beta| h / eps) error into the warm start); child marginals are the
  parent's split by fine mu (across children) and fine nu (across nodes);
* each eps stage is one ``domdec_solve`` warm-started from the previous
  stage's plan, cell duals and certificate duals.

``protocol="spec"`` (the default) is SPEC ``multiscale_solve`` / paper §4.3.1
(PAPER.md:1291-1294): per-layer eps ladder 2dx^2 -> dx^2/2 (seams coincide),
global unbalanced Sinkhorn at tolerance delta/4 on every layer below the
switch layer (l_switch = 8 for N >= 512, else log2 N - 1; layer l holds
2^(l+1) nodes per axis, so for N < 512 only the finest layer runs domdec),
a global Sinkhorn presolve at the switch layer (warm-started from the
prolonged duals, same delta/4) whose plan is cut along the basic cells
(``warm_start_plan``), and domdec (staggered) from there on.  ``protocol="ladder"`` keeps the round-1 schedule
(one loose warm start at the coarsest level, domdec at every level).

All numerical work runs in libdomdec_b200; host code here only builds the
pyramid (input preparation) and sequences the stages.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .decomposition import make_decomposition
from .engine import (EngineConfig, PlanState, StitchedGapEvaluator, StrategyConfig, _member_boxes,
                     _tables, domdec_solve, warm_start_plan)
from .grids import Grid, GridMeasure, TransportProblem
from .report import SolveReport
from .sinkhorn import DeviceProblem, SolverConfig, mass_balanced_start, sinkhorn_solve

__all__ = ["Level", "build_pyramid", "stage_pyramid", "eps_schedule", "spec_eps_schedule",
           "switch_layer", "layer_index", "refine_plan", "prolong_duals", "MultiscaleReport",
           "multiscale_solve"]


@dataclass
class Level:
    grid: Grid
    mu: np.ndarray
    nu: np.ndarray
    dp: object = None      # DeviceProblem once staged on the device
    decs: dict = field(default_factory=dict)   # cell size -> Decomposition (staged pyramids)


def stage_pyramid(levels: list, div, eps: float) -> list:
    """Copy every level's measures to the device once (DeviceProblem per level); the
    partition tables built by the first solve on a level are kept with it."""
    for lv in levels:
        prob = TransportProblem(GridMeasure(lv.grid, lv.mu), GridMeasure(lv.grid, lv.nu), div, eps)
        if lv.grid.ndim == 3:
            from .volume import VolumeProblem
            lv.dp = VolumeProblem(prob)
        else:
            lv.dp = DeviceProblem(prob)
    return levels


def coarsen(mass: np.ndarray) -> np.ndarray:
    m = np.asarray(mass, dtype=np.float64)
    if m.ndim == 1:
        return m.reshape(-1, 2).sum(axis=1)
    if m.ndim == 3:
        n0, n1, n2 = m.shape
        return m.reshape(n0 // 2, 2, n1 // 2, 2, n2 // 2, 2).sum(axis=(1, 3, 5))
    n0, n1 = m.shape
    return m.reshape(n0 // 2, 2, n1 // 2, 2).sum(axis=(1, 3))


def build_pyramid(mu: GridMeasure, nu: GridMeasure, n_min: int) -> list:
    """Levels coarsest -> finest; coarse node = sum of its 2^d children, at their centre."""
    g = mu.grid
    if any(n & (n - 1) for n in g.dims):
        raise ValueError("multiscale needs power-of-two grid dims")
    levels = [Level(g, np.asarray(mu.mass, dtype=np.float64), np.asarray(nu.mass, dtype=np.float64))]
    while min(levels[0].grid.dims) > n_min:
        f = levels[0]
        dims = tuple(n // 2 for n in f.grid.dims)
        grid = Grid(dims, 2.0 * f.grid.dx, tuple(o + 0.5 * f.grid.dx for o in f.grid.origin))
        levels.insert(0, Level(grid, coarsen(f.mu), coarsen(f.nu)))
    return levels


def eps_schedule(levels: list, eps_start: float, eps_final: float, final_stages: int = 1) -> list:
    """Per level, the eps values it solves (halving ladder eps_start -> eps_final).

    The last ``final_stages`` ladder values always run on the finest level.
    """
    ladder = []
    e = float(eps_start)
    while e > eps_final * (1.0 + 1e-12):
        ladder.append(e)
        e *= 0.5
    ladder.append(float(eps_final))
    per = [[] for _ in levels]
    for k, e in enumerate(ladder):
        if k >= len(ladder) - max(1, final_stages):
            per[-1].append(e)
            continue
        idx = len(levels) - 1
        for li, lv in enumerate(levels):
            if lv.grid.dx ** 2 <= e * (1.0 + 1e-12):
                idx = li
                break
        per[idx].append(e)
    # keep the ladder monotone across levels
    for li in range(1, len(per)):
        if per[li - 1] and per[li]:
            per[li] = [e for e in per[li] if e <= per[li - 1][-1]]
    return per


def layer_index(n: int) -> int:
    """Paper layer number of an n-node axis: layer l holds 2^(l+1) nodes (finest = log2 N - 1)."""
    return int(round(math.log2(n))) - 1


def switch_layer(n_finest: int) -> int:
    """First domdec layer: 8 for N >= 512, else floor(log2 N) - 1."""
    return 8 if n_finest >= 512 else int(math.floor(math.log2(n_finest))) - 1


def spec_eps_schedule(levels: list, eps_start: float, eps_final: float) -> list:
    """Per level, its eps ladder (SPEC eps_schedule): 2dx^2, dx^2, dx^2/2 on every
    layer, so a layer's last value is the next layer's first; clipped to
    [eps_final, eps_start].  A layer whose whole ladder lies above eps_start
    runs eps_start; the finest layer ends on eps_final."""
    per = []
    top = float(eps_start)
    for li, lv in enumerate(levels):
        d2 = lv.grid.dx ** 2
        lad = [2.0 * d2, d2, 0.5 * d2]
        if li == len(levels) - 1:
            lad.append(0.25 * d2)
        row = [e for e in lad if eps_final * (1 - 1e-12) <= e <= top * (1 + 1e-12)]
        if not row:
            row = [min(top, max(lad[0], eps_final))]
        if li == len(levels) - 1 and abs(row[-1] - eps_final) > 1e-12 * eps_final:
            row = [e for e in row if e > eps_final] + [float(eps_final)]
        per.append(row)
        top = row[-1]
    return per


def prolong_duals(duals, coarse_geom, fine_geom):
    """Bilinear prolongation of an (alpha, beta) pair to the next finer layer (dd_prolong)."""
    import torch

    ca, cb = duals
    fa = torch.empty(fine_geom.nx0 * fine_geom.nx1, dtype=torch.float64, device=ca.device)
    fb = torch.empty(fine_geom.ny0 * fine_geom.ny1, dtype=torch.float64, device=ca.device)
    L = _lib.lib()
    _lib.check(L.dd_prolong(fine_geom.nx0, fine_geom.nx1, coarse_geom.nx0, coarse_geom.nx1,
                            ca.data_ptr(), fa.data_ptr(), _lib.stream_handle()))
    _lib.check(L.dd_prolong(fine_geom.ny0, fine_geom.ny1, coarse_geom.ny0, coarse_geom.ny1,
                            cb.data_ptr(), fb.data_ptr(), _lib.stream_handle()))
    return fa, fb


def refine_plan(coarse: PlanState, fine_problem: TransportProblem, fine_dec,
                coarse_duals=None, trunc_threshold: float = 1e-15, dp=None) -> PlanState:
    """Fine-level state from a solved coarse state (SPEC multiscale.refine_plan).

    Each child basic cell keeps its share f_j = mu(X_j)/mu(X_i) of the parent's
    Y-marginal mass, split over fine Y nodes by fine nu mass (``dd_refine``), so
    the summed children stay consistent with the coarse plan's Y-marginal;
    children are truncated at the threshold and carry product-plan fragments;
    duals are prolonged bilinearly.
    """
    import torch

    cb = coarse.basic
    fb = fine_dec.basic
    if fb.s != cb.s:
        raise ValueError("refinement keeps the basic cell size in nodes")
    dp = dp if dp is not None else DeviceProblem(fine_problem)
    dp.problem = fine_problem
    dp.geom.eps = float(fine_problem.eps)
    boxes = coarse.ybox.view(-1, 4).cpu().numpy()
    cmax = int((boxes[:, 1].astype(np.int64) * boxes[:, 3]).max(initial=1))
    st = PlanState(fine_problem, fb, dp, cap=4 * cmax)
    pos = fb.positions
    lat = cb.lattice_to_cell
    parent = lat[tuple((pos // 2).T)] if pos.shape[1] > 1 else lat[pos[:, 0] // 2]
    if np.any(parent < 0):
        raise ValueError("fine basic cell without a coarse parent")
    parent_d = torch.from_numpy(parent.astype(np.int32)).to(dp.device)
    trunc_out = torch.zeros(fb.n_cells, dtype=torch.float64, device=dp.device)
    g = dp.geom
    L = _lib.lib()
    fa = fbeta = None
    if coarse_duals is not None:
        ca, cbeta = coarse_duals
        cg = coarse.dp.geom
        fa = dp.empty_x()
        fbeta = dp.empty_y()
        _lib.check(L.dd_prolong(g.nx0, g.nx1, cg.nx0, cg.nx1, ca.data_ptr(), fa.data_ptr(),
                                _lib.stream_handle()))
        _lib.check(L.dd_prolong(g.ny0, g.ny1, cg.ny0, cg.ny1, cbeta.data_ptr(), fbeta.data_ptr(),
                                _lib.stream_handle()))
    _lib.check(L.dd_refine(dp.geom, st.state_struct(), parent_d.data_ptr(),
                           coarse.ybox.data_ptr(), coarse.yval.data_ptr(), coarse.cap,
                           coarse.basic_mass.data_ptr(), coarse.dp.nu.data_ptr(),
                           coarse.dp.geom.ny1, float(trunc_threshold), trunc_out.data_ptr(),
                           _lib.stream_handle()))
    st.sync_boxes()
    st.truncated_mass = coarse.truncated_mass + float(trunc_out.sum().item())
    if fa is not None:
        for part in fine_dec.composites:
            pt = _tables(part)
            yb = _member_boxes(st, pt, np.arange(pt.ncomp))
            store = st.store(pt)
            store.ensure(int((yb[:, 1].astype(np.int64) * yb[:, 3]).max(initial=1)))
            xb_d = torch.from_numpy(pt.xbox.ravel().copy()).to(dp.device)
            yb_d = torch.from_numpy(yb.ravel().copy()).to(dp.device)
            _lib.check(L.dd_seed_duals(dp.geom, st.state_struct(store), pt.ncomp, pt.nw0, pt.nw1,
                                       xb_d.data_ptr(), yb_d.data_ptr(), fa.data_ptr(),
                                       fbeta.data_ptr(), _lib.stream_handle()))
        st.global_duals = (fa, fbeta)
    return st


@dataclass
class MultiscaleReport:
    converged: bool
    stages: list = field(default_factory=list)   # (level n, eps, SolveReport)
    timings: dict = field(default_factory=dict)
    final_score: dict = field(default_factory=dict)
    rel_pd_gap: float = float("nan")
    total_iterations: int = 0


def _with_eps(lv: Level, lam_div, eps: float) -> TransportProblem:
    return TransportProblem(GridMeasure(lv.grid, lv.mu), GridMeasure(lv.grid, lv.nu), lam_div, eps)


def _global_report(res, eps: float, t: float, delta: float) -> SolveReport:
    return SolveReport(converged=bool(res.converged), iterations=int(res.iterations),
                       final_score={}, rel_pd_gap=float("nan"), x_err=0.0, y_err=0.0,
                       timings={"total": t, "solve": t, "score": 0.0, "commit": 0.0},
                       diagnostics={"solver": "sinkhorn", "gap": float(res.gap), "delta": delta,
                                    "cell_iterations": 0, "cell_flops": 0.0,
                                    "nonconverged_cells": 0, "safe_fallbacks": 0})


def multiscale_solve(problem: TransportProblem, cell_size: int, n_coarsest: int, eps_start: float,
                     eps_final: float | None = None, strategy: StrategyConfig = StrategyConfig(),
                     config: EngineConfig = EngineConfig(), warm_delta: float = 1e-3,
                     warm_max_iters: int = 20_000, progress=None, levels: list | None = None,
                     final_stages: int = 1, protocol: str = "spec", switch: int | None = None,
                     global_delta: float | None = None, global_max_iters: int = 100_000,
                     switch_delta: float | None = None, switch_iters: int = 20_000):
    """Solve ``problem`` coarse-to-fine; returns (fine PlanState, MultiscaleReport).

    ``levels`` may carry a pre-built (and device-staged) pyramid from
    :func:`build_pyramid` / :func:`stage_pyramid`.  ``protocol="spec"``:
    global Sinkhorn at ``global_delta`` (default delta/4) below layer
    ``switch`` (default :func:`switch_layer`), then domdec; at the switch layer
    the plan comes from ``warm_start_plan`` warm-started with the prolonged
    duals: global Sinkhorn to ``switch_delta`` (default: the coarse-layer
    tolerance delta/4, so the first marginal handed to domdec is as close to
    optimal as on the layers below), at most ``switch_iters``
    iterations, then the plan cut along the basic cells.  ``protocol="ladder"``: the round-1 schedule
    (``warm_delta`` warm start at the coarsest level, domdec at every level).
    """
    if protocol not in ("spec", "ladder"):
        raise ValueError(f"unknown multiscale protocol {protocol!r}")
    if problem.mu.grid.ndim == 3:
        if protocol != "spec":
            raise ValueError("the three-axis path runs the SPEC protocol only")
        from .volume import multiscale_solve3
        return multiscale_solve3(problem, cell_size, n_coarsest, eps_start, eps_final, strategy,
                                 config, progress, levels, switch, global_delta,
                                 global_max_iters, switch_iters)
    t_all = time.perf_counter()
    eps_final = problem.eps if eps_final is None else eps_final
    if levels is None:
        levels = build_pyramid(problem.mu, problem.nu, n_coarsest)
    n_fine = max(levels[-1].grid.dims)
    lsw = (switch_layer(n_fine) if switch is None else int(switch)) if protocol == "spec" else -1
    sched = (spec_eps_schedule(levels, eps_start, eps_final) if protocol == "spec"
             else eps_schedule(levels, eps_start, eps_final, final_stages))
    gdelta = config.delta / 4.0 if global_delta is None else float(global_delta)
    rep = MultiscaleReport(converged=True)
    state = None
    duals = None
    duals_geom = None
    timings = {"global": 0.0, "warm": 0.0, "refine": 0.0, "domdec": 0.0}
    for li, lv in enumerate(levels):
        eps_list = sched[li] or [None]
        first_eps = eps_list[0] if eps_list[0] is not None else (
            next((e for row in sched[li:] for e in row), eps_final))
        prob = _with_eps(lv, problem.div, first_eps)
        if lv.dp is not None:
            lv.dp.problem = prob
            lv.dp.geom.eps = float(prob.eps)
        if protocol == "spec" and layer_index(max(lv.grid.dims)) < lsw and li < len(levels) - 1:
            # coarse layer: global unbalanced Sinkhorn at delta/4
            dp = lv.dp if lv.dp is not None else DeviceProblem(prob)
            if duals is not None:
                a0, b0 = prolong_duals(duals, duals_geom, dp.geom)
            else:
                dp.geom.eps = float(eps_list[0])
                a0, b0 = mass_balanced_start(dp)
            for eps in eps_list:
                dp.problem = _with_eps(lv, problem.div, eps)
                dp.geom.eps = float(eps)
                t0 = time.perf_counter()
                res = sinkhorn_solve(dp, a0, b0, SolverConfig(delta=gdelta,
                                                              max_iters=global_max_iters))
                t = time.perf_counter() - t0
                timings["global"] += t
                a0, b0 = res.alpha, res.beta
                r = _global_report(res, eps, t, gdelta)
                rep.stages.append((lv.grid.dims[0], eps, r))
                rep.converged = rep.converged and r.converged
                if progress is not None:
                    progress(lv.grid.dims[0], eps, r)
            duals, duals_geom = (a0, b0), dp.geom
            continue
        # a staged pyramid (stage_pyramid) keeps its partition tables with the
        # device copies of the measures; host pyramids rebuild them every solve
        dec = lv.decs.get(cell_size) if lv.dp is not None else None
        if dec is None:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                dec = make_decomposition(prob.mu, cell_size)
            if lv.dp is not None:
                lv.decs[cell_size] = dec
        t0 = time.perf_counter()
        if state is None:
            if protocol == "spec":
                a0 = b0 = None
                if duals is not None:
                    dp = lv.dp if lv.dp is not None else DeviceProblem(prob)
                    a0, b0 = prolong_duals(duals, duals_geom, dp.geom)
                state = warm_start_plan(prob, dec,
                                        delta=gdelta if switch_delta is None else switch_delta,
                                        max_iters=switch_iters,
                                        dp=lv.dp, alpha0=a0, beta0=b0)
            else:
                state = warm_start_plan(prob, dec, delta=warm_delta, max_iters=warm_max_iters,
                                        dp=lv.dp)
            timings["warm"] += time.perf_counter() - t0
        else:
            state = refine_plan(state, prob, dec, duals, config.cell.trunc_threshold, dp=lv.dp)
            timings["refine"] += time.perf_counter() - t0
        for eps in eps_list:
            if eps is None:
                continue
            prob = _with_eps(lv, problem.div, eps)
            state.problem = prob
            state.dp.problem = prob
            state.dp.geom.eps = float(eps)
            ev = StitchedGapEvaluator(prob, dp=state.dp)
            t0 = time.perf_counter()
            state, r = domdec_solve(prob, dec, strategy, config, state=state, evaluator=ev)
            timings["domdec"] += time.perf_counter() - t0
            best = ev._best
            if best is not None:
                state.global_duals = (best[0], best[1])
            duals = state.global_duals
            rep.stages.append((lv.grid.dims[0], eps, r))
            rep.total_iterations += r.iterations
            rep.converged = rep.converged and r.converged
            rep.final_score = r.final_score
            rep.rel_pd_gap = r.rel_pd_gap
            if progress is not None:
                progress(lv.grid.dims[0], eps, r)
        duals = state.global_duals
        duals_geom = state.dp.geom
    timings["total"] = time.perf_counter() - t_all
    rep.timings = timings
    return state, rep
