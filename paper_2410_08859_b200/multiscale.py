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
* the coarsest level starts from ``warm_start_plan`` (global device Sinkhorn
  plus plan cut); every later level starts from ``refine_plan`` — each coarse
  basic-cell Y-marginal mass split over its 2^d child cells by fine mu mass,
  duals prolonged bilinearly
  (``dd_prolong``; piecewise-constant potentials would put an
  O(|grad beta| h / eps) error into the warm start); child marginals are the
  parent's split by fine mu (across children) and fine nu (across nodes);
* each eps stage is one ``domdec_solve`` warm-started from the previous
  stage's plan, cell duals and certificate duals.

All numerical work runs in libdomdec_b200; host code here only builds the
pyramid (input preparation) and sequences the stages.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .decomposition import make_decomposition
from .engine import (EngineConfig, PlanState, StitchedGapEvaluator, StrategyConfig, _member_boxes,
                     _tables, domdec_solve, warm_start_plan)
from .grids import Grid, GridMeasure, TransportProblem
from .sinkhorn import DeviceProblem

__all__ = ["Level", "build_pyramid", "stage_pyramid", "eps_schedule", "refine_plan",
           "MultiscaleReport", "multiscale_solve"]


@dataclass
class Level:
    grid: Grid
    mu: np.ndarray
    nu: np.ndarray
    dp: object = None      # DeviceProblem once staged on the device


def stage_pyramid(levels: list, div, eps: float) -> list:
    """Copy every level's measures to the device once (DeviceProblem per level)."""
    for lv in levels:
        lv.dp = DeviceProblem(TransportProblem(GridMeasure(lv.grid, lv.mu),
                                               GridMeasure(lv.grid, lv.nu), div, eps))
    return levels


def coarsen(mass: np.ndarray) -> np.ndarray:
    m = np.asarray(mass, dtype=np.float64)
    if m.ndim == 1:
        return m.reshape(-1, 2).sum(axis=1)
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


def refine_plan(coarse: PlanState, fine_problem: TransportProblem, fine_dec,
                coarse_duals=None, trunc_threshold: float = 1e-15, dp=None,
                shape: str = "split") -> PlanState:
    """Fine-level state from a solved coarse state (SPEC multiscale.refine_plan).

    Each child basic cell keeps its share f_j = mu(X_j)/mu(X_i) of the parent's
    Y-marginal mass.  ``shape="split"`` (default) splits the parent marginal
    over fine Y nodes by fine nu mass (``dd_refine``), which keeps the summed
    children consistent with the coarse plan's Y-marginal.  ``shape="dual"``
    shapes each child by the plan of the prolonged duals restricted to its
    block (``dd_refine_dual``): tighter boxes, but the children no longer sum
    to the coarse marginal and the first fine sweeps pay for it (measured: many
    more cell iterations), so it is opt-in.  Both truncate at the threshold and
    install product-plan fragments; duals are prolonged bilinearly.
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
    if shape == "dual" and fa is not None and st.block[0] <= 8 and st.bs <= 64:
        tcap = 4 * cmax
        tmp = torch.empty(fb.n_cells * tcap, dtype=torch.float64, device=dp.device)
        max_fe = 2 * int(max(boxes[:, 1].max(initial=1), boxes[:, 3].max(initial=1)))
        _lib.check(L.dd_refine_dual(dp.geom, st.state_struct(), parent_d.data_ptr(),
                                    coarse.ybox.data_ptr(), coarse.yval.data_ptr(), coarse.cap,
                                    coarse.basic_mass.data_ptr(), fa.data_ptr(), fbeta.data_ptr(),
                                    float(trunc_threshold), trunc_out.data_ptr(), tmp.data_ptr(),
                                    tcap, max_fe, _lib.stream_handle()))
        torch.cuda.synchronize()
        del tmp
    else:
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


def multiscale_solve(problem: TransportProblem, cell_size: int, n_coarsest: int, eps_start: float,
                     eps_final: float | None = None, strategy: StrategyConfig = StrategyConfig(),
                     config: EngineConfig = EngineConfig(), warm_delta: float = 1e-3,
                     warm_max_iters: int = 20_000, progress=None, levels: list | None = None,
                     final_stages: int = 1):
    """Solve ``problem`` coarse-to-fine; returns (fine PlanState, MultiscaleReport).

    ``levels`` may carry a pre-built (and device-staged) pyramid from
    :func:`build_pyramid` / :func:`stage_pyramid`.
    """
    t_all = time.perf_counter()
    eps_final = problem.eps if eps_final is None else eps_final
    if levels is None:
        levels = build_pyramid(problem.mu, problem.nu, n_coarsest)
    sched = eps_schedule(levels, eps_start, eps_final, final_stages)
    rep = MultiscaleReport(converged=True)
    state = None
    duals = None
    timings = {"warm": 0.0, "refine": 0.0, "domdec": 0.0}
    for li, lv in enumerate(levels):
        eps_list = sched[li] or [None]
        first_eps = eps_list[0] if eps_list[0] is not None else (
            next((e for row in sched[li:] for e in row), eps_final))
        prob = _with_eps(lv, problem.div, first_eps)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            dec = make_decomposition(prob.mu, cell_size)
        t0 = time.perf_counter()
        if lv.dp is not None:
            lv.dp.problem = prob
            lv.dp.geom.eps = float(prob.eps)
        if state is None:
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
    timings["total"] = time.perf_counter() - t_all
    rep.timings = timings
    return state, rep
