"""Run the device engine on a golden fixture's inputs (GPU tests only)."""

from __future__ import annotations

import warnings

import numpy as np


def problem_from_golden(g):
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem

    mu, nu = g["mu"], g["nu"]
    dims = mu.shape
    grid = Grid(dims, float(g["dx"]), tuple(float(o) for o in g["origin"]))
    return TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu),
                            DivergenceSpec(float(g["lam"])), float(g["eps"]))


def run_device(g):
    from paper_2410_08859_b200.decomposition import make_decomposition
    from paper_2410_08859_b200.engine import (CellSolverConfig, EngineConfig, StrategyConfig,
                                              domdec_solve, warm_start_plan)
    from _golden import cell_cap

    prob = problem_from_golden(g)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(prob.mu, int(g["s"]))
    cfg = EngineConfig(delta=float(g["delta"]), max_iters=int(g["max_iters"]),
                       cell=CellSolverConfig(max_iters=cell_cap(g)),
                       cell_delta_factor=float(g["cell_delta_factor"]) if "cell_delta_factor" in g
                       else 0.25)
    state = warm_start_plan(prob, dec, delta=1e-3) if bool(g["warm"]) else None
    st, rep = domdec_solve(prob, dec, StrategyConfig(kind=str(g["strategy"])), cfg, state=state)
    return prob, dec, st, rep


def box4(box):
    b = [c for ax in box for c in ax]
    if len(b) == 2:
        b = [0, 1 if b[1] else 0] + b
    if b[1] == 0 or b[3] == 0:
        return (0, 0, 0, 0)
    return tuple(int(x) for x in b)
