"""CPU baseline sample: oracle cell solves of recorded ms_1024 subproblems.

TEST / BASELINE INFRASTRUCTURE ONLY (imported by bench.py's cpu_baseline leg
and reference arm, never by the product package).  The sample file
(tests/golden/ms1024_cells.npz, written by scripts/make_cell_sample.py on a
GPU box) holds complete composite-cell subproblems from the first staggered
batch of the 1024^2 stage of BASELINE configs[2].  Each is solved by the
oracle's restatement of the reference cell solver (cells.py:235-393 via
``ref_cell.solve_batch``, one cell per call, as the reference does for a
chunk of one), process-parallel over the host cores (cells of a batch are
independent, SPEC concurrency model).
"""

from __future__ import annotations

import os
import time
from types import SimpleNamespace

import numpy as np

from .ref_cell import CellProb, solve_batch
from .ref_sweep import CellCfg

SAMPLE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                      "golden", "ms1024_cells.npz")


def load_sample(path: str = SAMPLE):
    with np.load(path, allow_pickle=False) as f:
        d = {k: f[k] for k in f.files}
    probs = []
    for q in range(int(d["n_cells"])):
        p = lambda k: d[f"c{q}_{k}"]  # noqa: E731
        m = p("m_win")
        probs.append(CellProb(
            j=int(p("j")), xbox=tuple(int(x) for x in p("xbox")), mu_win=p("mu_win"),
            ybox=tuple(int(x) for x in p("ybox")), nu_win=p("nu_win"),
            m_win=m if m.size else None, alpha0=p("alpha0"), beta0=p("beta0"),
            members=[int(x) for x in p("members")], rows=list(p("rows")), masses=p("masses"),
            xc=[p("xc0"), p("xc1")], yc=[p("yc0"), p("yc1")], n_clamped=0, cell_sum=None))
    iters = np.array([int(d[f"c{q}_gpu_iters"]) for q in range(int(d["n_cells"]))])
    ctx = SimpleNamespace(eps=float(d["eps"]), lam=float(d["lam"]), nu_total=float(d["nu_total"]))
    return probs, iters, ctx, d


def _solve_one(args):
    p, ctx, delta, cap = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    t0 = time.perf_counter()
    s = solve_batch([p], ctx, CellCfg(delta=delta, max_iters=cap))[0]
    return s.iterations, time.perf_counter() - t0


def run_sample(cap: int, workers: int | None = None, path: str = SAMPLE):
    """Solve every sample cell with the cell iteration cap ``cap``; returns
    (wall seconds, iterations per cell, cores used, sample dict)."""
    from concurrent.futures import ProcessPoolExecutor

    probs, _, ctx, d = load_sample(path)
    workers = workers or os.cpu_count() or 1
    workers = max(1, min(workers, len(probs)))
    args = [(p, ctx, float(d["delta"]), cap) for p in probs]
    t0 = time.perf_counter()
    if workers == 1:
        res = [_solve_one(a) for a in args]
    else:
        with ProcessPoolExecutor(max_workers=workers) as ex:
            res = list(ex.map(_solve_one, args))
    wall = time.perf_counter() - t0
    return wall, np.array([r[0] for r in res]), workers, d, probs


def sample_flops(probs, iters, nw0: int, nw1: int) -> float:
    """Algorithmic cell-sweep FLOPs (engine.cell_lse_flops) of the sample's iterations."""
    tot = 0.0
    for p, it in zip(probs, iters):
        ny0, ny1 = p.ybox[1], p.ybox[3]
        nx = nw0 * nw1
        tot += it * 2.0 * (ny0 * nw1 * ny1 + nx * ny0 + nw0 * ny1 * nw1 + ny0 * ny1 * nw0)
    return tot
