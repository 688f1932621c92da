"""Report serialization and the multiscale host logic (pyramid, eps ladder)."""

import numpy as np
import pytest

from paper_2410_08859_b200 import Grid, GridMeasure
from paper_2410_08859_b200.multiscale import build_pyramid, coarsen, eps_schedule
from paper_2410_08859_b200.report import (SolveReport, TraceRow, report_from_json,
                                          report_to_json, trace_from_csv, trace_to_csv)


def test_report_round_trips_bit_exact():
    rows = [TraceRow(k=k, label="AB"[k % 2], action="greedy", transport=0.1 / 3 * k,
                     entropy=1e-7 * k, d1=np.pi * k, d2=np.e, total=1.0 / 7 + k, gap=float("nan"),
                     x_err=1e-300, y_err=0.0, wall_time=0.123) for k in range(1, 4)]
    rep = SolveReport(converged=True, iterations=3, final_score={"total": 1.0 / 3},
                      rel_pd_gap=2e-5, x_err=0.1, y_err=0.2, trace=rows)
    back = report_from_json(report_to_json(rep))
    assert back.final_score == rep.final_score and back.trace[1].d1 == rows[1].d1
    again = trace_from_csv(trace_to_csv(rep))
    assert [r.total for r in again] == [r.total for r in rows]
    with pytest.raises(ValueError):
        SolveReport(converged=True, iterations=2, final_score={}, rel_pd_gap=0, x_err=0, y_err=0,
                    trace=[rows[1], rows[0]])


def test_pyramid_preserves_mass_and_centres():
    n = 64
    g = Grid((n, n), 1.0 / n, (0.5 / n, 0.5 / n))
    rng = np.random.default_rng(0)
    mu = GridMeasure(g, rng.uniform(0.1, 1, (n, n)))
    nu = GridMeasure(g, rng.uniform(0.1, 1, (n, n)))
    levels = build_pyramid(mu, nu, 8)
    assert [lv.grid.dims[0] for lv in levels] == [8, 16, 32, 64]
    for lv in levels:
        assert lv.mu.sum() == pytest.approx(mu.total_mass, rel=1e-12)
        assert lv.grid.origin[0] == pytest.approx(0.5 * lv.grid.dx)
    blk = mu.mass.reshape(8, 8, 8, 8).sum(axis=(1, 3))
    np.testing.assert_allclose(levels[0].mu, blk, rtol=1e-13)
    np.testing.assert_allclose(coarsen(np.ones(8)), 2 * np.ones(4))


def test_eps_schedule_halves_and_ends_on_finest():
    n = 1024
    g = Grid((n, n), 1.0 / n, (0.5 / n, 0.5 / n))
    m = GridMeasure(g, np.ones((n, n)))
    levels = build_pyramid(m, m, 64)
    h2 = g.dx ** 2
    sched = eps_schedule(levels, 256 * h2, 2 * h2)
    flat = [e for row in sched for e in row]
    assert flat[0] == pytest.approx(256 * h2) and flat[-1] == pytest.approx(2 * h2)
    assert all(b == pytest.approx(a / 2) for a, b in zip(flat, flat[1:]))
    assert sched[-1][-1] == pytest.approx(2 * h2)
    for lv, row in zip(levels, sched):
        for e in row[:-1] if lv is levels[-1] else row:
            assert lv.grid.dx ** 2 <= e * (1 + 1e-12)
