"""Host measure utilities: KL conventions, truncation, assembly, file IO, API errors."""

import numpy as np
import pytest

from paper_2410_08859_b200 import (DivergenceSpec, Grid, GridMeasure, GridMismatchError,
                                   SparseCellMarginal, TransportProblem, assemble_y_marginal,
                                   kl_divergence, truncate_and_rebox)


def test_kl_closed_forms():
    s = np.array([0.2, 0.5, 0.3])
    assert kl_divergence(s, s) == 0.0
    assert kl_divergence(np.zeros(3), s) == pytest.approx(1.0)
    assert kl_divergence(2 * s, s) == pytest.approx((2 * np.log(2) - 1) * s.sum())
    assert kl_divergence(np.array([1.0, 0.0]), np.array([0.0, 1.0])) == np.inf
    with pytest.raises(GridMismatchError):
        kl_divergence(np.ones(3), np.ones(4))


def test_kl_marginal_against_measure_counts_off_box_mass():
    g = Grid((6,), 1.0, (0.0,))
    nu = GridMeasure(g, np.linspace(0.1, 0.6, 6))
    m = SparseCellMarginal(((2, 2),), np.array([0.1, 0.2]))
    dense = np.zeros(6)
    dense[2:4] = m.values
    assert kl_divergence(m, nu) == pytest.approx(kl_divergence(dense, nu.mass), rel=1e-14)


@pytest.mark.parametrize("s,lam", [(0.3, 1.0), (2.0, 0.1), (1.0, 5.0)])
def test_fenchel_identity(s, lam):
    d = DivergenceSpec(lam)
    assert d.phi_star(d.phi_prime(s)) + d.phi(s) == pytest.approx(s * d.phi_prime(s), rel=1e-12)
    with pytest.raises(ValueError):
        DivergenceSpec(0.0)


def test_truncation_cases():
    v = np.array([[1e-16, 1e-16, 1e-16], [1e-16, 0.5, 1e-16], [1e-16, 1e-16, 1e-16]])
    m, removed = truncate_and_rebox(SparseCellMarginal(((3, 3), (4, 3)), v), 1e-15)
    assert m.box == ((4, 1), (5, 1)) and removed == pytest.approx(8e-16)
    e, removed = truncate_and_rebox(SparseCellMarginal(((0, 2),), np.array([1e-17, 1e-18])), 1e-15)
    assert e.is_empty and removed == pytest.approx(1.1e-17)
    rng = np.random.default_rng(0)
    v = rng.uniform(0, 1, (5, 7)) * (rng.uniform(size=(5, 7)) > 0.4)
    m1, r1 = truncate_and_rebox(SparseCellMarginal(((0, 5), (0, 7)), v), 0.3)
    m2, r2 = truncate_and_rebox(m1, 0.3)
    assert r2 == 0.0 and m2.box == m1.box
    assert m1.total_mass + r1 == pytest.approx(v.sum(), rel=1e-14)


def test_assemble_matches_brute_force():
    g = Grid((10, 10), 0.1, (0.0, 0.0))
    rng = np.random.default_rng(3)
    cells, dense = [], np.zeros((10, 10))
    for _ in range(16):
        o0, o1 = rng.integers(0, 6, 2)
        e0, e1 = rng.integers(1, 5, 2)
        v = rng.uniform(0, 1, (e0, e1))
        cells.append(SparseCellMarginal(((o0, e0), (o1, e1)), v))
        dense[o0:o0 + e0, o1:o1 + e1] += v
    np.testing.assert_allclose(assemble_y_marginal(cells, g).mass, dense, rtol=1e-14)
    with pytest.raises(GridMismatchError):
        assemble_y_marginal([SparseCellMarginal(((8, 4), (0, 1)), np.ones((4, 1)))], g)


@pytest.mark.parametrize("encoding", ["csv", "f64"])
def test_measure_file_round_trip(tmp_path, encoding):
    g = Grid((4, 5), 0.25, (0.125, 0.1))
    m = GridMeasure(g, np.random.default_rng(1).uniform(0, 1, (4, 5)))
    p = tmp_path / f"m.{encoding}"
    m.save(p, encoding=encoding)
    back = GridMeasure.load(p)
    assert back.grid == g and np.array_equal(back.mass, m.mass)


def test_problem_validation():
    g = Grid((4,), 0.25, (0.0,))
    with pytest.raises(ValueError):
        TransportProblem(GridMeasure(g, np.ones(4)), GridMeasure(g, np.array([1.0, 0, 1, 1])),
                         DivergenceSpec(1.0), 0.1)
    TransportProblem(GridMeasure(g, np.array([1.0, 0, 1, 1])), GridMeasure(g, np.ones(4)),
                     DivergenceSpec(1.0), 0.1)
