"""Host partition builder: the properties the reference tests for partitions.py."""

import itertools
import warnings

import numpy as np
import pytest

from paper_2410_08859_b200 import Grid, GridMeasure
from paper_2410_08859_b200.decomposition import (build_basic_partition, build_composite_partitions,
                                                 build_staggered_batches, make_decomposition)


def measure(shape, seed=0, zero_frac=0.0):
    rng = np.random.default_rng(seed)
    m = rng.uniform(0.1, 1.0, shape)
    if zero_frac:
        m[rng.uniform(size=shape) < zero_frac] = 0.0
    return GridMeasure(Grid(shape, 1.0 / shape[-1], (0.0,) * len(shape)), m)


def test_basic_counts():
    assert build_basic_partition(measure((32,)), 1).n_cells == 32
    assert build_basic_partition(measure((8, 8)), 4).n_cells == 4
    assert build_basic_partition(measure((256, 256)), 4).n_cells == 4096


def test_non_divisor_raises():
    with pytest.raises(ValueError):
        build_basic_partition(measure((10, 10)), 4)


def test_zero_block_dropped_and_zero_nodes_excluded():
    mu = measure((8, 8))
    m = mu.mass.copy()
    m[:4, :4] = 0.0
    m[5, 5] = 0.0
    basic = build_basic_partition(GridMeasure(mu.grid, m), 4)
    assert basic.n_cells == 3
    assert basic.cell_of_node[5 * 8 + 5] == -1
    assert all(m.ravel()[ids].min() > 0 for ids in basic.nodes_of_cell)


@pytest.mark.parametrize("shape,s,seed", [((16, 16), 2, 0), ((32,), 4, 1), ((12, 8), 4, 2)])
def test_disjoint_cover_of_positive_nodes(shape, s, seed):
    mu = measure(shape, seed, zero_frac=0.1)
    basic = build_basic_partition(mu, s)
    ids = np.concatenate(basic.nodes_of_cell)
    assert len(ids) == len(set(ids.tolist())) == int((mu.mass > 0).sum())


def test_composite_counts():
    basic = build_basic_partition(measure((32,)), 1)
    a, b = build_composite_partitions(basic)
    assert a.n_cells == 16 and b.n_cells == 17
    assert sorted(len(b.real_members(j)) for j in range(b.n_cells))[:2] == [1, 1]
    basic = build_basic_partition(measure((16, 16)), 4)
    a, b = build_composite_partitions(basic)
    assert a.n_cells == 4 and b.n_cells == 9


def test_each_basic_cell_in_exactly_one_composite():
    basic = build_basic_partition(measure((16, 16), zero_frac=0.05), 2)
    for part in build_composite_partitions(basic):
        seen = sorted(i for j in range(part.n_cells) for i in part.real_members(j))
        assert seen == list(range(basic.n_cells))
        shapes = {tuple(e for _, e in box) for box in part.boxes}
        assert len(shapes) == 1


def test_single_cell_degenerates_with_warning():
    with pytest.warns(UserWarning):
        a, b = build_composite_partitions(build_basic_partition(measure((8,)), 8))
    assert a.n_cells == b.n_cells == 1


@pytest.mark.parametrize("lat,seed", [((6, 6), 0), ((5, 7), 1), ((9,), 2)])
def test_staggered_batches_have_no_adjacent_cells(lat, seed):
    s = 2
    shape = tuple(n * s for n in lat)
    basic = build_basic_partition(measure(shape, seed), s)
    for part in build_composite_partitions(basic):
        allc = sorted(j for b in part.batches for j in b)
        assert allc == list(range(part.n_cells))
        for batch in part.batches:
            pos = [np.array(part.positions[j]) for j in batch]
            for p, q in itertools.combinations(pos, 2):
                assert np.abs(p - q).sum() != 1
        assert build_staggered_batches(part, len(lat)) == part.batches


def test_make_decomposition_single_partition():
    dec = make_decomposition(measure((16, 16)), 4, single_partition=True)
    assert len(dec.composites) == 1 and dec.composites[0].label == "A"


@pytest.mark.parametrize("shape,s", [((64, 64), 8), ((16, 16, 16), 4), ((12, 8), 4), ((32,), 2)])
def test_vectorised_basic_partition_matches_block_loop(shape, s):
    """The whole-array builder gives the block-by-block loop's cells, node lists and
    masses bitwise (partitions.py:77-118 restated as a loop)."""
    rng = np.random.default_rng(7)
    m = rng.uniform(0.0, 1.0, shape) ** 3
    m[rng.uniform(size=shape) < 0.1] = 0.0
    mu = GridMeasure(Grid(shape, 1.0 / shape[-1], (0.0,) * len(shape)), m)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        basic = build_basic_partition(mu, s)
    lat = tuple(n // s for n in shape)
    flat = np.arange(m.size).reshape(shape)
    nodes, masses, boxes = [], [], []
    for pos in itertools.product(*(range(n) for n in lat)):
        sl = tuple(slice(p * s, p * s + s) for p in pos)
        keep = m[sl] > 0
        if not keep.any():
            continue
        nodes.append(flat[sl][keep].ravel())
        masses.append(float(m[sl].sum()))
        boxes.append(tuple((p * s, s) for p in pos))
    assert basic.cell_boxes == boxes
    assert np.array_equal(basic.masses, np.array(masses))
    assert all(np.array_equal(a, b) for a, b in zip(basic.nodes_of_cell, nodes))
