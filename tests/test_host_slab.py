"""Host logic of the row-slab sharding (slab.py): bounds, ownership, halo sets."""

import warnings

import numpy as np
import pytest

from paper_2410_08859_b200 import Grid, GridMeasure, make_decomposition
from paper_2410_08859_b200.engine import _tables
from paper_2410_08859_b200.slab import basic_owners, composite_owners, halo_sets, slab_bounds


@pytest.mark.parametrize("rows,world", [(16, 2), (16, 3), (128, 8), (64, 5), (7, 2), (4, 4)])
def test_slab_bounds_even_monotone_cover(rows, world):
    b = slab_bounds(rows, world)
    assert b[0] == 0 and b[-1] == rows and len(b) == world + 1
    assert np.all(np.diff(b) >= 0)
    assert all(x % 2 == 0 for x in b[1:-1])         # A composites never straddle


def _dec(n, s, dims=2):
    g = Grid((n, n) if dims == 2 else (n,), 1.0 / n, (0.5 / n,) * dims)
    mass = np.ones((n, n) if dims == 2 else (n,))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return make_decomposition(GridMeasure(g, mass), s)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_ownership_and_halo_are_the_boundary_rows(world):
    n, s = 128, 4                       # 32 x 32 basic lattice
    dec = _dec(n, s)
    lat = dec.basic.lattice_to_cell.shape
    bounds = slab_bounds(lat[0], world)
    owners = []
    for part in dec.composites:
        pt = _tables(part)
        comp = composite_owners(np.floor_divide(pt.xbox[:, 0], s), bounds)
        basic = basic_owners(pt.mem, pt.nmem, comp, dec.basic.n_cells)
        assert np.all(basic >= 0)                    # every basic cell has an owner
        # a composite's members all sit in its owner's slab, except the B boundary row
        owners.append(basic)
    ba, bb = owners
    rows = dec.basic.positions[:, 0]
    # under A every basic cell belongs to the slab holding its row
    assert np.array_equal(ba, np.searchsorted(bounds, rows, side="right") - 1)
    moved_rows = sorted(set(rows[ba != bb].tolist()))
    assert moved_rows == sorted(int(r) for r in bounds[1:-1] if 0 < r < lat[0])
    # the halo each rank receives at the A -> B switch is its lower neighbour's...
    # boundary row cells moving down one rank
    for r in range(world):
        send, recv = halo_sets(ba, bb, r)
        for q, ids in send.items():
            assert q == r - 1 and set(rows[ids].tolist()) == {int(bounds[r])}
        for q, ids in recv.items():
            assert q == r + 1 and set(rows[ids].tolist()) == {int(bounds[r + 1])}


def test_one_dimensional_problems_slab_along_the_lattice():
    from paper_2410_08859_b200.slab import ShardSpec

    dec = _dec(64, 2, dims=1)                       # 32 basic cells in a row
    sp = object.__new__(ShardSpec)
    sp.world, sp.rank, sp._cache = 2, 0, {}
    pt = _tables(dec.composites[0])
    lat = dec.basic.lattice_to_cell.shape
    comp, basic = sp.layout(pt, (1, 2), dec.basic.n_cells, 1, lat[0])
    assert set(comp.tolist()) == {0, 1}
    assert np.array_equal(basic[:16], np.zeros(16)) and np.array_equal(basic[16:], np.ones(16))
