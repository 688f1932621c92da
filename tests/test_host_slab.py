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


def test_three_axis_zslab_layout_halo_is_the_boundary_layer():
    """configs[4]-shaped decomposition (16^3, 4^3 cells, 2^3 composites) sharded over 2
    ranks along z: A composites never straddle the slab boundary, B composites that do
    belong to the lower rank, and the basic cells changing owner between the A and
    B sweeps are exactly the boundary z-layer of the block lattice."""
    import warnings

    import numpy as np

    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.decomposition import make_decomposition
    from paper_2410_08859_b200.slab import ShardSpec, halo_sets
    from paper_2410_08859_b200.volume import _PartTables3

    n, s = 16, 4
    mu = np.ones((n, n, n))
    prob = TransportProblem(GridMeasure(Grid((n, n, n), 1 / n, (0.0,) * 3), mu),
                            GridMeasure(Grid((n, n, n), 1 / n, (0.0,) * 3), mu),
                            DivergenceSpec(1.0), 1e-3)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(prob.mu, s)
    sh = object.__new__(ShardSpec)
    sh.world, sh.rank, sh._cache = 2, 0, {}
    import types
    owners = {}
    for part in dec.composites:
        pt = _PartTables3(part)
        view = types.SimpleNamespace(xbox=pt.xbox[:, 0:4], mem=pt.mem, nmem=pt.nmem)
        comp, basic = sh.layout(view, (s, s), dec.basic.n_basic if hasattr(dec.basic, "n_basic")
                                else dec.basic.n_cells, 4, 4)
        owners[part.label] = (pt, comp, basic)
    pos = dec.basic.positions           # (n_cells, 3) block-lattice coordinates
    pa, ca, ba = owners["A"]
    pb, cb, bb = owners["B"]
    assert set(np.unique(ba)) == {0, 1} and set(np.unique(bb)) == {0, 1}
    # A: z-slab {0,1} -> rank 0, {2,3} -> rank 1
    assert np.array_equal(ba, (pos[:, 0] >= 2).astype(np.int64))
    moved = np.flatnonzero(ba != bb)
    assert set(pos[moved, 0].tolist()) == {2}      # the boundary layer z = 2 only
    send, recv = halo_sets(ba, bb, 1)
    assert list(send) == [0] and np.array_equal(np.sort(send[0]), np.sort(moved))
