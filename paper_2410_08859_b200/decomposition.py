"""Basic / composite partitions of the X grid and their staggered batches.

Host-side setup mirroring the reference partition API (``domdec.partitions``:
BasicPartition :27, CompositePartition :54, build_basic_partition :77,
build_composite_partitions :160, build_staggered_batches :191;
``domdec.engine``: Decomposition :139, make_decomposition :146).

Semantics (paper Def. 2.4 and §4.3.1):
* basic cells are s^d node blocks enumerated row-major over the block
  lattice; blocks whose mu mass is identically zero are dropped;
* composite partition A groups 2^d blocks starting at even lattice
  coordinates, B is shifted by one block on every axis; slots that fall off
  the lattice (or on a dropped block) are virtual padding members;
* with fewer than two blocks on some axis both partitions degenerate to one
  cell holding every basic cell (with a warning);
* each partition splits into 2^d batches by composite-lattice parity.

The engine builds the integer tables the CUDA library consumes from these
objects (1D problems embedded as 2D grids of shape (1, n)).
"""

from __future__ import annotations

import logging
import warnings
from dataclasses import dataclass
from itertools import product

import numpy as np

from .grids import Grid, GridMeasure

logger = logging.getLogger(__name__)

__all__ = [
    "BasicPartition", "CompositePartition", "Decomposition", "build_basic_partition",
    "build_composite_partitions", "build_staggered_batches", "make_decomposition",
]


@dataclass(frozen=True)
class BasicPartition:
    grid: Grid
    s: int
    cell_of_node: np.ndarray
    nodes_of_cell: list
    cell_boxes: list
    lattice_dims: tuple
    lattice_to_cell: np.ndarray
    positions: np.ndarray
    masses: np.ndarray

    @property
    def n_cells(self) -> int:
        return len(self.nodes_of_cell)

    @property
    def ndim(self) -> int:
        return len(self.lattice_dims)


@dataclass(frozen=True)
class CompositePartition:
    label: str
    cells: list
    boxes: list
    positions: list
    batches: list
    n_basic: int

    @property
    def n_cells(self) -> int:
        return len(self.cells)

    def real_members(self, j: int) -> list:
        return [i for i in self.cells[j] if i < self.n_basic]


def _blocks(arr: np.ndarray, s: int) -> np.ndarray:
    """(n_blocks, s^d) view-copy of an s^d-blocked array: blocks in row-major lattice
    order, nodes row-major inside each block (the order of itertools.product loops)."""
    d = arr.ndim
    lat = tuple(n // s for n in arr.shape)
    shp = []
    for n in lat:
        shp += [n, s]
    perm = tuple(range(0, 2 * d, 2)) + tuple(range(1, 2 * d, 2))
    return arr.reshape(shp).transpose(perm).reshape(int(np.prod(lat)), s ** d)


def build_basic_partition(mu: GridMeasure, s: int) -> BasicPartition:
    """s^d blocks of the grid, zero-mass blocks dropped (partitions.py:77-118); built with
    whole-array operations (the same cells, order, node lists and masses as a
    block-by-block loop)."""
    grid = mu.grid
    dims = grid.dims
    if s < 1 or any(n % s for n in dims):
        raise ValueError(f"cell size {s} must divide the grid dims {dims}")
    lat = tuple(n // s for n in dims)
    mass = np.asarray(mu.mass)
    flat = np.arange(mass.size).reshape(dims)
    blk_mass = _blocks(mass, s)
    blk_ids = _blocks(flat, s)
    keep = blk_mass > 0
    live = keep.any(axis=1)
    n_dropped = int((~live).sum())
    if n_dropped:
        logger.warning("dropped %d of %d zero-mass basic cells", n_dropped, len(live))
    if not live.any():
        raise ValueError("no basic cell has positive mass")
    which = np.flatnonzero(live)
    lattice_to_cell = np.full(len(live), -1, dtype=np.int64)
    lattice_to_cell[which] = np.arange(len(which))
    lattice_to_cell = lattice_to_cell.reshape(lat)
    kept = keep[which]
    counts = kept.sum(axis=1)
    ids = blk_ids[which][kept]
    nodes = np.split(ids, np.cumsum(counts)[:-1])
    # block masses: numpy sums a strided block through a contiguous buffer, so the row
    # sums equal the reference's float(block.sum()) bitwise (checked in the host tests)
    sl_mass = blk_mass[which].sum(axis=1)
    positions = np.stack(np.unravel_index(which, lat), axis=1).astype(np.int64)
    boxes = [tuple((p, s) for p in row) for row in (positions * s).tolist()]
    cell_of_node = np.full(mass.size, -1, dtype=np.int64)
    cell_of_node[ids] = np.repeat(np.arange(len(which)), counts)
    return BasicPartition(
        grid=grid, s=s, cell_of_node=cell_of_node, nodes_of_cell=nodes, cell_boxes=boxes,
        lattice_dims=lat, lattice_to_cell=lattice_to_cell,
        positions=positions.reshape(len(which), len(dims)),
        masses=np.asarray(sl_mass, dtype=np.float64),
    )


def build_staggered_batches(part: CompositePartition, ndim: int) -> list:
    """2^d parity groups of composite cells (no two cells of a group share an edge)."""
    groups = [[] for _ in range(1 << ndim)]
    for j, pos in enumerate(part.positions):
        key = sum((int(pos[a]) & 1) << a for a in range(ndim))
        groups[key].append(j)
    return [g for g in groups if g]


def _group(basic: BasicPartition, starts: list, label: str) -> CompositePartition:
    """Composite cells of 2^d blocks at the given per-axis starts (partitions.py:121-157):
    member slots row-major over the 2-per-axis window, padding ids numbered in slot order
    over every window (kept or not), windows without a real member dropped."""
    s, lat, d = basic.s, basic.lattice_dims, basic.ndim
    grids = np.meshgrid(*[np.asarray(st, dtype=np.int64) for st in starts], indexing="ij")
    origin = np.stack([g.ravel() for g in grids], axis=1)                # (nc, d)
    cgrid = np.meshgrid(*[np.arange(len(st)) for st in starts], indexing="ij")
    cpos = np.stack([g.ravel() for g in cgrid], axis=1)
    offs = np.array(list(product(range(2), repeat=d)), dtype=np.int64)   # (2^d, d)
    b = origin[:, None, :] + offs[None, :, :]                           # (nc, 2^d, d)
    inside = np.all((b >= 0) & (b < np.asarray(lat)), axis=2)
    bc = np.clip(b, 0, np.asarray(lat) - 1)
    cid = np.where(inside, basic.lattice_to_cell[tuple(bc[..., a] for a in range(d))], -1)
    pad_flag = cid < 0
    pad_ids = basic.n_cells + np.cumsum(pad_flag.ravel()).reshape(pad_flag.shape) - 1
    slots = np.where(pad_flag, pad_ids, cid)
    real = (~pad_flag).sum(axis=1)
    keep = np.flatnonzero(real > 0)
    cells = slots[keep].tolist()
    boxes = [tuple((int(o) * s, 2 * s) for o in origin[j]) for j in keep]
    positions = [tuple(int(x) for x in cpos[j]) for j in keep]
    part = CompositePartition(label, cells, boxes, positions, [], basic.n_cells)
    return CompositePartition(label, cells, boxes, positions, build_staggered_batches(part, d),
                              basic.n_cells)


def build_composite_partitions(basic: BasicPartition) -> tuple:
    lat = basic.lattice_dims
    if min(lat) < 2:
        warnings.warn("fewer than 2 basic cells along an axis; partitions degenerate to one "
                      "global cell", stacklevel=2)
        everyone = list(range(basic.n_cells))
        return tuple(
            CompositePartition(lb, [everyone], [basic.grid.full_box()], [(0,) * len(lat)], [[0]],
                               basic.n_cells)
            for lb in ("A", "B"))
    a = _group(basic, [list(range(0, n, 2)) for n in lat], "A")
    b = _group(basic, [list(range(-1, n, 2)) for n in lat], "B")
    return a, b


@dataclass(frozen=True)
class Decomposition:
    basic: BasicPartition
    composites: tuple


def make_decomposition(mu: GridMeasure, s: int, single_partition: bool = False) -> Decomposition:
    basic = build_basic_partition(mu, s)
    a, b = build_composite_partitions(basic)
    return Decomposition(basic=basic, composites=(a,) if single_partition else (a, b))


# -- device export ---------------------------------------------------------------

MAX_MEMBERS = 64


def as2d_box(box) -> tuple:
    """Embed a 1D box as the 2D box ((0, 1), box[0])."""
    return tuple(box) if len(box) == 2 else ((0, 1), tuple(box[0]))


