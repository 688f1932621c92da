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


def build_basic_partition(mu: GridMeasure, s: int) -> BasicPartition:
    grid = mu.grid
    dims = grid.dims
    if s < 1 or any(n % s for n in dims):
        raise ValueError(f"cell size {s} must divide the grid dims {dims}")
    lat = tuple(n // s for n in dims)
    flat = np.arange(mu.mass.size).reshape(dims)
    lattice_to_cell = np.full(lat, -1, dtype=np.int64)
    nodes, boxes, masses, positions = [], [], [], []
    n_dropped = 0
    for pos in product(*[range(n) for n in lat]):
        sl = tuple(slice(p * s, p * s + s) for p in pos)
        blk = mu.mass[sl]
        keep = blk > 0
        if not keep.any():
            n_dropped += 1
            continue
        lattice_to_cell[pos] = len(nodes)
        nodes.append(flat[sl][keep].ravel())
        boxes.append(tuple((p * s, s) for p in pos))
        masses.append(float(blk.sum()))
        positions.append(pos)
    if n_dropped:
        logger.warning("dropped %d of %d zero-mass basic cells", n_dropped, n_dropped + len(nodes))
    if not nodes:
        raise ValueError("no basic cell has positive mass")
    cell_of_node = np.full(mu.mass.size, -1, dtype=np.int64)
    for c, ids in enumerate(nodes):
        cell_of_node[ids] = c
    return BasicPartition(
        grid=grid, s=s, cell_of_node=cell_of_node, nodes_of_cell=nodes, cell_boxes=boxes,
        lattice_dims=lat, lattice_to_cell=lattice_to_cell,
        positions=np.array(positions, dtype=np.int64).reshape(len(nodes), len(dims)),
        masses=np.asarray(masses, dtype=np.float64),
    )


def build_staggered_batches(part: CompositePartition, ndim: int) -> list:
    """2^d parity groups of composite cells (no two cells of a group share an edge)."""
    groups = [[] for _ in range(1 << ndim)]
    for j, pos in enumerate(part.positions):
        key = sum((int(pos[a]) & 1) << a for a in range(ndim))
        groups[key].append(j)
    return [g for g in groups if g]


def _group(basic: BasicPartition, starts: list, label: str) -> CompositePartition:
    s, lat, d = basic.s, basic.lattice_dims, basic.ndim
    pad = basic.n_cells
    cells, boxes, positions = [], [], []
    for cpos in product(*[range(len(st)) for st in starts]):
        origin = tuple(starts[a][cpos[a]] for a in range(d))
        slots, real = [], 0
        for off in product(range(2), repeat=d):
            b = tuple(o + k for o, k in zip(origin, off))
            cid = int(basic.lattice_to_cell[b]) if all(0 <= p < n for p, n in zip(b, lat)) else -1
            if cid < 0:
                slots.append(pad)
                pad += 1
            else:
                slots.append(cid)
                real += 1
        if real:
            cells.append(slots)
            boxes.append(tuple((o * s, 2 * s) for o in origin))
            positions.append(cpos)
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


