"""Oracle problem setup: embed a (mu, nu) pair and its decomposition in 2D.

Test-only.  Partition tables come from the host partition builder
(``paper_2410_08859_b200.decomposition``, which restates the reference's
partitions.py); golden fixtures pin both.
"""

from __future__ import annotations

import warnings

import numpy as np

from paper_2410_08859_b200.decomposition import as2d_box, make_decomposition
from paper_2410_08859_b200.grids import Grid, GridMeasure

from .ref_cell import Ctx


def embed(arr, org):
    arr = np.asarray(arr, dtype=np.float64)
    if arr.ndim == 1:
        return arr.reshape(1, -1), (0.0, float(org[0]))
    return arr, (float(org[0]), float(org[1]))


def make_ctx(mu, nu, dx: float, origin, lam: float, eps: float, s: int,
             single_partition: bool = False, y_dx: float | None = None, y_origin=None) -> Ctx:
    """Ctx for mu on grid (dx, origin) and nu on (y_dx, y_origin) (defaults: same grid)."""
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    y_dx = dx if y_dx is None else y_dx
    y_origin = origin if y_origin is None else y_origin
    gx = Grid(mu.shape, dx, tuple(origin))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(GridMeasure(gx, mu), s, single_partition)
    mu2, xo = embed(mu, origin)
    nu2, yo = embed(nu, y_origin)
    parts = []
    for p in dec.composites:
        parts.append(dict(label=p.label,
                          xbox=[tuple(c for ax in as2d_box(b) for c in ax) for b in p.boxes],
                          members=[p.real_members(j) for j in range(p.n_cells)],
                          batches=[list(b) for b in p.batches]))
    boxes = [tuple(c for ax in as2d_box(b) for c in ax) for b in dec.basic.cell_boxes]
    return Ctx(mu=mu2, nu=nu2, x_dx=float(dx), x_org=xo, y_dx=float(y_dx), y_org=yo,
               lam=float(lam), eps=float(eps), basic_box=boxes,
               basic_mass=dec.basic.masses.copy(), parts=parts)
