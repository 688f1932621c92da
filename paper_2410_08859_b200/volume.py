"""Three-axis domain decomposition on the device (BASELINE configs[4]: 3D 128^3).

The reference's solve path (``domdec.engine`` / ``domdec.cells`` /
``domdec.sinkhorn``) laid out for grids of up to three axes.  The reference
itself is dimension-generic except for two guards: ``Grid`` accepts only 1D/2D
(measures.py:76-77) and ``SeparableKernel._sweep`` reduces at most two axes
(sinkhorn.py:159-175).  Here a problem of d <= 3 axes is embedded as a 3D grid
(leading unit axes: (n0, n1) -> (1, n0, n1)); the separable sweep reduces axis
2, then 1, then 0 -- the 2D sweep's order extended by one axis.  Because the
embedding is exact, the whole path is checked against every 1D/2D reference
fixture as well as against 3D fixtures the reference produced with its two
guards lifted (``scripts/make_golden.py vol3``).

Kernels (csrc/vol.cu, C ABI ``dd3_*`` in include/domdec_b200.h): one CTA per
composite cell runs window assembly, the Sinkhorn loop with the Newton Y-step,
splitting, balancing, truncation, fragments and X-marginals
(``dd3_cell_solve``); ``dd3_cell_delta`` / ``dd3_gather`` give the staggered
strategy's blend energies; ``dd3_cell_commit`` installs a batch; ``dd3_gather``
is the fixed-order assembly; ``dd3_grid_lse`` the full-grid three-axis sweep of
the global Sinkhorn solver and the stopping certificate.

Strategies: ``staggered`` (the reference default), ``fast`` and ``safe``.
Multi-GPU: under ``engine.set_shard()`` the solve is slab-sharded along the first
real axis (z-slabs for 3D, configs[4]) with the 2D path's slab layer (slab.py).
There is no CPU path: every call goes through libdomdec_b200.
"""

from __future__ import annotations

import ctypes
import math
import time
import warnings

import numpy as np

from . import _lib
from .decomposition import CompositePartition, Decomposition, make_decomposition
from .grids import GridMeasure, SparseCellMarginal, TransportProblem
from .report import SolveReport, TraceRow
from .sinkhorn import SolverConfig, mass_balanced_start, sinkhorn_solve

__all__ = ["VolumeProblem", "GridSweeper3", "PlanState3", "initial_plan_state3",
           "warm_start_plan3", "iteration_parallel3", "domdec_solve3", "multiscale_solve3",
           "STRATEGIES_3D"]

STRATEGIES_3D = ("staggered", "fast", "safe", "swift", "opt", "sequential")
MAX_MEMBERS = 64


def _dims3(dims) -> tuple:
    d = tuple(int(n) for n in dims)
    return (1,) * (3 - len(d)) + d


def _box6(box) -> list:
    b = [(0, 1)] * (3 - len(box)) + [tuple(int(x) for x in ax) for ax in box]
    return [c for ax in b for c in ax]


def _box_from6(b6, ndim: int) -> tuple:
    b = [int(x) for x in b6]
    if b[1] == 0 or b[3] == 0 or b[5] == 0:
        return ((0, 0),) * ndim
    axes = ((b[0], b[1]), (b[2], b[3]), (b[4], b[5]))
    return axes[3 - ndim:]


class VolumeProblem:
    """Device copies of mu, nu (3D-embedded), their logs and the dd3 geometry.

    Duck-types :class:`sinkhorn.DeviceProblem` for the global solver and the
    certificate (``make_sweeper`` gives the three-axis sweep)."""

    device_loop = True    # sinkhorn_solve runs its loop on the device (dd3_sinkhorn_run)

    def __init__(self, problem: TransportProblem, device=None):
        import torch

        _lib.lib()
        self.problem = problem
        self.device = torch.device(device or "cuda")
        gx, gy = problem.mu.grid, problem.nu.grid
        self.ndim = gx.ndim
        if self.ndim > 3:
            raise ValueError("at most three grid axes")
        self.shape_x, self.shape_y = _dims3(gx.dims), _dims3(gy.dims)
        mu = np.asarray(problem.mu.mass, dtype=np.float64).reshape(self.shape_x)
        nu = np.asarray(problem.nu.mass, dtype=np.float64).reshape(self.shape_y)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).ravel()).to(self.device)  # noqa
        self.mu, self.nu = t(mu), t(nu)
        with np.errstate(divide="ignore"):
            self.log_mu, self.log_nu = t(np.log(mu)), t(np.log(nu))
        pad = 3 - self.ndim
        g = _lib.Geom3()
        for a in range(3):
            g.nx[a] = self.shape_x[a]
            g.ny[a] = self.shape_y[a]
            g.x_org[a] = 0.0 if a < pad else float(gx.origin[a - pad])
            g.y_org[a] = 0.0 if a < pad else float(gy.origin[a - pad])
        g.first_axis = pad
        g.x_dx, g.y_dx = float(gx.dx), float(gy.dx)
        g.eps, g.lam = float(problem.eps), float(problem.div.lam)
        g.nu_total = float(problem.nu.total_mass)
        self.geom = g
        self.nx, self.ny = mu.size, nu.size
        self.mu_total = float(problem.mu.total_mass)
        self.nu_total = float(problem.nu.total_mass)
        self.partial = torch.empty(max(8192, self.ny // 32 + 64), dtype=torch.float64,
                                   device=self.device)
        self.sums = torch.zeros(8, dtype=torch.float64, device=self.device)

    def set_eps(self, eps: float) -> None:
        self.geom.eps = float(eps)

    def make_sweeper(self) -> "GridSweeper3":
        return GridSweeper3(self)

    def sinkhorn_ws(self) -> int:
        return int(_lib.lib().dd3_sinkhorn_ws(self.geom))

    def sinkhorn_run(self, *args) -> int:
        return _lib.lib().dd3_sinkhorn_run(self.geom, *args)

    def empty_x(self):
        import torch
        return torch.empty(self.nx, dtype=torch.float64, device=self.device)

    def empty_y(self):
        import torch
        return torch.empty(self.ny, dtype=torch.float64, device=self.device)


class GridSweeper3:
    """Three-axis separable log-sum-exp over the full grids (``dd3_grid_lse``)."""

    def __init__(self, dp: VolumeProblem):
        import torch

        self.dp = dp
        n = int(_lib.lib().dd3_grid_ws(dp.geom))
        self.work = torch.empty(n, dtype=torch.float64, device=dp.device)
        self.sweeps = 0
        self._tab_eps = {0: None, 1: None}   # eps each direction's tables were built for

    def _sweep(self, v, to_x: int, out=None):
        out = out if out is not None else (self.dp.empty_x() if to_x else self.dp.empty_y())
        eps = float(self.dp.geom.eps)
        ready = 1 if self._tab_eps[to_x] == eps else 0
        _lib.check(_lib.lib().dd3_grid_lse(self.dp.geom, v.data_ptr(), out.data_ptr(), to_x,
                                           self.work.data_ptr(), ready, _lib.stream_handle()))
        self._tab_eps[to_x] = eps
        self.sweeps += 1
        return out

    def lse_x(self, b, out=None):
        return self._sweep(b, 1, out)

    def lse_y(self, a, out=None):
        return self._sweep(a, 0, out)


def _shard():
    """The active slab sharding (engine.set_shard) when it spans more than one rank."""
    from . import engine

    sh = engine._SHARD
    return sh if (sh is not None and sh.world > 1) else None


def _slab_layout3(st: "PlanState3", pt: "_PartTables3"):
    """(composite owner, basic-cell owner) under the active sharding: slabs of the first
    real grid axis (z for 3D), cut as in slab.py (``ShardSpec.layout``)."""
    import types

    lat = st.basic.lattice_dims
    nd = len(lat)
    a0 = 3 - nd if nd > 1 else 1        # first two real axes of the 6-int boxes
    rows, cols = (lat[0], lat[1]) if nd > 1 else (1, lat[0])
    view = types.SimpleNamespace(xbox=pt.xbox[:, 2 * a0:2 * a0 + 4], mem=pt.mem, nmem=pt.nmem)
    return _shard().layout(view, (st.block[a0], st.block[a0 + 1]), st.n_basic, rows, cols)


def _i32(vals) -> ctypes.Array:
    v = [int(x) for x in vals]
    return (ctypes.c_int32 * len(v))(*v)


# -- the iterate ----------------------------------------------------------------------

class _PartTables3:
    def __init__(self, part: CompositePartition):
        self.part = part
        self.label = part.label
        self.ncomp = part.n_cells
        self.xbox = np.array([_box6(b) for b in part.boxes], dtype=np.int32).reshape(-1, 6)
        self.nxw = (int(self.xbox[0, 1]), int(self.xbox[0, 3]), int(self.xbox[0, 5]))
        if any(np.any(self.xbox[:, 2 * a + 1] != self.nxw[a]) for a in range(3)):
            raise ValueError("composite cells of one partition must share the window shape")
        mems = [part.real_members(j) for j in range(self.ncomp)]
        width = max(1, max(len(m) for m in mems))
        if width > MAX_MEMBERS:
            raise ValueError(f"composite cell with {width} members exceeds {MAX_MEMBERS}")
        self.mem = np.full((self.ncomp, width), -1, dtype=np.int32)
        for j, m in enumerate(mems):
            self.mem[j, :len(m)] = m
        self.nmem = np.array([len(m) for m in mems], dtype=np.int32)
        self.batches = [np.asarray(b, dtype=np.int64) for b in part.batches]


_TABLES: dict = {}


def _tables(part: CompositePartition) -> _PartTables3:
    hit = _TABLES.get(id(part))
    if hit is None or hit.part is not part:
        hit = _PartTables3(part)
        _TABLES[id(part)] = hit
    return hit


class _Store3:
    """Warm-start duals of one partition: alpha per cell, boxed beta per cell."""

    def __init__(self, ncomp: int, nx: int, dcap: int, device):
        import torch

        self.ncomp, self.nx = ncomp, nx
        self.alpha = torch.zeros(ncomp * nx, dtype=torch.float64, device=device)
        self.has = torch.zeros(ncomp, dtype=torch.int32, device=device)
        self.box = torch.zeros(ncomp * 6, dtype=torch.int32, device=device)
        self.dcap = int(max(1, dcap))
        self.beta = torch.zeros(ncomp * self.dcap, dtype=torch.float64, device=device)

    def ensure(self, need: int):
        import torch

        if need <= self.dcap:
            return
        new = max(int(need), int(self.dcap * 1.25) + 1)
        nb = torch.zeros(self.ncomp * new, dtype=torch.float64, device=self.beta.device)
        nb.view(self.ncomp, new)[:, :self.dcap] = self.beta.view(self.ncomp, self.dcap)
        self.beta, self.dcap = nb, new

    def resize(self, cap: int):
        """Exactly ``cap`` beta entries per cell (>= the current capacity); ranks of a
        sharded solve agree on one size before their stores are summed."""
        import torch

        if cap == self.dcap:
            return
        nb = torch.zeros(self.ncomp * cap, dtype=torch.float64, device=self.beta.device)
        nb.view(self.ncomp, cap)[:, :self.dcap] = self.beta.view(self.ncomp, self.dcap)
        self.beta, self.dcap = nb, cap

    def clone(self):
        c = object.__new__(_Store3)
        c.ncomp, c.nx, c.dcap = self.ncomp, self.nx, self.dcap
        c.alpha, c.has, c.box, c.beta = (self.alpha.clone(), self.has.clone(), self.box.clone(),
                                         self.beta.clone())
        return c


class _Bufs:
    def __init__(self, device):
        self.device, self.bufs = device, {}

    def get(self, name: str, n: int, dtype):
        import torch

        n = max(1, int(n))
        t = self.bufs.get(name)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.empty(int(n * 1.25) + 16, dtype=dtype, device=self.device)
            self.bufs[name] = t
        return t


class PlanState3:
    """Device-resident iterate of the three-axis path (engine.py:157-216): per basic
    cell a boxed Y-marginal (6-int box, fixed-capacity slot), a dense X-marginal over
    its block, score fragments, and per-partition dual stores."""

    def __init__(self, problem: TransportProblem, basic, dp: VolumeProblem | None = None,
                 cap: int = 1):
        import torch

        self.problem = problem
        self.basic = basic
        self.dp = dp if dp is not None else VolumeProblem(problem)
        dev = self.dp.device
        self.ndim = problem.mu.grid.ndim
        nb = basic.n_cells
        self.n_basic = nb
        bx = np.array([_box6(b) for b in basic.cell_boxes], dtype=np.int32).reshape(-1, 6)
        self.block = (int(bx[0, 1]), int(bx[0, 3]), int(bx[0, 5]))
        self.bs = self.block[0] * self.block[1] * self.block[2]
        self.basic_xbox = torch.from_numpy(bx.ravel().copy()).to(dev)
        self.basic_mass = torch.from_numpy(np.asarray(basic.masses, dtype=np.float64)).to(dev)
        self.cap = int(max(1, cap))
        self.ybox = torch.zeros(nb * 6, dtype=torch.int32, device=dev)
        self.yval = torch.zeros(nb * self.cap, dtype=torch.float64, device=dev)
        self.ybox_h = np.zeros((nb, 6), dtype=np.int32)
        self.x_marg_d = torch.zeros(nb * self.bs, dtype=torch.float64, device=dev)
        self.transport_d = torch.zeros(nb, dtype=torch.float64, device=dev)
        self.kl_d = torch.zeros(nb, dtype=torch.float64, device=dev)
        self.stores: dict = {}
        self.truncated_mass = 0.0
        self.global_duals = None
        self.buf = _Bufs(dev)
        self.terms = torch.zeros(nb * 4, dtype=torch.float64, device=dev)
        # slab mode (engine.set_shard): owning rank of each basic cell (None: all here)
        self.owner = None
        self._mask_d = None
        self.comp_owner: dict = {}

    box_width = 6

    def set_owner(self, owner) -> None:
        """Slab mode: the owning rank of every basic cell (None: all current here)."""
        import torch

        sh = _shard()
        self.owner = None if owner is None else np.asarray(owner, dtype=np.int64).copy()
        if self.owner is None or sh is None:
            self._mask_d = None
        else:
            m = (self.owner == sh.rank).astype(np.float64)
            self._mask_d = torch.from_numpy(m).to(self.dp.device)

    def _sharded(self) -> bool:
        return _shard() is not None and self._mask_d is not None

    def state_struct(self, store: _Store3 | None = None) -> _lib.State3:
        dp = self.dp
        s = _lib.State3(mu=dp.mu.data_ptr(), nu=dp.nu.data_ptr(), log_mu=dp.log_mu.data_ptr(),
                        log_nu=dp.log_nu.data_ptr(), n_basic=self.n_basic,
                        basic_xbox=self.basic_xbox.data_ptr(),
                        basic_mass=self.basic_mass.data_ptr(), ybox=self.ybox.data_ptr(),
                        yval=self.yval.data_ptr(), cap=self.cap, x_marg=self.x_marg_d.data_ptr(),
                        transport=self.transport_d.data_ptr(), kl=self.kl_d.data_ptr())
        for a in range(3):
            s.block[a] = self.block[a]
        if store is not None:
            s.d_alpha = store.alpha.data_ptr()
            s.d_has = store.has.data_ptr()
            s.d_box = store.box.data_ptr()
            s.d_beta = store.beta.data_ptr()
            s.d_cap = store.dcap
        return s

    def ensure_cap(self, need: int):
        import torch

        if need <= self.cap:
            return
        new = max(int(need), int(self.cap * 1.25) + 1)
        nv = torch.zeros(self.n_basic * new, dtype=torch.float64, device=self.yval.device)
        nv.view(self.n_basic, new)[:, :self.cap] = self.yval.view(self.n_basic, self.cap)
        self.yval, self.cap = nv, new

    def store(self, pt: _PartTables3) -> _Store3:
        st = self.stores.get(pt.label)
        if st is None:
            st = _Store3(pt.ncomp, pt.nxw[0] * pt.nxw[1] * pt.nxw[2], 1, self.dp.device)
            self.stores[pt.label] = st
        return st

    def sync_boxes(self):
        self.ybox_h = self.ybox.view(-1, 6).cpu().numpy().copy()

    # ---- energy (engine.py:182-196)
    def assemble_device(self, out=None):
        """Fixed-order sum of the basic-cell marginals (measures.py:410-425).  Slab
        mode: each rank sums its own basic cells (mask as item scale) and one dense
        all-reduce completes the grid."""
        out = out if out is not None else self.dp.empty_y()
        sharded = self._sharded()
        _lib.check(_lib.lib().dd3_gather(
            self.dp.geom, self.n_basic, self.ybox.data_ptr(), 6, self.yval.data_ptr(), self.cap,
            None, self._mask_d.data_ptr() if sharded else None, None, out.data_ptr(), 0, None,
            None, None, _lib.stream_handle()))
        if sharded:
            _shard().all_reduce(out[:self.dp.ny])
        return out

    def _partial(self, y):
        return self.buf.get("partial", self.dp.ny // 32 + 4096, y.dtype)

    def grid_kl(self, y, clip: bool = False, base=None) -> float:
        """KL(y | nu) over the Y grid (y clipped at 0 first with ``clip``); with
        ``base`` the argument is base + y."""
        import torch

        sy = self.dp.shape_y
        full = self.buf.get("fullbox", 6, torch.int32)
        full[:6] = torch.tensor([0, sy[0], 0, sy[1], 0, sy[2]], dtype=torch.int32)
        part = self._partial(y)
        npart = ctypes.c_int(0)
        _lib.check(_lib.lib().dd3_gather(
            self.dp.geom, 1, full.data_ptr(), 6, y.data_ptr(), 0, None, None,
            base.data_ptr() if base is not None else None, None, 2 if clip else 1,
            self.dp.nu.data_ptr(), part.data_ptr(), ctypes.byref(npart), _lib.stream_handle()))
        return float(part[:npart.value].sum().item())

    def cell_terms(self) -> np.ndarray:
        """Per basic cell [transport, kl, KL(x_marg | mu), 0]; slab mode: every rank's
        owned rows summed (other rows are zero), so all ranks hold the full table."""
        _lib.check(_lib.lib().dd3_cell_terms(self.dp.geom, self.state_struct(),
                                             self.terms.data_ptr(), _lib.stream_handle()))
        t = self.terms.view(self.n_basic, 4).cpu().numpy().copy()
        if self._sharded():
            t[self.owner != _shard().rank] = 0.0
            t = _shard().reduce_np(t.ravel(), "sum", self.dp.device).reshape(self.n_basic, 4)
        return t

    def energy(self):
        from .engine import ScoreBreakdown

        y = self.assemble_device(self.buf.get("energy_y", self.dp.ny, self.dp.mu.dtype))
        d2 = self.grid_kl(y)
        t = self.cell_terms()
        lam, eps = self.problem.div.lam, self.problem.eps
        d1 = float(np.cumsum(t[:, 2])[-1]) if self.n_basic else 0.0   # sequential (engine.py:187)
        return ScoreBreakdown(transport=float(t[:, 0].sum()), entropy=eps * float(t[:, 1].sum()),
                              d1=lam * d1, d2=lam * d2)

    def assemble(self) -> GridMeasure:
        y = self.assemble_device().cpu().numpy()
        return GridMeasure(self.problem.nu.grid, y.reshape(self.problem.nu.grid.dims))

    # ---- host views (reference-shaped)
    @property
    def nu_i(self) -> list:
        boxes, flat, offs = self.download_marginals()
        out = []
        for i in range(self.n_basic):
            b = boxes[i]
            box = _box_from6(b, self.ndim)
            if b[1] == 0 or b[3] == 0 or b[5] == 0:
                out.append(SparseCellMarginal.empty(self.ndim))
                continue
            out.append(SparseCellMarginal(box, flat[offs[i]:offs[i + 1]].reshape(
                [e for _, e in box])))
        return out

    def download_marginals(self):
        """(boxes [n_basic, 6], concatenated values, offsets), compacted on the device."""
        import torch

        b = self.ybox.view(-1, 6).to(torch.int64)
        sizes = b[:, 1] * b[:, 3] * b[:, 5]
        vals = self.yval.view(self.n_basic, self.cap)
        idx = torch.arange(self.cap, device=vals.device)[None, :] < sizes[:, None]
        flat = vals[idx].cpu().numpy()
        boxes = self.ybox.view(-1, 6).cpu().numpy()
        szh = boxes[:, 1].astype(np.int64) * boxes[:, 3] * boxes[:, 5]
        offs = np.concatenate([[0], np.cumsum(szh)])
        return boxes, flat, offs

    @property
    def mu_nodes(self) -> list:
        flat = self.problem.mu.mass.ravel()
        return [flat[ids] for ids in self.basic.nodes_of_cell]

    @property
    def x_marg(self) -> list:
        xm = self.x_marg_d.view(self.n_basic, self.bs).cpu().numpy()
        mu = np.asarray(self.problem.mu.mass, dtype=np.float64).reshape(self.dp.shape_x)
        bx = self.basic_xbox.view(-1, 6).cpu().numpy()
        out = []
        for i in range(self.n_basic):
            b = bx[i]
            blk = mu[b[0]:b[0] + b[1], b[2]:b[2] + b[3], b[4]:b[4] + b[5]].ravel()
            out.append(xm[i][blk > 0])
        return out

    @property
    def transport(self) -> np.ndarray:
        return self.transport_d.cpu().numpy()

    @property
    def kl(self) -> np.ndarray:
        return self.kl_d.cpu().numpy()

    @property
    def duals(self) -> dict:
        from .engine import CellDuals

        out = {}
        for label, st in self.stores.items():
            has = st.has.cpu().numpy()
            al = st.alpha.view(st.ncomp, st.nx).cpu().numpy()
            bx = st.box.view(st.ncomp, 6).cpu().numpy()
            be = st.beta.view(st.ncomp, st.dcap).cpu().numpy()
            for j in range(st.ncomp):
                if not has[j]:
                    continue
                b = bx[j]
                out[(label, j)] = CellDuals(alpha=al[j].copy(),
                                            beta_box=_box_from6(b, self.ndim),
                                            beta=be[j, :b[1] * b[3] * b[5]].copy())
        return out

    def sparsity(self) -> dict:
        """Stored and non-zero entries of the basic-cell marginals, counted on the device."""
        import torch

        b = self.ybox.view(-1, 6).to(torch.int64)
        sizes = b[:, 1] * b[:, 3] * b[:, 5]
        vals = self.yval.view(self.n_basic, self.cap)
        idx = torch.arange(self.cap, device=vals.device)[None, :] < sizes[:, None]
        nz = int(((vals != 0) & idx).sum().item())
        return {"stored_entries": int(sizes.sum().item()), "nonzero_entries": nz}

    def clone(self) -> "PlanState3":
        c = object.__new__(PlanState3)
        c.__dict__.update(self.__dict__)
        c.ybox, c.yval = self.ybox.clone(), self.yval.clone()
        c.ybox_h = self.ybox_h.copy()
        c.x_marg_d, c.transport_d, c.kl_d = (self.x_marg_d.clone(), self.transport_d.clone(),
                                             self.kl_d.clone())
        c.stores = {k: v.clone() for k, v in self.stores.items()}
        c.buf = _Bufs(self.dp.device)
        c.terms = self.terms.clone()
        c.owner = None if self.owner is None else self.owner.copy()
        c.comp_owner = dict(self.comp_owner)
        return c


def initial_plan_state3(problem: TransportProblem, basic,
                        dp: VolumeProblem | None = None) -> PlanState3:
    """Product start nu_i = (|mu_i|/|mu|) nu on the full box (engine.py:234-257)."""
    st = PlanState3(problem, basic, dp, cap=problem.nu.grid.nnodes)
    _lib.check(_lib.lib().dd3_product_init(st.dp.geom, st.state_struct(), st.dp.mu_total,
                                           _lib.stream_handle()))
    st.sync_boxes()
    return st


def _union6(boxes: np.ndarray, full: np.ndarray) -> np.ndarray:
    """Row-wise union of member boxes (n, MW, 6); rows with no valid box get ``full``."""
    valid = (boxes[..., 1] > 0) & (boxes[..., 3] > 0) & (boxes[..., 5] > 0)
    big = np.iinfo(np.int32).max
    cols = []
    for a in range(3):
        lo = np.where(valid, boxes[..., 2 * a], big).min(axis=1)
        hi = np.where(valid, boxes[..., 2 * a] + boxes[..., 2 * a + 1], -big).max(axis=1)
        cols += [lo, hi - lo]
    out = np.stack(cols, axis=1).astype(np.int32)
    out[~valid.any(axis=1)] = full
    return out


def _member_boxes(st: PlanState3, pt: _PartTables3, ids) -> np.ndarray:
    mem = pt.mem[ids]
    bx = st.ybox_h[np.where(mem >= 0, mem, 0)]
    bx = np.where((mem >= 0)[..., None], bx, 0)
    sy = st.dp.shape_y
    return _union6(bx, np.array([0, sy[0], 0, sy[1], 0, sy[2]], dtype=np.int32))


def _seed_stores(st: PlanState3, partitions: Decomposition, alpha, beta) -> None:
    import torch

    L = _lib.lib()
    for part in partitions.composites:
        pt = _tables(part)
        yb = _member_boxes(st, pt, np.arange(pt.ncomp))
        store = st.store(pt)
        store.ensure(int((yb[:, 1].astype(np.int64) * yb[:, 3] * yb[:, 5]).max(initial=1)))
        xb_d = torch.from_numpy(pt.xbox.ravel().copy()).to(st.dp.device)
        yb_d = torch.from_numpy(yb.ravel().copy()).to(st.dp.device)
        _lib.check(L.dd3_seed_duals(st.dp.geom, st.state_struct(store), pt.ncomp, _i32(pt.nxw),
                                    xb_d.data_ptr(), yb_d.data_ptr(), alpha.data_ptr(),
                                    beta.data_ptr(), _lib.stream_handle()))


def warm_start_plan3(problem: TransportProblem, partitions: Decomposition, delta: float = 1e-3,
                     max_iters: int = 20_000, trunc_threshold: float = 1e-15,
                     dp: VolumeProblem | None = None, alpha0=None, beta0=None,
                     cut_log: float | None = None) -> PlanState3:
    """Global presolve, plan cut along the basic cells, duals seeded (engine.py:260-345).

    ``cut_log``: terms of the cut plan whose log value (log of alpha+beta-c over eps
    plus log mu nu) lies below it are skipped, and so are whole 4^3 tiles of Y nodes
    bounded below it.  The default keeps every term that is not exactly zero in
    double precision on small grids (-800) and drops terms below e^-60 (1e-26 of a
    node's mass, far under the 1e-15 truncation) from 64^3 nodes up."""
    import torch

    dp = dp if dp is not None else VolumeProblem(problem)
    if cut_log is None:
        cut_log = -60.0 if dp.ny >= 64 ** 3 else -800.0
    import torch as _t
    _t.cuda.synchronize()
    t0 = time.perf_counter()
    res = sinkhorn_solve(dp, alpha0, beta0, config=SolverConfig(delta=delta, max_iters=max_iters))
    _t.cuda.synchronize()
    t1 = time.perf_counter()
    st = PlanState3(problem, partitions.basic, dp, cap=1)
    L = _lib.lib()
    trunc_out = torch.zeros(st.n_basic, dtype=torch.float64, device=dp.device)
    boxes = torch.zeros(st.n_basic * 6, dtype=torch.int32, device=dp.device)
    tiles = torch.empty(int(L.dd3_cut_tiles(dp.geom)), dtype=torch.float64, device=dp.device)
    s = st.state_struct()
    s.yval = None
    _lib.check(L.dd3_cut_plan(dp.geom, s, res.alpha.data_ptr(), res.beta.data_ptr(),
                              float(trunc_threshold), float(cut_log), tiles.data_ptr(),
                              trunc_out.data_ptr(), boxes.data_ptr(), _lib.stream_handle()))
    bh = boxes.view(-1, 6).cpu().numpy().astype(np.int64)
    st.ensure_cap(int((bh[:, 1] * bh[:, 3] * bh[:, 5]).max(initial=1)))
    _lib.check(L.dd3_cut_plan(dp.geom, st.state_struct(), res.alpha.data_ptr(),
                              res.beta.data_ptr(), float(trunc_threshold), float(cut_log),
                              tiles.data_ptr(), trunc_out.data_ptr(), boxes.data_ptr(),
                              _lib.stream_handle()))
    st.sync_boxes()
    st.truncated_mass = float(trunc_out.sum().item())
    st.warm_timing = {"presolve_s": t1 - t0, "presolve_iters": int(res.iterations),
                      "cut_s": time.perf_counter() - t1}
    _seed_stores(st, partitions, res.alpha, res.beta)
    st.global_duals = (res.alpha.clone(), res.beta.clone())
    st.presolve = res
    return st


# -- one batch ----------------------------------------------------------------------------

def _ws_total(w, n0, n1, n2) -> np.ndarray:
    """dd3_cell_ws_size, vectorized (mirrors ws_layout in csrc/vol.cu)."""
    w0, w1, w2 = (int(x) for x in w)
    nx = w0 * w1 * w2
    ny = n0 * n1 * n2
    s1 = np.maximum(w0 * w1 * n2, n0 * n1 * w2)
    s2 = np.maximum(w0 * n1 * n2, n0 * w1 * w2)
    return 5 * nx + 5 * ny + w0 * n0 + w1 * n1 + w2 * n2 + n0 + n1 + n2 + s1 + s2 + 1


def _hot_doubles(w, n0, n1, n2) -> np.ndarray:
    """Shared-memory doubles of a cell's hot arrays (z, beta, stage scratch, axis tables;
    mirrors the kernel's placement in csrc/vol.cu)."""
    w0, w1, w2 = (int(x) for x in w)
    ny = n0 * n1 * n2
    s1 = np.maximum(w0 * w1 * n2, n0 * n1 * w2)
    s2 = np.maximum(w0 * n1 * n2, n0 * w1 * w2)
    return 2 * ny + s1 + s2 + w0 * n0 + w1 * n1 + w2 * n2 + n0 + n1 + n2


class _Batch3:
    """Device arenas and host tables of one solved batch of composite cells."""

    def __init__(self, st: PlanState3, pt: _PartTables3, ids, snapshot, cfg):
        import torch

        dev = st.dp.device
        self.st, self.pt, self.cfg = st, pt, cfg
        ids = np.asarray(ids, dtype=np.int64)
        self.ids = ids
        n = len(ids)
        self.n = n
        yb = _member_boxes(st, pt, ids)
        self.ybox = yb
        ne = [yb[:, 2 * a + 1].astype(np.int64) for a in range(3)]
        ny = ne[0] * ne[1] * ne[2]
        self.ny = ny
        nmem = pt.nmem[ids].astype(np.int64)
        members = [pt.mem[j, :pt.nmem[j]] for j in ids]
        membase = np.concatenate([[0], np.cumsum(nmem)[:-1]]).astype(np.int64)
        yoff = np.concatenate([[0], np.cumsum(ny)[:-1]]).astype(np.int64)
        moff = np.concatenate([[0], np.cumsum(5 * nmem * ny)[:-1]]).astype(np.int64)
        xoff = np.concatenate([[0], np.cumsum(nmem * st.bs)[:-1]]).astype(np.int64)
        ws = _ws_total(pt.nxw, ne[0], ne[1], ne[2]).astype(np.int64)
        woff = np.concatenate([[0], np.cumsum(ws)[:-1]]).astype(np.int64)
        desc = np.zeros((n, 16), dtype=np.int32)
        desc[:, 0] = ids
        desc[:, 1:7] = pt.xbox[ids]
        desc[:, 7:13] = yb
        desc[:, 13] = nmem
        desc[:, 14] = membase
        offs = np.stack([yoff, moff, woff, xoff], axis=1).astype(np.int64)
        mflat = np.concatenate(members).astype(np.int32) if n else np.zeros(0, np.int32)
        self.mflat = mflat
        need = int(ny.max(initial=1))
        st.ensure_cap(need)
        store = st.store(pt)
        store.ensure(need)
        self.store = store
        tot_y, tot_mem = int(ny.sum()), int(nmem.sum())
        B = st.buf
        f64, i32 = torch.float64, torch.int32
        self.desc_d = torch.from_numpy(desc.ravel().copy()).to(dev)
        self.ybox_d = torch.from_numpy(yb.ravel().copy()).to(dev)
        self.offs_d = torch.from_numpy(offs.ravel().copy()).to(dev)
        self.yoff_d = torch.from_numpy(yoff.copy()).to(dev)
        self.mem_d = torch.from_numpy(mflat).to(dev) if tot_mem else B.get("mem", 1, i32)
        nxw = pt.nxw[0] * pt.nxw[1] * pt.nxw[2]
        self.alpha = B.get("alpha", n * nxw, f64)
        self.beta = B.get("beta", tot_y, f64)
        self.mdens = B.get("mdens", tot_y, f64)
        self.work = B.get("work", int(ws.sum()) + 1, f64)
        self.marena = B.get("marena", int((5 * nmem * ny).sum()), f64)
        self.xarena = B.get("xarena", tot_mem * st.bs, f64)
        self.mbox = B.get("mbox", tot_mem * 6, i32)
        self.mstat = B.get("mstat", tot_mem * 4, f64)
        self.cstat = B.get("cstat", n * 8, f64)
        self.cstat2 = B.get("cstat2", n * 8, f64)
        self.snapshot = snapshot
        self.batch = _lib.Batch3(
            n_cells=n, desc=self.desc_d.data_ptr(), offs=self.offs_d.data_ptr(),
            members=self.mem_d.data_ptr(), snapshot=snapshot.data_ptr(),
            alpha=self.alpha.data_ptr(), beta=self.beta.data_ptr(), mdens=self.mdens.data_ptr(),
            work=self.work.data_ptr(), marena=self.marena.data_ptr(),
            xarena=self.xarena.data_ptr(), mbox=self.mbox.data_ptr(), mstat=self.mstat.data_ptr(),
            cstat=self.cstat.data_ptr(), cstat2=self.cstat2.data_ptr(), delta=cfg.delta,
            max_iters=cfg.max_iters, newton_max_iters=cfg.newton_max_iters,
            newton_tol=cfg.newton_tol, trunc=cfg.trunc_threshold,
            smem_doubles=int(_hot_doubles(pt.nxw, ne[0], ne[1], ne[2]).max(initial=0)),
            precision=1 if getattr(cfg, "precision", "fp64") == "fp32" else 0)
        for a in range(3):
            self.batch.nxw[a] = pt.nxw[a]
        self.tot_y = tot_y

    def solve(self):
        _lib.check(_lib.lib().dd3_cell_solve(self.st.dp.geom, self.st.state_struct(self.store),
                                             self.batch, _lib.stream_handle()))

    def stats(self):
        c1 = self.cstat[:self.n * 8].view(self.n, 8).cpu().numpy()
        c2 = self.cstat2[:self.n * 8].view(self.n, 8).cpu().numpy()
        return c1, c2

    def commit(self, theta: np.ndarray, alpha_grid=None, yrun=None) -> np.ndarray:
        import torch

        st = self.st
        th = torch.from_numpy(np.ascontiguousarray(theta, dtype=np.float64)).to(st.dp.device)
        errs = st.buf.get("errs", self.n * 4, torch.float64)
        _lib.check(_lib.lib().dd3_cell_commit(st.dp.geom, st.state_struct(self.store), self.batch,
                                              th.data_ptr(), _lib.ptr(alpha_grid), _lib.ptr(yrun),
                                              errs.data_ptr(), _lib.stream_handle()))
        e = errs[:self.n * 4].view(self.n, 4).cpu().numpy().copy()
        if len(self.mflat):
            idx = self.mflat.astype(np.int64)
            st.ybox_h[idx] = st.ybox.view(-1, 6)[torch.from_numpy(idx).to(st.dp.device)].cpu().numpy()
        return e


class BlendScorer3:
    """Tracked energy of uniformly weighted blends of one batch (engine.py:378-456):
    per-cell scalars from ``dd3_cell_delta`` combined on the host in the reference's
    order, and the Y-side KL of clip(snapshot + theta sum dy) from ``dd3_gather``.

    Slab mode: ``batch`` holds this rank's cells of the staggered batch; ``pos`` are
    their positions in the whole batch of ``n_all`` cells.  The per-cell scalars are
    summed into the whole batch's table and sum_c theta dy_c is all-reduced, so every
    rank takes the same decision."""

    def __init__(self, plan: PlanState3, batch: _Batch3, snapshot, theta_safe: float,
                 pos=None, n_all: int | None = None):
        import torch

        self.plan, self.batch, self.snapshot = plan, batch, snapshot
        self.lam, self.eps = plan.problem.div.lam, plan.problem.eps
        t = plan.cell_terms()
        self.base_t = float(t[:, 0].sum())
        self.base_kl = float(t[:, 1].sum())
        self.base_d1 = self.lam * float(t[:, 2].sum())
        dev = plan.dp.device
        self.dy = plan.buf.get("dy", batch.tot_y, torch.float64)
        cd = plan.buf.get("cd", batch.n * 8, torch.float64)
        _lib.check(_lib.lib().dd3_cell_delta(plan.dp.geom, plan.state_struct(batch.store),
                                             batch.batch, float(theta_safe), self.dy.data_ptr(),
                                             cd.data_ptr(), _lib.stream_handle()))
        mine = cd[:batch.n * 8].view(batch.n, 8).cpu().numpy().copy()
        self.sharded = pos is not None
        if self.sharded:
            full = np.zeros((n_all, 8))
            full[pos] = mine
            mine = _shard().reduce_np(full.ravel(), "sum", dev).reshape(n_all, 8)
        self.cd = mine
        self.n_all = len(self.cd)
        self.theta_safe = float(theta_safe)
        self.dev = dev

    def opt_state(self) -> "_OptState3":
        return _OptState3(self)

    def _energy_vec(self, th) -> float:
        """energy_at of a per-cell weight vector (engine.py:441-456): per-cell pieces
        in cell order, d1 of each blended cell from ``dd3_blend_d1``, then the Y-side
        KL of clip(snapshot + sum_c theta_c dy_c)."""
        import torch

        if self.sharded:
            raise ValueError("per-cell weight vectors need the whole batch on one rank")
        b, p = self.batch, self.plan
        thd = torch.from_numpy(np.ascontiguousarray(th, dtype=np.float64)).to(self.dev)
        d1c = p.buf.get("blend_d1", max(b.n, 1), torch.float64)
        _lib.check(_lib.lib().dd3_blend_d1(p.dp.geom, p.state_struct(b.store), b.batch,
                                           thd.data_ptr(), d1c.data_ptr(), _lib.stream_handle()))
        d1n = d1c[:b.n].cpu().numpy()
        t, kl, d1 = self.base_t, self.base_kl, self.base_d1
        for c in range(self.n_all):
            tc = float(th[c])
            if tc:
                t += tc * self.cd[c, 0]
                kl += tc * self.cd[c, 1]
                d1 += float(d1n[c]) - self.cd[c, 2]
        y = p.buf.get("blend_y", p.dp.ny, torch.float64)
        part = p._partial(y)
        npart = ctypes.c_int(0)
        _lib.check(_lib.lib().dd3_gather(
            p.dp.geom, b.n, b.ybox_d.data_ptr(), 6, self.dy.data_ptr(), 0,
            b.yoff_d.data_ptr(), thd.data_ptr(), self.snapshot.data_ptr(), y.data_ptr(), 2,
            p.dp.nu.data_ptr(), part.data_ptr(), ctypes.byref(npart), _lib.stream_handle()))
        d2 = self.lam * float(part[:npart.value].sum().item())
        return t + self.eps * kl + d1 + d2

    def energy_at(self, theta) -> float:
        import torch

        if np.ndim(theta) == 1:
            return self._energy_vec(np.asarray(theta, dtype=np.float64))
        b, p = self.batch, self.plan
        t, kl, d1 = self.base_t, self.base_kl, self.base_d1
        th = float(theta)
        if th:
            col = 3 if th == 1.0 else 4
            if th not in (1.0, self.theta_safe):
                raise ValueError("BlendScorer3 evaluates theta in {0, 1, theta_safe}")
            for c in range(self.n_all):
                t += th * self.cd[c, 0]
                kl += th * self.cd[c, 1]
                d1 += self.cd[c, col] - self.cd[c, 2]
        scale = torch.full((max(b.n, 1),), th, dtype=torch.float64, device=self.dev)
        y = p.buf.get("blend_y", p.dp.ny, torch.float64)
        if not self.sharded:
            part = p._partial(y)
            npart = ctypes.c_int(0)
            _lib.check(_lib.lib().dd3_gather(
                p.dp.geom, b.n, b.ybox_d.data_ptr(), 6, self.dy.data_ptr(), 0,
                b.yoff_d.data_ptr(), scale.data_ptr(), self.snapshot.data_ptr(), y.data_ptr(), 2,
                p.dp.nu.data_ptr(), part.data_ptr(), ctypes.byref(npart), _lib.stream_handle()))
            d2 = self.lam * float(part[:npart.value].sum().item())
        else:
            # rank-local sum_c theta dy_c, all-reduced, then KL(clip(snapshot + sum))
            _lib.check(_lib.lib().dd3_gather(
                p.dp.geom, b.n, b.ybox_d.data_ptr(), 6, self.dy.data_ptr(), 0,
                b.yoff_d.data_ptr(), scale.data_ptr(), None, y.data_ptr(), 0, None, None, None,
                _lib.stream_handle()))
            _shard().all_reduce(y[:p.dp.ny])
            d2 = self.lam * p.grid_kl(y, clip=True, base=self.snapshot)
        return t + self.eps * kl + d1 + d2


class _OptState3:
    """Incremental blend view for coordinate descent on the three-axis path
    (BlendScorer.set_theta / minimize_coordinate, engine.py:458-470), on the device."""

    def __init__(self, scorer: BlendScorer3):
        import torch

        self.sc = scorer
        p = scorer.plan
        ny = p.dp.ny
        self.ycur = p.buf.get("opt_ycur", ny, torch.float64)
        self.ycur[:ny].copy_(scorer.snapshot[:ny])
        self.out = p.buf.get("opt_out", 4, torch.float64)
        self.lin = scorer.cd[:, 0] + scorer.eps * scorer.cd[:, 1]
        self.theta = np.zeros(scorer.n_all)

    def set_theta(self, i: int, th: float) -> None:
        sc = self.sc
        dth = th - self.theta[i]
        if dth:
            _lib.check(_lib.lib().dd3_opt_set(sc.plan.dp.geom, sc.batch.batch, sc.dy.data_ptr(),
                                              int(i), float(dth), self.ycur.data_ptr(),
                                              _lib.stream_handle()))
        self.theta[i] = th

    def minimize_coordinate(self, i: int, tol: float) -> float:
        from .engine import _coordinate_root

        sc = self.sc
        p, b = sc.plan, sc.batch
        lam = sc.lam
        lin = float(self.lin[i])
        th_cur = float(self.theta[i])
        sstruct = p.state_struct(b.store)

        def gh(th):
            _lib.check(_lib.lib().dd3_opt_gh(p.dp.geom, sstruct, b.batch, sc.dy.data_ptr(), int(i),
                                             float(th), th_cur, self.ycur.data_ptr(),
                                             self.out.data_ptr(), _lib.stream_handle()))
            o = self.out[:4].cpu().numpy()
            with np.errstate(invalid="ignore"):
                g = lin + lam * float(o[0]) + lam * float(o[2])
                h = lam * float(o[1]) + lam * float(o[3])
            return g, h

        return _coordinate_root(gh, tol)


# -- iterations ---------------------------------------------------------------------------

def _absorb(stats, batch: _Batch3) -> None:
    c1, c2 = batch.stats()
    w = batch.pt.nxw
    n = [batch.ybox[:, 2 * a + 1].astype(np.float64) for a in range(3)]
    fl = cell_lse_flops3(w, n[0], n[1], n[2])
    sums = np.array([(c2[:, 2] * fl).sum(), c1[:, 1].sum(), c1[:, 6].sum(), c1[:, 4].sum(),
                     (c1[:, 3] == 0).sum(), c2[:, 0].sum(), c1[:, 2].sum(), c2[:, 3].sum()],
                    dtype=np.float64)
    maxs = np.array([c1[:, 5].max(initial=0), c1[:, 7].max(initial=0.0)], dtype=np.float64)
    sh = _shard()
    if sh is not None:
        sums = sh.reduce_np(sums, "sum", batch.st.dp.device)
        maxs = sh.reduce_np(maxs, "max", batch.st.dp.device)
    stats.cell_flops += float(sums[0])
    stats.entry_gap += float(sums[1])
    stats.balance_fallbacks += int(sums[2])
    stats.nu_minus_clamped += int(sums[3])
    stats.nonconverged_cells += int(sums[4])
    stats.nu_j_drift_nodes += int(sums[5])
    stats.cell_iterations += int(sums[6])
    stats.sweep_fallbacks = getattr(stats, "sweep_fallbacks", 0) + int(sums[7])
    stats.newton_clamped = max(stats.newton_clamped, int(maxs[0]))
    stats.balance_target_miss = max(stats.balance_target_miss, float(maxs[1]))


def cell_lse_flops3(w, n0, n1, n2):
    """Algorithmic FLOPs of one Sinkhorn iteration of a three-axis cell: the six
    separable contractions (2 per FMA) of the X and Y sweeps."""
    w0, w1, w2 = (float(x) for x in w)
    y_sweep = w0 * w1 * w2 * n2 + w0 * w1 * n2 * n1 + w0 * n1 * n2 * n0
    x_sweep = n0 * n1 * n2 * w2 + n0 * n1 * w2 * w1 + n0 * w1 * w2 * w0
    return 2.0 * (y_sweep + x_sweep)


def iteration_sequential3(plan: PlanState3, part: CompositePartition, config, stats):
    """Cell-by-cell pass in lattice row-major order on a running Y-marginal, each
    cell committed at theta = 1 before the next is set up (engine.py:799-836).
    The running marginal is updated on the device by the commit kernel."""
    import torch

    if _shard() is not None:
        raise ValueError("the sequential sweep is inherently serial; run it on one rank")
    cfg = config.cell_config()
    pt = _tables(part)
    if stats.alpha is None:
        stats.alpha = torch.zeros(plan.dp.nx, dtype=torch.float64, device=plan.dp.device)
    t0 = time.perf_counter()
    y_run = plan.assemble_device(plan.buf.get("yrun", plan.dp.ny, torch.float64))
    stats.assemble_time += time.perf_counter() - t0
    for j in range(pt.ncomp):
        t0 = time.perf_counter()
        bt = _Batch3(plan, pt, np.array([j], dtype=np.int64), y_run, cfg)
        bt.solve()
        _absorb(stats, bt)
        stats.solve_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        e = bt.commit(np.ones(1), stats.alpha, y_run)
        stats.commit_time += time.perf_counter() - t0
        stats.x_err += float(e[0, 0])
        stats.y_err += float(e[0, 1])
        plan.truncated_mass += float(e[0, 2])
        stats.truncated_mass += float(e[0, 2])
    stats.action = "sequential"
    return plan


def iteration_parallel3(plan: PlanState3, part: CompositePartition, strategy, config, stats):
    """Snapshot, batch solve, weighted commit (engine.py:839-922), on the device.

    Slab mode (``engine.set_shard``): every rank solves and commits the composites
    of its slab (slabs of the first real axis, z for 3D); the boundary layer's basic
    cells move to their new owner before each partition sweep (halo exchange); the
    snapshot, the blend energies, the residuals and the stitched alpha are reduced
    over the ranks (slab.py)."""
    import torch

    if strategy.kind not in STRATEGIES_3D:
        raise NotImplementedError(f"the three-axis path runs strategies {STRATEGIES_3D}, "
                                  f"not {strategy.kind!r}")
    cfg = config.cell_config()
    pt = _tables(part)
    batches = pt.batches if strategy.kind == "staggered" else [np.arange(pt.ncomp)]
    if stats.alpha is None:
        stats.alpha = torch.zeros(plan.dp.nx, dtype=torch.float64, device=plan.dp.device)
    sh = _shard()
    comp_owner = None
    if sh is not None:
        comp_owner, basic_owner = _slab_layout3(plan, pt)
        sh.halo_exchange(plan, basic_owner)
        plan.comp_owner[pt.label] = comp_owner
    actions = []
    for batch in batches:
        batch = np.asarray(batch, dtype=np.int64)
        t0 = time.perf_counter()
        snapshot = plan.assemble_device(plan.buf.get("snapshot", plan.dp.ny, torch.float64))
        stats.assemble_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        pos = None
        ids = batch
        if sh is not None:
            pos = np.flatnonzero(comp_owner[batch] == sh.rank)
            ids = batch[pos]
        bt = _Batch3(plan, pt, ids, snapshot, cfg)
        bt.solve()
        _absorb(stats, bt)
        stats.solve_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        kb = len(batch)
        if strategy.kind == "fast":
            th = 1.0
            actions.append("greedy")
        elif strategy.kind == "safe":
            th = 1.0 / kb
            actions.append("safe")
        elif strategy.kind == "swift":
            # better of greedy (ones) and safe (1/K), ties to greedy (engine.py:543-554)
            scorer = BlendScorer3(plan, bt, snapshot, 1.0 / kb, pos, kb)
            greedy = scorer.energy_at(1.0) <= scorer.energy_at(1.0 / kb)
            th = 1.0 if greedy else 1.0 / kb
            actions.append("greedy" if greedy else "safe")
        elif strategy.kind == "opt":
            # cyclic coordinate descent on per-cell weights (engine.py:557-588)
            if sh is not None:
                raise ValueError("the opt strategy needs per-cell global coordination inside a "
                                 "batch; slab-sharded solves support safe, fast, swift and "
                                 "staggered")
            from .engine import get_weights_opt
            scorer = BlendScorer3(plan, bt, snapshot, 1.0 / kb)
            w = get_weights_opt(None, list(range(kb)), part, scorer, strategy.opt_max_sweeps,
                                strategy.opt_tol).theta
            th = np.array([w[c] for c in range(kb)])
            actions.append("opt")
        else:
            scorer = BlendScorer3(plan, bt, snapshot, 1.0 / kb, pos, kb)
            e_base = scorer.energy_at(0.0)
            e_greedy = scorer.energy_at(1.0)
            e_safe = scorer.energy_at(1.0 / kb)
            allowance = strategy.leniency * max(0.0, e_base - e_safe)
            if e_greedy <= e_base + allowance:
                th = 1.0
                actions.append("greedy")
            else:
                th = 1.0 / kb
                actions.append("safe-fallback")
                stats.safe_fallbacks += 1
        stats.score_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        e = bt.commit(th if np.ndim(th) == 1 else np.full(bt.n, th), stats.alpha)
        es = e[:, :3].sum(axis=0)
        if sh is not None:
            es = sh.reduce_np(es, "sum", plan.dp.device)
        stats.x_err += float(es[0])
        stats.y_err += float(es[1])
        plan.truncated_mass += float(es[2])
        stats.truncated_mass += float(es[2])
        stats.commit_time += time.perf_counter() - t0
    if sh is not None:
        sh.all_reduce(stats.alpha)   # each rank stitched its own composites' blocks
    if len(actions) == 1:
        stats.action = actions[0]
    else:
        n_fb = actions.count("safe-fallback")
        stats.action = "greedy" if n_fb == 0 else f"safe-fallback({n_fb}/{len(actions)})"
    return plan


def domdec_solve3(problem: TransportProblem, partitions: Decomposition, strategy=None,
                  config=None, state: PlanState3 | None = None, evaluator=None,
                  dp: VolumeProblem | None = None):
    """Alternate composite partitions until the certificate falls below
    lam * delta * |mu| (engine.py:938-1037); returns (PlanState3, SolveReport)."""
    from .engine import EngineConfig, IterationStats, StitchedGapEvaluator, StrategyConfig, \
        _score_dict

    strategy = strategy if strategy is not None else StrategyConfig()
    config = config if config is not None else EngineConfig()
    if state is None:
        state = initial_plan_state3(problem, partitions.basic, dp)
    lam = problem.div.lam
    mu_total = problem.mu.total_mass
    ev = evaluator if evaluator is not None else StitchedGapEvaluator(problem, dp=state.dp)
    if state.global_duals is not None:
        ev.seed(*state.global_duals)
    check_every = max(1, config.gap_check_every)
    trace = []
    timings = {"assemble": 0.0, "solve": 0.0, "score": 0.0, "commit": 0.0, "total": 0.0}
    diag = {"balance_fallbacks": 0, "safe_fallbacks": 0, "nonconverged_cells": 0,
            "newton_clamped": 0, "nu_minus_clamped": 0, "balance_target_miss": 0.0,
            "nu_j_drift_nodes": 0, "cell_iterations": 0, "cell_flops": 0.0,
            "sweep_fallbacks": 0, "strategy": strategy.kind, "leniency": strategy.leniency,
            "delta": config.delta}
    converged = False
    last_gap = float("inf")
    stats = IterationStats()
    sb = state.energy()
    t_all = time.perf_counter()
    for k in range(1, config.max_iters + 1):
        part = partitions.composites[(k - 1) % len(partitions.composites)]
        stats = IterationStats(k=k, label=part.label)
        t0 = time.perf_counter()
        if strategy.kind == "sequential":
            iteration_sequential3(state, part, config, stats)
        else:
            iteration_parallel3(state, part, strategy, config, stats)
        sb = state.energy()
        if k % check_every == 0 or k == config.max_iters:
            t1 = time.perf_counter()
            stats.gap = ev.evaluate(stats.alpha, sb.total)
            stats.score_time += time.perf_counter() - t1
            last_gap = stats.gap
        wall = time.perf_counter() - t0
        trace.append(TraceRow(k=k, label=part.label, action=stats.action,
                              transport=sb.transport, entropy=sb.entropy, d1=sb.d1, d2=sb.d2,
                              total=sb.total, gap=stats.gap, x_err=stats.x_err, y_err=stats.y_err,
                              wall_time=wall))
        for key in ("assemble", "solve", "score", "commit"):
            timings[key] += getattr(stats, f"{key}_time")
        for key in ("balance_fallbacks", "safe_fallbacks", "nonconverged_cells",
                    "nu_minus_clamped", "nu_j_drift_nodes"):
            diag[key] += getattr(stats, key)
        diag["sweep_fallbacks"] += getattr(stats, "sweep_fallbacks", 0)
        diag["cell_iterations"] += stats.cell_iterations
        diag["cell_flops"] += stats.cell_flops
        diag["newton_clamped"] = max(diag["newton_clamped"], stats.newton_clamped)
        diag["balance_target_miss"] = max(diag["balance_target_miss"], stats.balance_target_miss)
        if last_gap / lam <= config.delta * mu_total:
            converged = True
            break
    if _shard() is not None:
        _shard().replicate(state)     # the whole plan current on every rank again
    timings["total"] = time.perf_counter() - t_all
    diag["truncated_mass"] = state.truncated_mass
    report = SolveReport(converged=converged, iterations=len(trace), final_score=_score_dict(sb),
                         rel_pd_gap=last_gap / max(abs(sb.total), 1e-300), x_err=stats.x_err,
                         y_err=stats.y_err, trace=trace, timings=timings,
                         sparsity=state.sparsity(), diagnostics=diag)
    return state, report


# -- coarse-to-fine (SPEC multiscale_solve, paper section 4.3.1) --------------------------

def prolong_duals3(duals, coarse: VolumeProblem, fine: VolumeProblem):
    """Trilinear prolongation of an (alpha, beta) pair to the next finer layer."""
    ca, cb = duals
    fa, fb = fine.empty_x(), fine.empty_y()
    L = _lib.lib()
    _lib.check(L.dd3_prolong(_i32(fine.shape_x), _i32(coarse.shape_x), ca.data_ptr(),
                             fa.data_ptr(), _lib.stream_handle()))
    _lib.check(L.dd3_prolong(_i32(fine.shape_y), _i32(coarse.shape_y), cb.data_ptr(),
                             fb.data_ptr(), _lib.stream_handle()))
    return fa, fb


def multiscale_solve3(problem: TransportProblem, cell_size: int, n_coarsest: int,
                      eps_start: float, eps_final: float | None = None, strategy=None,
                      config=None, progress=None, levels: list | None = None,
                      switch: int | None = None, global_delta: float | None = None,
                      global_max_iters: int = 100_000, switch_iters: int = 20_000):
    """SPEC ``multiscale_solve`` on the three-axis path: global unbalanced Sinkhorn at
    delta/4 on every layer below the switch layer (duals prolonged trilinearly; the
    coarsest starts from the mass-balanced constant pair), ``warm_start_plan3`` at the
    switch layer, domdec (staggered) from there on.  For N < 512 the switch layer is
    the finest (SPEC: l_switch = log2 N - 1), which is every BASELINE 3D case; plan
    refinement between domdec layers is not needed there and not provided."""
    from .engine import EngineConfig, StitchedGapEvaluator, StrategyConfig
    from .multiscale import (MultiscaleReport, _global_report, build_pyramid, layer_index,
                             spec_eps_schedule, switch_layer)

    strategy = strategy if strategy is not None else StrategyConfig()
    config = config if config is not None else EngineConfig()
    t_all = time.perf_counter()
    eps_final = problem.eps if eps_final is None else eps_final
    if levels is None:
        levels = build_pyramid(problem.mu, problem.nu, n_coarsest)
    n_fine = max(levels[-1].grid.dims)
    lsw = switch_layer(n_fine) if switch is None else int(switch)
    sched = spec_eps_schedule(levels, eps_start, eps_final)
    gdelta = config.delta / 4.0 if global_delta is None else float(global_delta)
    rep = MultiscaleReport(converged=True)
    state = None
    duals, dprev = None, None
    timings = {"global": 0.0, "warm": 0.0, "refine": 0.0, "domdec": 0.0}
    for li, lv in enumerate(levels):
        eps_list = sched[li]
        prob = TransportProblem(GridMeasure(lv.grid, lv.mu), GridMeasure(lv.grid, lv.nu),
                                problem.div, eps_list[0])
        dp = lv.dp if isinstance(lv.dp, VolumeProblem) else VolumeProblem(prob)
        lv.dp = dp
        dp.problem = prob
        dp.set_eps(eps_list[0])
        if layer_index(max(lv.grid.dims)) < lsw and li < len(levels) - 1:
            if duals is not None:
                a0, b0 = prolong_duals3(duals, dprev, dp)
            else:
                a0, b0 = mass_balanced_start(dp)
            for eps in eps_list:
                dp.problem = TransportProblem(prob.mu, prob.nu, problem.div, eps)
                dp.set_eps(eps)
                t0 = time.perf_counter()
                res = sinkhorn_solve(dp, a0, b0, SolverConfig(delta=gdelta,
                                                              max_iters=global_max_iters))
                t = time.perf_counter() - t0
                timings["global"] += t
                a0, b0 = res.alpha, res.beta
                r = _global_report(res, eps, t, gdelta)
                rep.stages.append((lv.grid.dims[0], eps, r))
                rep.converged = rep.converged and r.converged
                if progress is not None:
                    progress(lv.grid.dims[0], eps, r)
            duals, dprev = (a0, b0), dp
            continue
        if state is not None:
            raise NotImplementedError("the three-axis path runs domdec on the finest layer only "
                                      "(switch layer = finest, SPEC for N < 512)")
        dec = lv.decs.get(cell_size)
        if dec is None:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                dec = make_decomposition(prob.mu, cell_size)
            lv.decs[cell_size] = dec
        t0 = time.perf_counter()
        a0 = b0 = None
        if duals is not None:
            a0, b0 = prolong_duals3(duals, dprev, dp)
        state = warm_start_plan3(prob, dec, delta=gdelta, max_iters=switch_iters, dp=dp,
                                 alpha0=a0, beta0=b0)
        timings["warm"] += time.perf_counter() - t0
        timings.update({f"warm_{k}": v for k, v in getattr(state, "warm_timing", {}).items()})
        for eps in eps_list:
            prob = TransportProblem(prob.mu, prob.nu, problem.div, eps)
            state.problem = prob
            dp.problem = prob
            dp.set_eps(eps)
            ev = StitchedGapEvaluator(prob, dp=dp)
            t0 = time.perf_counter()
            state, r = domdec_solve3(prob, dec, strategy, config, state=state, evaluator=ev)
            timings["domdec"] += time.perf_counter() - t0
            if ev._best is not None:
                state.global_duals = (ev._best[0], ev._best[1])
            rep.stages.append((lv.grid.dims[0], eps, r))
            rep.total_iterations += r.iterations
            rep.converged = rep.converged and r.converged
            rep.final_score = r.final_score
            rep.rel_pd_gap = r.rel_pd_gap
            if progress is not None:
                progress(lv.grid.dims[0], eps, r)
        duals, dprev = state.global_duals, dp
    timings["total"] = time.perf_counter() - t_all
    rep.timings = timings
    return state, rep
