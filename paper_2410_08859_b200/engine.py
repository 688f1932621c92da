"""Domain-decomposition driver on the device: plan state, strategies, stopping.

Mirror of the reference solver API (``domdec.engine``: StrategyConfig :94,
WeightAssignment :110, EngineConfig :122, Decomposition/make_decomposition
:139-150, PlanState :157, initial_plan_state :234, warm_start_plan :260,
BlendScorer :378, get_weights_safe/swift/opt :533-588, StitchedGapEvaluator
:594, iteration_sequential :799, iteration_parallel :839, domdec_solve :938;
``domdec.cells``: CellSolverConfig :63, make_cell_problems + solve_cell_batch
:165-393).  The algorithm is the reference's; the data path is B200-native:

* the iterate lives in HBM — per-basic-cell Y-marginal boxes and values in
  fixed-capacity slots, dense per-block X-marginals, score fragments and the
  per-partition dual store;
* one batch of composite cells is one ``dd_cell_solve`` launch (a CTA per
  cell: window assembly, Sinkhorn to tolerance, split, balancing,
  truncation, fragments), followed by ``dd_cell_delta`` / ``dd_blend_energy``
  for the weight strategy and ``dd_cell_commit``;
* the stopping certificate runs full-grid separable sweeps (``dd_grid_lse``).

The host keeps only control flow, the box mirror used to size the next
batch's windows, and scalars for traces.  There is no CPU compute path: a
missing library or device raises.
"""

from __future__ import annotations

import logging
import time
import warnings
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .decomposition import (BasicPartition, CompositePartition, Decomposition, as2d_box,
                            make_decomposition)
from .grids import GridMeasure, SparseCellMarginal, TransportProblem
from .report import SolveReport, TraceRow
from .sinkhorn import (DeviceProblem, GridSweeper, SolverConfig, axpb, dual_sums,
                       sinkhorn_solve)
from .slab import ShardSpec

log = logging.getLogger(__name__)

__all__ = [
    "STRATEGY_KINDS", "StrategyConfig", "WeightAssignment", "CellSolverConfig", "EngineConfig",
    "Decomposition", "make_decomposition", "ScoreBreakdown", "CellDuals", "PlanState",
    "initial_plan_state", "warm_start_plan", "BlendScorer", "get_weights_safe",
    "get_weights_swift", "get_weights_opt", "StitchedGapEvaluator", "IterationStats",
    "iteration_sequential", "iteration_parallel", "domdec_solve", "ShardSpec", "set_shard",
    "clear_shard", "ExecMode", "set_exec_mode", "get_exec_mode",
]

STRATEGY_KINDS = ("sequential", "safe", "fast", "swift", "opt", "staggered")
import os as _os

# dynamic shared memory budget per CTA: 227 KB opt-in on sm_100a minus the solve
# kernel's ~3 KB of static shared memory, split over the CTAs the build keeps
# resident per SM (dd_cell_min_blocks; queried lazily, so importing the package
# maps no library).
CLUSTER_SIZES = (2, 4, 8, 16)
_OCC_CACHE: list = []


def _occupancy() -> int:
    if not _OCC_CACHE:
        _OCC_CACHE.append(int(_lib.lib().dd_cell_min_blocks()))
    return _OCC_CACHE[0]


_SM_COUNT: dict = {}


def _sm_count(device) -> int:
    import torch

    key = str(device)
    if key not in _SM_COUNT:
        _SM_COUNT[key] = int(torch.cuda.get_device_properties(device).multi_processor_count)
    return _SM_COUNT[key]


def _smem_budget() -> int:
    occ = _occupancy()
    return (220 * 1024) // occ - 1024 * (occ - 1)


@dataclass
class ExecMode:
    """Which execution path the cell solves take (runtime-settable; tests cover each).

    ``force_cluster=C`` runs every cell's Sinkhorn loop on a C-CTA thread-block
    cluster; ``force_global_ws`` puts every cell's workspace in the global arena
    (single-CTA kernel); ``no_cluster`` keeps large cells on the single-CTA
    global-workspace path; ``smem_budget`` lowers the per-CTA shared-memory budget
    the size rule uses, so mid-size windows take the cluster path by the same
    rule large windows do.  Defaults come from DD_FORCE_CLUSTER /
    DD_FORCE_GLOBAL_WS / DD_NO_CLUSTER."""

    force_cluster: int = 0
    force_global_ws: bool = False
    no_cluster: bool = False
    skip_stagnant: bool = True
    smem_budget: int = 0        # bytes per CTA for the size rule (0: the hardware budget)
    # 2-CTA clusters for the few cells expected at the cap (latency).  Off by default:
    # on ms_1024's 512^2 layer it changed the trajectory (the eps = 4h^2 stage stopped
    # converging in one sweep and its windows grew) although every golden case
    # passes through the cluster path; DD_CLUSTER_CAPPED=1 turns it on
    cluster_capped: bool = False
    # throughput-bound batches (many cells): shared-memory cells run their Sinkhorn loop
    # in a separate kernel at two CTAs per SM (<= 64 registers) and the epilogue after
    # measured slower on ms_1024's 1024^2 stage (2.98 -> 3.78 s: 64 registers spill and
    # a capped cell's latency grows), so opt-in (DD_SPLIT=1); parity-tested either way
    split_loop: bool = False
    force_split: bool = False   # split every fitting shared-memory cell (tests)


def _env_mode() -> ExecMode:
    return ExecMode(force_cluster=int(_os.environ.get("DD_FORCE_CLUSTER", "0") or 0),
                    force_global_ws=_os.environ.get("DD_FORCE_GLOBAL_WS") == "1",
                    no_cluster=_os.environ.get("DD_NO_CLUSTER") == "1",
                    skip_stagnant=_os.environ.get("DD_NO_SKIP") != "1",
                    cluster_capped=_os.environ.get("DD_CLUSTER_CAPPED") == "1",
                    split_loop=_os.environ.get("DD_SPLIT") == "1")


_MODE = [_env_mode()]


def set_exec_mode(mode: ExecMode | None = None, **kw) -> ExecMode:
    """Set the cell-solve execution path; returns the previous mode."""
    prev = _MODE[0]
    _MODE[0] = mode if mode is not None else ExecMode(**kw)
    return prev


def get_exec_mode() -> ExecMode:
    return _MODE[0]


def _cluster_ws(nw0: int, nw1: int, ny0: np.ndarray, ny1: np.ndarray, C: int) -> np.ndarray:
    """dd_cell_cluster_ws, vectorized (mirrors clu_layout in csrc/cell.cu)."""
    nx = nw0 * nw1
    rows = (ny0 + C - 1) // C + 1
    nyl = rows * ny1
    wsz = np.maximum(np.maximum(np.maximum(nw1 * ny0, ny1 * nw0), nx), nyl)
    rm = np.maximum(np.maximum(ny0, ny1), max(nw0, nw1))
    return (nw0 + nw1 + ny0 + ny1 + 6 * nx + 3 * nyl + nw0 * ny0 + nw1 * ny1 + rows * nw1
            + 2 * nx + nw0 * ny1 + wsz + nw1 * ny0 + rm)
MAX_MEMBERS = 64


@dataclass(frozen=True)
class StrategyConfig:
    kind: str = "staggered"
    leniency: float = 0.005
    opt_max_sweeps: int = 50
    opt_tol: float = 1e-9

    def __post_init__(self):
        if self.kind not in STRATEGY_KINDS:
            raise ValueError(f"unknown strategy {self.kind!r}; pick one of {STRATEGY_KINDS}")
        if self.leniency < 0:
            raise ValueError("leniency must be nonnegative")


@dataclass(frozen=True)
class WeightAssignment:
    theta: dict

    def __post_init__(self):
        for j, t in self.theta.items():
            if not 0.0 <= t <= 1.0:
                raise ValueError(f"weight {t!r} for cell {j} is outside [0, 1]")


@dataclass(frozen=True)
class CellSolverConfig:
    delta: float = 2e-5
    max_iters: int = 10_000
    newton_tol: float = 1e-12
    newton_max_iters: int = 100
    trunc_threshold: float = 1e-15
    chunk_entries: int = 4_000_000  # kept for API parity; batches are not chunked on device
    # "fp64" (reference arithmetic) or "fp32" (north_star fp32 mode: the cell sweeps'
    # tables, weights and contractions in fp32; potentials, Newton, gap, epilogue fp64)
    precision: str = "fp64"

    def __post_init__(self):
        if self.precision not in ("fp64", "fp32"):
            raise ValueError(f"precision must be 'fp64' or 'fp32', not {self.precision!r}")


@dataclass(frozen=True)
class EngineConfig:
    delta: float = 2e-5
    max_iters: int = 2000
    gap_check_every: int = 1
    cell_delta_factor: float = 0.25
    cell: CellSolverConfig = CellSolverConfig()

    def cell_config(self) -> CellSolverConfig:
        return replace(self.cell, delta=self.delta * self.cell_delta_factor)


@dataclass(frozen=True)
class ScoreBreakdown:
    transport: float
    entropy: float
    d1: float
    d2: float

    @property
    def total(self) -> float:
        return self.transport + self.entropy + self.d1 + self.d2


@dataclass
class CellDuals:
    alpha: np.ndarray
    beta_box: tuple
    beta: np.ndarray


# -- device tables ------------------------------------------------------------------

def _box4(box) -> list:
    return [c for ax in as2d_box(box) for c in ax]


def _box_from4(b4, ndim: int) -> tuple:
    b = tuple(int(x) for x in b4)
    if b[1] == 0 or b[3] == 0:
        return ((0, 0),) * ndim
    return ((b[2], b[3]),) if ndim == 1 else ((b[0], b[1]), (b[2], b[3]))


class _PartTables:
    """Integer tables of one composite partition (2D embedding)."""

    def __init__(self, part: CompositePartition):
        import torch  # noqa: F401

        self.part = part
        self.label = part.label
        self.ncomp = part.n_cells
        self.xbox = np.array([_box4(b) for b in part.boxes], dtype=np.int32).reshape(-1, 4)
        self.nw0 = int(self.xbox[0, 1])
        self.nw1 = int(self.xbox[0, 3])
        if np.any(self.xbox[:, 1] != self.nw0) or np.any(self.xbox[:, 3] != self.nw1):
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


class _DualStore:
    """Warm-start duals of one partition: alpha per cell, boxed beta per cell."""

    def __init__(self, ncomp: int, nx: int, dcap: int, device):
        import torch

        self.ncomp, self.nx = ncomp, nx
        self.alpha = torch.zeros(ncomp * nx, dtype=torch.float64, device=device)
        self.has = torch.zeros(ncomp, dtype=torch.int32, device=device)
        self.box = torch.zeros(ncomp * 4, dtype=torch.int32, device=device)
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
        c = object.__new__(_DualStore)
        c.ncomp, c.nx, c.dcap = self.ncomp, self.nx, self.dcap
        c.alpha, c.has, c.box, c.beta = (self.alpha.clone(), self.has.clone(), self.box.clone(),
                                         self.beta.clone())
        return c


class _Buffers:
    """Grow-only device scratch buffers, keyed by name."""

    def __init__(self, device):
        self.device = device
        self.bufs = {}

    def get(self, name: str, n: int, dtype):
        import torch

        n = max(1, int(n))
        t = self.bufs.get(name)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.empty(int(n * 1.25) + 16, dtype=dtype, device=self.device)
            self.bufs[name] = t
        return t


# -- the iterate ----------------------------------------------------------------------

class PlanState:
    """Device-resident iterate: per-basic-cell boxed Y-marginals, X-marginals,
    fragments and cell duals (engine.py:157-216).  ``nu_i``, ``x_marg``,
    ``transport``, ``kl`` and ``duals`` download on access."""

    def __init__(self, problem: TransportProblem, basic: BasicPartition, dp: DeviceProblem = None,
                 cap: int = 1):
        import torch

        self.problem = problem
        self.basic = basic
        self.dp = dp if dp is not None else DeviceProblem(problem)
        dev = self.dp.device
        self.ndim = problem.mu.grid.ndim
        nb = basic.n_cells
        self.n_basic = nb
        bx = np.array([_box4(b) for b in basic.cell_boxes], dtype=np.int32).reshape(-1, 4)
        self.block = (int(bx[0, 1]), int(bx[0, 3]))
        self.bs = self.block[0] * self.block[1]
        self.basic_xbox = torch.from_numpy(bx.ravel().copy()).to(dev)
        self.basic_mass = torch.from_numpy(np.asarray(basic.masses, dtype=np.float64)).to(dev)
        self.cap = int(max(1, cap))
        self.ybox = torch.zeros(nb * 4, dtype=torch.int32, device=dev)
        self.yval = torch.zeros(nb * self.cap, dtype=torch.float64, device=dev)
        self.ybox_h = np.zeros((nb, 4), dtype=np.int32)
        self.x_marg_d = torch.zeros(nb * self.bs, dtype=torch.float64, device=dev)
        self.transport_d = torch.zeros(nb, dtype=torch.float64, device=dev)
        self.kl_d = torch.zeros(nb, dtype=torch.float64, device=dev)
        self.stores: dict = {}
        self.truncated_mass = 0.0
        self.global_duals = None
        self.iter_hist: dict = {}   # partition label -> executed iterations of the last solve
        # slab mode: owning rank of each basic cell (None: every cell current here)
        self.owner = None
        self._mask_d = None
        self.comp_owner: dict = {}  # slab mode: partition label -> owner of each composite
        self.buf = _Buffers(dev)
        self.partial = torch.empty(8192 + 4 * nb, dtype=torch.float64, device=dev)
        self.sums = torch.zeros(8, dtype=torch.float64, device=dev)

    # ---- C structs
    def state_struct(self, store: _DualStore | None = None) -> _lib.State:
        dp = self.dp
        s = _lib.State(mu=dp.mu.data_ptr(), nu=dp.nu.data_ptr(), log_mu=dp.log_mu.data_ptr(),
                       log_nu=dp.log_nu.data_ptr(), n_basic=self.n_basic, block0=self.block[0],
                       block1=self.block[1], basic_xbox=self.basic_xbox.data_ptr(),
                       basic_mass=self.basic_mass.data_ptr(), ybox=self.ybox.data_ptr(),
                       yval=self.yval.data_ptr(), cap=self.cap, x_marg=self.x_marg_d.data_ptr(),
                       transport=self.transport_d.data_ptr(), kl=self.kl_d.data_ptr())
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

    def store(self, pt: _PartTables) -> _DualStore:
        st = self.stores.get(pt.label)
        if st is None:
            st = _DualStore(pt.ncomp, pt.nw0 * pt.nw1, 1, self.dp.device)
            self.stores[pt.label] = st
        return st

    def sync_boxes(self):
        self.ybox_h = self.ybox.view(-1, 4).cpu().numpy().copy()

    def set_owner(self, owner) -> None:
        """Slab mode: the owning rank of every basic cell (None: all current here)."""
        import torch

        self.owner = None if owner is None else np.asarray(owner, dtype=np.int64).copy()
        if self.owner is None or _SHARD is None:
            self._mask_d = None
        else:
            m = (self.owner == _SHARD.rank).astype(np.float64)
            self._mask_d = torch.from_numpy(m).to(self.dp.device)

    def _sharded(self) -> bool:
        return _SHARD is not None and _SHARD.world > 1 and self._mask_d is not None

    # ---- energy
    def assemble_device(self, out=None):
        out = out if out is not None else self.dp.empty_y()
        if self._sharded():
            # own basic cells, then one dense all-reduce over the slabs
            _lib.check(_lib.lib().dd_assemble_masked(self.dp.geom, self.state_struct(),
                                                     self._mask_d.data_ptr(), out.data_ptr(),
                                                     _lib.stream_handle()))
            _SHARD.all_reduce(out[:self.dp.ny])
            return out
        _lib.check(_lib.lib().dd_assemble(self.dp.geom, self.state_struct(), out.data_ptr(),
                                          _lib.stream_handle()))
        return out

    def energy_terms(self, y) -> np.ndarray:
        if self._sharded():
            _lib.check(_lib.lib().dd_energy_terms_masked(
                self.dp.geom, self.state_struct(), y.data_ptr(), self._mask_d.data_ptr(),
                self.partial.data_ptr(), self.sums.data_ptr(), _lib.stream_handle()))
            _SHARD.all_reduce(self.sums[:3])    # per-cell sums; sums[3] is KL of the global y
            return self.sums[:4].cpu().numpy().copy()
        _lib.check(_lib.lib().dd_energy_terms(self.dp.geom, self.state_struct(), y.data_ptr(),
                                              self.partial.data_ptr(), self.sums.data_ptr(),
                                              _lib.stream_handle()))
        return self.sums[:4].cpu().numpy().copy()

    def energy(self) -> ScoreBreakdown:
        y = self.assemble_device(self.buf.get("energy_y", self.dp.ny, self.dp.mu.dtype))
        s = self.energy_terms(y)
        lam, eps = self.problem.div.lam, self.problem.eps
        return ScoreBreakdown(transport=float(s[0]), entropy=eps * float(s[1]),
                              d1=lam * float(s[2]), d2=lam * float(s[3]))

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
            box = _box_from4(b, self.ndim)
            if b[1] == 0 or b[3] == 0:
                out.append(SparseCellMarginal.empty(self.ndim))
                continue
            v = flat[offs[i]:offs[i + 1]].reshape(b[1], b[3])
            out.append(SparseCellMarginal(box, v[0] if self.ndim == 1 else v))
        return out

    def download_marginals(self):
        """(boxes [n_basic, 4], concatenated values, offsets): the basic-cell Y-marginals
        compacted on the device (only the entries inside each box leave it)."""
        import torch

        b = self.ybox.view(-1, 4).to(torch.int64)
        sizes = b[:, 1] * b[:, 3]
        vals = self.yval.view(self.n_basic, self.cap)
        idx = torch.arange(self.cap, device=vals.device)[None, :] < sizes[:, None]
        flat = vals[idx].cpu().numpy()
        boxes = self.ybox.view(-1, 4).cpu().numpy()
        szh = boxes[:, 1].astype(np.int64) * boxes[:, 3]
        offs = np.concatenate([[0], np.cumsum(szh)])
        return boxes, flat, offs

    @property
    def mu_nodes(self) -> list:
        flat = self.problem.mu.mass.ravel()
        return [flat[ids] for ids in self.basic.nodes_of_cell]

    @property
    def x_marg(self) -> list:
        xm = self.x_marg_d.view(self.n_basic, self.bs).cpu().numpy()
        out = []
        mu = np.asarray(self.problem.mu.mass, dtype=np.float64)
        mu2 = mu.reshape(1, -1) if mu.ndim == 1 else mu
        bx = self.basic_xbox.view(-1, 4).cpu().numpy()
        for i in range(self.n_basic):
            b = bx[i]
            blk = mu2[b[0]:b[0] + b[1], b[2]:b[2] + b[3]].ravel()
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
        out = {}
        for label, st in self.stores.items():
            has = st.has.cpu().numpy()
            al = st.alpha.view(st.ncomp, st.nx).cpu().numpy()
            bx = st.box.view(st.ncomp, 4).cpu().numpy()
            be = st.beta.view(st.ncomp, st.dcap).cpu().numpy()
            for j in range(st.ncomp):
                if not has[j]:
                    continue
                b = bx[j]
                out[(label, j)] = CellDuals(alpha=al[j].copy(), beta_box=_box_from4(b, self.ndim),
                                            beta=be[j, :b[1] * b[3]].copy())
        return out

    def sparsity(self) -> dict:
        """Stored and non-zero entries of the basic-cell marginals (engine.py:198-201),
        counted on the device (only two scalars leave it)."""
        import torch

        b = self.ybox.view(-1, 4).to(torch.int64)
        sizes = b[:, 1] * b[:, 3]
        vals = self.yval.view(self.n_basic, self.cap)
        idx = torch.arange(self.cap, device=vals.device)[None, :] < sizes[:, None]
        nz = int(((vals != 0) & idx).sum().item())
        return {"stored_entries": int(sizes.sum().item()), "nonzero_entries": nz}

    def clone(self) -> "PlanState":
        c = object.__new__(PlanState)
        c.__dict__.update(self.__dict__)
        c.ybox, c.yval = self.ybox.clone(), self.yval.clone()
        c.ybox_h = self.ybox_h.copy()
        c.x_marg_d, c.transport_d, c.kl_d = (self.x_marg_d.clone(), self.transport_d.clone(),
                                             self.kl_d.clone())
        c.stores = {k: v.clone() for k, v in self.stores.items()}
        c.iter_hist = {k: v.copy() for k, v in self.iter_hist.items()}
        c.owner = None if self.owner is None else self.owner.copy()
        c.comp_owner = dict(self.comp_owner)
        c.buf = _Buffers(self.dp.device)
        c.partial = self.partial.clone()
        c.sums = self.sums.clone()
        return c


def initial_plan_state(problem: TransportProblem, basic: BasicPartition,
                       dp: DeviceProblem | None = None) -> PlanState:
    """Product start nu_i = (|mu_i|/|mu|) nu on the full box (engine.py:234-257)."""
    if problem.mu.grid.ndim == 3:
        from .volume import initial_plan_state3
        return initial_plan_state3(problem, basic, dp)
    st = PlanState(problem, basic, dp, cap=problem.nu.grid.nnodes)
    _lib.check(_lib.lib().dd_product_init(st.dp.geom, st.state_struct(), st.dp.mu_total,
                                          _lib.stream_handle()))
    st.sync_boxes()
    return st


def _union_boxes(boxes: np.ndarray, full: np.ndarray) -> np.ndarray:
    """Row-wise union over member boxes (n, MW, 4) with invalid rows flagged by ext 0."""
    valid = (boxes[..., 1] > 0) & (boxes[..., 3] > 0)
    big = np.iinfo(np.int32).max
    lo0 = np.where(valid, boxes[..., 0], big).min(axis=1)
    hi0 = np.where(valid, boxes[..., 0] + boxes[..., 1], -big).max(axis=1)
    lo1 = np.where(valid, boxes[..., 2], big).min(axis=1)
    hi1 = np.where(valid, boxes[..., 2] + boxes[..., 3], -big).max(axis=1)
    out = np.stack([lo0, hi0 - lo0, lo1, hi1 - lo1], axis=1).astype(np.int32)
    none = ~valid.any(axis=1)
    out[none] = full
    return out


def _member_boxes(st: PlanState, pt: _PartTables, ids) -> np.ndarray:
    mem = pt.mem[ids]
    bx = st.ybox_h[np.where(mem >= 0, mem, 0)]
    bx = np.where((mem >= 0)[..., None], bx, 0)
    full = np.array([0, st.dp.geom.ny0, 0, st.dp.geom.ny1], dtype=np.int32)
    return _union_boxes(bx, full)


def _cut_plan_embedded(st: "PlanState", dp: DeviceProblem, alpha, beta, trunc: float,
                       trunc_out, cut_log: float | None = None) -> None:
    """warm_start_plan's plan cut (engine.py:294-322) through the three-axis kernel
    (``dd3_cut_plan``: candidate boxes from tile bounds, separable column sums, X-marginals
    from one global X sweep) on the (1, n0, n1) embedding of this 2D state: slots,
    X-marginals and fragments share their layout; the boxes come back as (0, 1) + box4.
    Terms below e^``cut_log`` are culled from 512^2 nodes up (-60, default), every
    non-zero term is kept on smaller grids."""
    import torch

    g = dp.geom
    g3 = _lib.Geom3()
    for a, (nx, ny, ox, oy) in enumerate(((1, 1, 0.0, 0.0), (g.nx0, g.ny0, g.x_org0, g.y_org0),
                                          (g.nx1, g.ny1, g.x_org1, g.y_org1))):
        g3.nx[a], g3.ny[a], g3.x_org[a], g3.y_org[a] = nx, ny, ox, oy
    g3.first_axis = 3 - st.ndim
    g3.x_dx, g3.y_dx, g3.eps, g3.lam, g3.nu_total = g.x_dx, g.y_dx, g.eps, g.lam, g.nu_total
    if cut_log is None:
        cut_log = -60.0 if dp.ny >= 512 * 512 else -800.0
    nb = st.n_basic
    dev = dp.device
    bx6 = torch.zeros((nb, 6), dtype=torch.int32, device=dev)
    bx6[:, 1] = 1
    bx6[:, 2:] = st.basic_xbox.view(nb, 4)
    yb6 = torch.zeros(nb * 6, dtype=torch.int32, device=dev)
    work = torch.empty(int(_lib.lib().dd3_cut_tiles(g3)), dtype=torch.float64, device=dev)

    def state3(with_values: bool):
        s3 = _lib.State3(mu=dp.mu.data_ptr(), nu=dp.nu.data_ptr(), log_mu=dp.log_mu.data_ptr(),
                         log_nu=dp.log_nu.data_ptr(), n_basic=nb, basic_xbox=bx6.data_ptr(),
                         basic_mass=st.basic_mass.data_ptr(), ybox=yb6.data_ptr(),
                         yval=st.yval.data_ptr() if with_values else None, cap=st.cap,
                         x_marg=st.x_marg_d.data_ptr(), transport=st.transport_d.data_ptr(),
                         kl=st.kl_d.data_ptr())
        s3.block[0], s3.block[1], s3.block[2] = 1, st.block[0], st.block[1]
        return s3

    boxes = torch.zeros(nb * 6, dtype=torch.int32, device=dev)
    lib = _lib.lib()
    _lib.check(lib.dd3_cut_plan(g3, state3(False), alpha.data_ptr(), beta.data_ptr(), trunc,
                                float(cut_log), work.data_ptr(), trunc_out.data_ptr(),
                                boxes.data_ptr(), _lib.stream_handle()))
    bh = boxes.view(-1, 6).cpu().numpy().astype(np.int64)
    st.ensure_cap(int((bh[:, 1] * bh[:, 3] * bh[:, 5]).max(initial=1)))
    _lib.check(lib.dd3_cut_plan(g3, state3(True), alpha.data_ptr(), beta.data_ptr(), trunc,
                                float(cut_log), work.data_ptr(), trunc_out.data_ptr(),
                                boxes.data_ptr(), _lib.stream_handle()))
    st.ybox.view(nb, 4).copy_(yb6.view(nb, 6)[:, 2:])


def warm_start_plan(problem: TransportProblem, partitions: Decomposition, delta: float = 1e-3,
                    max_iters: int = 20_000, trunc_threshold: float = 1e-15,
                    dp: DeviceProblem | None = None, alpha0=None, beta0=None) -> PlanState:
    """Loose global presolve, plan cut along basic cells, duals seeded (engine.py:260-345).

    ``alpha0``/``beta0`` warm-start the presolve (the multiscale driver passes
    duals prolonged from the previous layer; ``max_iters=0`` cuts the plan of
    those duals directly)."""
    import torch

    if problem.mu.grid.ndim == 3:
        from .volume import warm_start_plan3
        return warm_start_plan3(problem, partitions, delta, max_iters, trunc_threshold, dp,
                                alpha0, beta0)

    dp = dp if dp is not None else DeviceProblem(problem)
    res = sinkhorn_solve(dp, alpha0, beta0, config=SolverConfig(delta=delta, max_iters=max_iters))
    st = PlanState(problem, partitions.basic, dp, cap=1)
    L = _lib.lib()
    trunc_out = torch.zeros(st.n_basic, dtype=torch.float64, device=dp.device)
    _cut_plan_embedded(st, dp, res.alpha, res.beta, float(trunc_threshold), trunc_out)
    st.sync_boxes()
    st.truncated_mass = float(trunc_out.sum().item())
    for part in partitions.composites:
        pt = _tables(part)
        ids = np.arange(pt.ncomp)
        yb = _member_boxes(st, pt, ids)
        store = st.store(pt)
        store.ensure(int((yb[:, 1].astype(np.int64) * yb[:, 3]).max(initial=1)))
        xb_d = torch.from_numpy(pt.xbox.ravel().copy()).to(dp.device)
        yb_d = torch.from_numpy(yb.ravel().copy()).to(dp.device)
        _lib.check(L.dd_seed_duals(dp.geom, st.state_struct(store), pt.ncomp, pt.nw0, pt.nw1,
                                   xb_d.data_ptr(), yb_d.data_ptr(), res.alpha.data_ptr(),
                                   res.beta.data_ptr(), _lib.stream_handle()))
    st.global_duals = (res.alpha.clone(), res.beta.clone())
    return st


_SHARD: ShardSpec | None = None


def set_shard(group=None) -> ShardSpec:
    """Row-slab sharding of every domdec solve over ``group`` (default: WORLD);
    see :mod:`paper_2410_08859_b200.slab`."""
    global _SHARD
    _SHARD = ShardSpec(group)
    return _SHARD


def clear_shard() -> None:
    global _SHARD
    _SHARD = None


_TABLE_CACHE: dict = {}
_SIDE_STREAMS: dict = {}


def _side_stream(device):
    """Second stream for the large-window cells of a batch (one per device)."""
    import torch

    key = str(device)
    s = _SIDE_STREAMS.get(key)
    if s is None:
        s = torch.cuda.Stream(device=device)
        _SIDE_STREAMS[key] = s
    return s


def C_void(v):
    import ctypes
    return ctypes.c_void_p(v)


def _tables(part: CompositePartition) -> _PartTables:
    key = id(part)
    hit = _TABLE_CACHE.get(key)
    if hit is None or hit.part is not part:
        hit = _PartTables(part)
        _TABLE_CACHE[key] = hit
    return hit


def _slab_layout(st: "PlanState", pt: _PartTables):
    """(composite owner, basic-cell owner) of a partition under the active slab sharding."""
    lat = st.basic.lattice_to_cell.shape
    rows, cols = (lat[0], lat[1]) if len(lat) == 2 else (1, lat[0])
    return _SHARD.layout(pt, st.block, st.n_basic, rows, cols)


# -- one batch on the device -----------------------------------------------------------

def _ws_total(nw0: int, nw1: int, ny0: np.ndarray, ny1: np.ndarray) -> np.ndarray:
    """dd_cell_ws_size, vectorized (mirrors ws_layout in csrc/cell.cu)."""
    nx = nw0 * nw1
    ny = ny0 * ny1
    ms = np.maximum(ny0 * nw1, nw0 * ny1)
    rm = np.maximum(np.maximum(ny0, ny1), max(nw0, nw1))
    return (nw0 + nw1 + ny0 + ny1 + 7 * nx + 3 * ny + nw0 * ny0 + nw1 * ny1 + 5 * ms + rm
            + nw0 * ny0 + nw1 * ny1 + ny0 + ny1)   # Y-sweep normalised tables, c0, c1


class _Batch:
    """Device arenas and host tables of one solved batch of composite cells."""

    def __init__(self, st: PlanState, pt: _PartTables, ids, snapshot, cfg: CellSolverConfig):
        import torch

        dev = st.dp.device
        self.st, self.pt = st, pt
        ids = np.asarray(ids, dtype=np.int64)
        self.ids = ids
        n = len(ids)
        self.n = n
        yb = _member_boxes(st, pt, ids)
        self.ybox = yb
        ny0 = yb[:, 1].astype(np.int64)
        ny1 = yb[:, 3].astype(np.int64)
        ny = ny0 * ny1
        self.ny = ny
        nmem = pt.nmem[ids].astype(np.int64)
        self.nmem = nmem
        members = [pt.mem[j, :pt.nmem[j]] for j in ids]
        self.members_h = members
        membase = np.concatenate([[0], np.cumsum(nmem)[:-1]]).astype(np.int64)
        self.membase = membase
        yoff = np.concatenate([[0], np.cumsum(ny)[:-1]]).astype(np.int64)
        moff = np.concatenate([[0], np.cumsum(6 * nmem * ny)[:-1]]).astype(np.int64)
        xoff = np.concatenate([[0], np.cumsum(nmem * st.bs)[:-1]]).astype(np.int64)
        ws = _ws_total(pt.nw0, pt.nw1, ny0, ny1).astype(np.int64)
        mode = _MODE[0]
        budget = mode.smem_budget or _smem_budget()
        fits = ws * 8 <= (0 if mode.force_global_ws else budget)
        if mode.force_cluster:
            fits = np.zeros_like(fits)
        clu = np.zeros(n, dtype=bool)
        csize = np.zeros(n, dtype=np.int64)
        csmem = np.zeros(n, dtype=np.int64)
        # latency: cells whose last solve ran to the cap will again hold the batch
        # open for max_iters iterations.  When they are few (2 CTAs each fit the SMs
        # with room to spare) each runs on a 2-CTA cluster, its Y rows split over two
        # otherwise idle SMs
        hist = st.iter_hist.get(pt.label)
        if (hist is not None and mode.cluster_capped and not mode.force_cluster
                and not mode.no_cluster and not mode.force_global_ws):
            capped = fits & (hist[ids] >= cfg.max_iters) & (ny0 >= 2)
            nc = int(capped.sum())
            if 0 < nc and 2 * nc <= _sm_count(dev):
                cws = _cluster_ws(pt.nw0, pt.nw1, ny0, ny1, 2) * 8
                ok = capped & (cws <= budget)
                csize[ok] = 2
                csmem[ok] = cws[ok]
                clu |= ok
                fits = fits & ~ok
        # cells whose workspace fits run in shared memory (sized for the largest
        # of them); the rest get global-arena slots
        smem_bytes = int(ws[fits].max()) * 8 if fits.any() else 0
        smem_mode = bool(fits.any())
        gws = np.where(fits, 0, ws)
        self.n_big = int((~fits).sum())
        # large cells: Sinkhorn loop on a thread-block cluster, each cell on the
        # smallest cluster (2, 4, 8, 16 CTAs) whose per-CTA workspace fits;
        # one launch per cluster size
        big = ~fits
        if big.any() and not mode.no_cluster and not mode.force_global_ws:
            sizes = (mode.force_cluster,) if mode.force_cluster else CLUSTER_SIZES
            for C in sizes:
                cws = _cluster_ws(pt.nw0, pt.nw1, ny0, ny1, C) * 8
                ok = big & ~clu & (cws <= budget) & (ny0 >= C)
                csize[ok] = C
                csmem[ok] = cws[ok]
                clu |= ok
        # slab mode: composites of other ranks' slabs are skipped (desc flag bit 1)
        owned = np.ones(n, dtype=bool)
        self.shard = _SHARD if st._sharded() else None
        if self.shard is not None:
            comp, _ = _slab_layout(st, pt)
            owned = comp[ids] == self.shard.rank
            clu &= owned
        self.owned = owned
        # expected cost of each cell: window size x the executed iterations of its
        # previous solve (the iteration count is strongly persistent across sweeps);
        # CTAs and cluster launches take cells longest-first
        hist = st.iter_hist.get(pt.label)
        prev = hist[ids] if hist is not None else np.zeros(n)
        cost = ny.astype(np.float64) * (prev + 1.0)
        self.order_h = np.argsort(-cost, kind="stable").astype(np.int32)
        groups = []
        for C in sorted(set(csize[clu].tolist())):
            sel = np.flatnonzero(clu & (csize == C))
            sel = sel[np.argsort(-cost[sel], kind="stable")]
            groups.append((int(C), sel, int(csmem[sel].max())))
        self.clu_groups = groups
        self.n_clu = int(clu.sum())
        # split loop: when the batch has many more cells than SMs (throughput-bound),
        # the shared-memory cells whose workspace fits half an SM run the loop kernel
        # two CTAs per SM, then their epilogue in the solve kernel (desc flag 4)
        split = np.zeros(n, dtype=bool)
        split_smem = 0
        if ((mode.split_loop or mode.force_split) and not mode.force_cluster
                and not mode.force_global_ws
                and (mode.force_split or int(fits.sum()) >= 3 * _sm_count(dev))):
            half = (220 * 1024) // 2 - 1024
            split = fits & (ws * 8 <= half)
            split_smem = int(ws[split].max()) * 8 if split.any() else 0
        self.n_split = int(split.sum())
        woff = np.concatenate([[0], np.cumsum(gws)[:-1]]).astype(np.int64)
        desc = np.zeros((n, 12), dtype=np.int32)
        desc[:, 0] = ids
        desc[:, 1:5] = pt.xbox[ids]
        desc[:, 5:9] = yb
        desc[:, 9] = nmem
        desc[:, 10] = membase
        desc[:, 11] = (clu.astype(np.int32) | np.where(owned, 0, 2).astype(np.int32)
                       | np.where(split & owned, 4, 0).astype(np.int32))
        offs = np.stack([yoff, moff, woff, xoff], axis=1).astype(np.int64)
        mflat = np.concatenate(members).astype(np.int32) if n else np.zeros(0, np.int32)
        self.mflat = mflat
        # capacity for the new boxes (each lies inside its cell's Y window)
        need = int(ny.max(initial=1))
        st.ensure_cap(need)
        store = st.store(pt)
        store.ensure(need)
        self.store = store
        tot_y = int(ny.sum())
        tot_m = int((6 * nmem * ny).sum())
        tot_mem = int(nmem.sum())
        B = st.buf
        f64, i32, i64 = torch.float64, torch.int32, torch.int64
        self.desc_d = torch.from_numpy(desc.ravel()).to(dev)
        self.order_d = torch.from_numpy(self.order_h).to(dev) if n else B.get("order", 1, i32)
        self.offs_d = torch.from_numpy(offs.ravel()).to(dev)
        self.mem_d = torch.from_numpy(mflat).to(dev) if tot_mem else B.get("mem", 1, i32)
        self.alpha = B.get("alpha", n * pt.nw0 * pt.nw1, f64)
        self.beta = B.get("beta", tot_y, f64)
        self.mdens = B.get("mdens", tot_y, f64)
        self.lnuw = B.get("lnuw", tot_y, f64)
        self.lmw = B.get("lmw", tot_y, f64)
        self.lout = B.get("lout", n * pt.nw0 * pt.nw1, f64)
        clu_ids = (np.concatenate([sel for _, sel, _ in groups]).astype(np.int32) if groups
                   else np.zeros(0, np.int32))
        self.clu_ids = (torch.from_numpy(clu_ids).to(dev) if len(clu_ids)
                        else B.get("clu_ids", 1, i32))
        import ctypes
        ng = len(groups)
        goff = np.concatenate([[0], np.cumsum([len(sel) for _, sel, _ in groups])]).astype(np.int32)
        self.clu_n_groups = ng
        self.clu_goff = (ctypes.c_int32 * (ng + 1))(*goff.tolist())
        self.clu_gsize = (ctypes.c_int32 * max(1, ng))(*[C for C, _, _ in groups])
        self.clu_gsmem = (ctypes.c_int32 * max(1, ng))(*[m for _, _, m in groups])
        self.marena = B.get("marena", tot_m, f64)
        self.work = B.get("work", int(gws.sum()) + 1, f64)
        self.xarena = B.get("xarena", tot_mem * st.bs, f64)
        self.mbox = B.get("mbox", tot_mem * 4, i32)
        self.mstat = B.get("mstat", tot_mem * 4, f64)
        self.cstat = B.get("cstat", n * 8, f64)
        self.cstat2 = B.get("cstat2", n * 8, f64)
        self.dy = None
        self.tot = dict(y=tot_y, m=tot_m, mem=tot_mem)
        self.yoff = yoff
        self.snapshot = snapshot
        self.batch = _lib.Batch(
            n_cells=n, nxw0=pt.nw0, nxw1=pt.nw1, desc=self.desc_d.data_ptr(),
            offs=self.offs_d.data_ptr(), members=self.mem_d.data_ptr(),
            snapshot=snapshot.data_ptr(), alpha=self.alpha.data_ptr(), beta=self.beta.data_ptr(),
            mdens=self.mdens.data_ptr(), marena=self.marena.data_ptr(), work=self.work.data_ptr(),
            xarena=self.xarena.data_ptr(), mbox=self.mbox.data_ptr(), mstat=self.mstat.data_ptr(),
            cstat=self.cstat.data_ptr(), cstat2=self.cstat2.data_ptr(),
            smem_mode=1 if smem_mode else 0, smem_bytes=smem_bytes if smem_mode else 0,
            delta=cfg.delta, max_iters=cfg.max_iters, newton_max_iters=cfg.newton_max_iters,
            newton_tol=cfg.newton_tol, trunc=cfg.trunc_threshold, lnuw=self.lnuw.data_ptr(),
            lout=self.lout.data_ptr(), skip_stagnant=1 if mode.skip_stagnant else 0,
            order=self.order_d.data_ptr() if n else None, lmw=self.lmw.data_ptr(),
            split_smem_bytes=split_smem,
            precision=1 if cfg.precision == "fp32" else 0)
        self.cfg = cfg

    def solve(self):
        import torch

        st = self.st
        n_big = int(self.n_big)
        side = C_void(_side_stream(st.dp.device).cuda_stream) if n_big else None
        _lib.check(_lib.lib().dd_cell_solve2(st.dp.geom, st.state_struct(self.store), self.batch,
                                             _lib.stream_handle(), side, n_big,
                                             self.clu_ids.data_ptr(), self.clu_n_groups,
                                             self.clu_goff, self.clu_gsize, self.clu_gsmem))

    def stats(self):
        c1 = self.cstat[:self.n * 8].view(self.n, 8).cpu().numpy()
        c2 = self.cstat2[:self.n * 8].view(self.n, 8).cpu().numpy()
        return c1, c2

    def commit(self, theta: np.ndarray, alpha_grid=None, yrun=None) -> np.ndarray:
        import torch

        st = self.st
        th = torch.from_numpy(np.ascontiguousarray(theta, dtype=np.float64)).to(st.dp.device)
        errs = st.buf.get("errs", self.n * 4, torch.float64)
        _lib.check(_lib.lib().dd_cell_commit(st.dp.geom, st.state_struct(self.store), self.batch,
                                             th.data_ptr(), _lib.ptr(alpha_grid), _lib.ptr(yrun),
                                             errs.data_ptr(), _lib.stream_handle()))
        e = errs[:self.n * 4].view(self.n, 4).cpu().numpy().copy()
        # refresh the host box mirror for the committed members
        if len(self.mflat):
            idx = self.mflat.astype(np.int64)
            st.ybox_h[idx] = st.ybox.view(-1, 4)[torch.from_numpy(idx).to(st.dp.device)].cpu().numpy()
        return e


# -- blend scoring and weight strategies ---------------------------------------------

class BlendScorer:
    """Tracked energy of theta-blended batch updates (engine.py:378-470)."""

    def __init__(self, plan: PlanState, batch: _Batch, snapshot):
        import torch

        self.plan, self.batch = plan, batch
        st = plan
        self.lam, self.eps = plan.problem.div.lam, plan.problem.eps
        tot_y = int(batch.ny.sum())
        self.dy = st.buf.get("dy", tot_y, torch.float64)
        self.cd = st.buf.get("cd", batch.n * 4, torch.float64)
        self.ywork = st.buf.get("ywork", st.dp.ny, torch.float64)
        self.out = st.buf.get("bout", 8, torch.float64)
        _lib.check(_lib.lib().dd_cell_delta(st.dp.geom, st.state_struct(batch.store), batch.batch,
                                            self.dy.data_ptr(), self.cd.data_ptr(),
                                            _lib.stream_handle()))
        base = st.energy_terms(snapshot)
        self.base_t, self.base_k = float(base[0]), float(base[1])
        self.base_d1 = self.lam * float(base[2])
        self.snapshot = snapshot
        self.n = batch.n
        self.theta = np.zeros(self.n)
        self.evaluations = 0

    def opt_state(self) -> "_OptState":
        return _OptState(self)

    # reference-shaped incremental view (engine.py:458-470), kept on the device
    def _op(self) -> "_OptState":
        if getattr(self, "_opt", None) is None:
            self._opt = _OptState(self)
        return self._opt

    def set_theta(self, idx: int, theta: float) -> None:
        self._op().set_theta(int(idx), float(theta))
        self.theta = self._op().theta

    def minimize_coordinate(self, idx: int, tol: float) -> float:
        return self._op().minimize_coordinate(int(idx), float(tol))

    def energy_at(self, theta_vec) -> float:
        import torch

        st, b = self.plan, self.batch
        th = np.ascontiguousarray(theta_vec, dtype=np.float64)
        if b.shard is not None:
            # slab mode: this rank's cells only; dense sum of theta*dy and the per-cell
            # pieces are reduced over the slabs, then y = snapshot + sum, KL(y | nu)
            thd = torch.from_numpy(np.where(b.owned, th, 0.0)).to(st.dp.device)
            L = _lib.lib()
            _lib.check(L.dd_blend_parts(st.dp.geom, st.state_struct(b.store), b.batch,
                                        self.dy.data_ptr(), self.cd.data_ptr(), thd.data_ptr(),
                                        self.ywork.data_ptr(), st.partial.data_ptr(),
                                        self.out.data_ptr(), _lib.stream_handle()))
            ny = st.dp.ny
            b.shard.all_reduce(self.ywork[:ny])
            b.shard.all_reduce(self.out[1:4])
            axpb(self.ywork[:ny], 1.0, self.snapshot[:ny], out=self.ywork[:ny])
            _lib.check(L.dd_grid_kl(ny, self.ywork.data_ptr(), st.dp.nu.data_ptr(), 1,
                                    st.partial.data_ptr(), self.out.data_ptr(),
                                    _lib.stream_handle()))
        else:
            thd = torch.from_numpy(th).to(st.dp.device)
            _lib.check(_lib.lib().dd_blend_energy(st.dp.geom, st.state_struct(b.store), b.batch,
                                                  self.dy.data_ptr(), self.cd.data_ptr(),
                                                  thd.data_ptr(), self.ywork.data_ptr(),
                                                  st.partial.data_ptr(), self.out.data_ptr(),
                                                  _lib.stream_handle()))
        o = self.out[:4].cpu().numpy()
        self.evaluations += 1
        t = self.base_t + float(o[1])
        kl = self.base_k + float(o[2])
        d1 = self.base_d1 + float(o[3])
        return t + self.eps * kl + d1 + self.lam * float(o[0])


def _cell_ids(cells) -> list:
    """Composite ids of the updated cells: the reference passes CellSolution objects
    (their ``.j``), the device engine passes the ids themselves."""
    return [int(getattr(c, "j", c)) for c in cells]


def get_weights_safe(old_cells, new_cells, part) -> WeightAssignment:
    """theta = 1/K for the K updated cells (engine.py:533-540)."""
    ids = _cell_ids(new_cells)
    k = len(ids)
    return WeightAssignment({int(j): 1.0 / k for j in ids})


def get_weights_swift(old_cells, new_cells, part, scorer: BlendScorer) -> WeightAssignment:
    """Better of greedy (ones) and safe (1/K); ties to greedy (engine.py:543-554)."""
    ids = _cell_ids(new_cells)
    k = len(ids)
    ones, safe = np.ones(k), np.full(k, 1.0 / k)
    vec = ones if scorer.energy_at(ones) <= scorer.energy_at(safe) else safe
    return WeightAssignment({int(j): float(t) for j, t in zip(ids, vec)})


def _coordinate_root(gh, tol: float, max_iters: int = 60) -> float:
    """Safeguarded Newton on the increasing blend derivative over [0, 1] (engine.py:473-527)."""
    g0, _ = gh(0.0)
    if g0 >= 0.0:
        return 0.0
    g1, _ = gh(1.0)
    if g1 <= 0.0:
        return 1.0
    lo, hi, th = 0.0, 1.0, 0.5
    for _ in range(max_iters):
        g, h = gh(th)
        if g == 0.0:
            break
        if g > 0.0:
            hi = th
        else:
            lo = th
        cand = th - g / h if np.isfinite(g) and np.isfinite(h) and h > 0.0 else 0.5 * (lo + hi)
        if not lo < cand < hi:
            cand = 0.5 * (lo + hi)
        if abs(cand - th) <= tol * max(1.0, abs(th)):
            th = cand
            break
        th = cand
    return min(max(th, 0.0), 1.0)


class _OptState:
    """Incremental blend view for coordinate descent (BlendScorer.set_theta /
    minimize_coordinate, engine.py:458-470), kept on the device."""

    def __init__(self, scorer: BlendScorer):
        import torch

        self.sc = scorer
        st = scorer.plan
        self.ycur = st.buf.get("opt_ycur", st.dp.ny, torch.float64)
        self.ycur[:st.dp.ny].copy_(scorer.snapshot[:st.dp.ny])
        self.out = st.buf.get("opt_out", 4, torch.float64)
        cd = scorer.cd[:scorer.n * 4].view(scorer.n, 4).cpu().numpy()
        self.lin = cd[:, 0] + scorer.eps * cd[:, 1]
        self.theta = np.zeros(scorer.n)

    def set_theta(self, i: int, th: float) -> None:
        sc = self.sc
        dth = th - self.theta[i]
        if dth:
            _lib.check(_lib.lib().dd_opt_set(sc.plan.dp.geom, sc.batch.batch, sc.dy.data_ptr(),
                                             int(i), float(dth), self.ycur.data_ptr(),
                                             _lib.stream_handle()))
        self.theta[i] = th

    def minimize_coordinate(self, i: int, tol: float) -> float:
        sc = self.sc
        st, b = sc.plan, sc.batch
        lam = sc.lam
        lin = float(self.lin[i])
        th_cur = float(self.theta[i])
        sstruct = st.state_struct(b.store)

        def gh(th):
            _lib.check(_lib.lib().dd_opt_gh(st.dp.geom, sstruct, b.batch, sc.dy.data_ptr(), int(i),
                                            float(th), th_cur, self.ycur.data_ptr(),
                                            self.out.data_ptr(), _lib.stream_handle()))
            o = self.out[:4].cpu().numpy()
            with np.errstate(invalid="ignore"):
                g = lin + lam * float(o[0]) + lam * float(o[2])
                h = lam * float(o[1]) + lam * float(o[3])
            return g, h

        return _coordinate_root(gh, tol)


def get_weights_opt(old_cells, new_cells, part, scorer: BlendScorer, max_sweeps: int = 50,
                    tol: float = 1e-9) -> WeightAssignment:
    """Cyclic coordinate descent over theta in [0, 1]^K on the tracked energy,
    seeded with the better of safe and greedy; returns the best of {descent
    iterate, greedy, safe} (engine.py:557-588)."""
    ids = _cell_ids(new_cells)
    k = len(ids)
    if getattr(scorer, "sharded", False) or getattr(scorer.batch, "shard", None) is not None:
        raise ValueError("the opt strategy needs per-cell global coordination inside a batch; "
                         "slab-sharded solves support safe, fast, swift and staggered")
    ones, safe = np.ones(k), np.full(k, 1.0 / k)
    start = ones if scorer.energy_at(ones) <= scorer.energy_at(safe) else safe
    op = scorer.opt_state()
    for i in range(k):
        op.set_theta(i, float(start[i]))
    for _ in range(max_sweeps):
        moved = 0.0
        for i in range(k):
            th = op.minimize_coordinate(i, tol)
            moved = max(moved, abs(th - op.theta[i]))
            op.set_theta(i, th)
        if moved <= tol:
            break
    candidates = [op.theta.copy(), ones, safe]
    energies = [scorer.energy_at(v) for v in candidates]
    best = candidates[int(np.argmin(energies))]
    return WeightAssignment({int(j): float(t) for j, t in zip(ids, best)})


# -- stopping certificate -----------------------------------------------------------------

class StitchedGapEvaluator:
    """E(state) - D(stitched alpha, polished beta), best pair persisted (engine.py:594-682)."""

    def __init__(self, problem: TransportProblem, polish: int = 2, dp: DeviceProblem | None = None):
        if dp is None:
            if problem.mu.grid.ndim == 3:
                from .volume import VolumeProblem
                dp = VolumeProblem(problem)
            else:
                dp = DeviceProblem(problem)
        self.dp = dp
        self.sweeper = self.dp.make_sweeper()
        self.eps = float(problem.eps)
        self.lam = float(problem.div.lam)
        self.polish = int(polish)
        self.mass_product = self.dp.mu_total * self.dp.nu_total
        self._best = None

    def seed(self, alpha, beta) -> None:
        import torch

        a = torch.as_tensor(alpha).reshape(-1).to(self.dp.device, torch.float64).clone()
        b = torch.as_tensor(beta).reshape(-1).to(self.dp.device, torch.float64).clone()
        self._best = (a, b, self._dual_at(a, b))

    def _ascend(self, beta):
        eps, lam = self.eps, self.lam
        scale = eps * lam / (eps + lam)
        alpha = beta_new = None
        dp, sw = self.dp, self.sweeper
        for _ in range(max(1, self.polish)):
            alpha = axpb(sw.lse_x(axpb(beta, eps, dp.log_nu, divide=True)), -scale)
            beta_new = axpb(sw.lse_y(axpb(alpha, eps, dp.log_mu, divide=True)), -scale)
            beta = beta_new
        return alpha, beta_new

    def _dual_at(self, alpha, beta) -> float:
        eps, lam = self.eps, self.lam
        dp = self.dp
        z = self.sweeper.lse_y(axpb(alpha, eps, dp.log_mu, divide=True))
        coupling, sx, sy = dual_sums(dp, alpha, beta, z)
        return lam * sx + lam * sy - eps * (coupling - self.mass_product)

    def dual_value(self, alpha_flat) -> float:
        eps, lam = self.eps, self.lam
        scale = eps * lam / (eps + lam)
        dp = self.dp
        beta0 = axpb(self.sweeper.lse_y(axpb(alpha_flat, eps, dp.log_mu, divide=True)), -scale)
        a1, b1 = self._ascend(beta0)
        d1 = self._dual_at(a1, b1)
        if self._best is not None:
            a2, b2 = self._ascend(self._best[1])
            d2 = self._dual_at(a2, b2)
            if d2 > d1 or (d2 == d1 and self._best[2] > d1):
                a1, b1, d1 = a2, b2, d2
            d1 = max(d1, self._best[2])
        self._best = (a1, b1, d1)
        return d1

    def evaluate(self, alpha_flat, energy_total: float) -> float:
        return energy_total - self.dual_value(alpha_flat)


# -- iterations ------------------------------------------------------------------------

@dataclass
class IterationStats:
    k: int = 0
    label: str = ""
    action: str = ""
    gap: float = float("nan")
    entry_gap: float = 0.0
    alpha: object = None
    x_err: float = 0.0
    y_err: float = 0.0
    assemble_time: float = 0.0
    solve_time: float = 0.0
    score_time: float = 0.0
    commit_time: float = 0.0
    balance_fallbacks: int = 0
    safe_fallbacks: int = 0
    truncated_mass: float = 0.0
    newton_clamped: int = 0
    nu_minus_clamped: int = 0
    nonconverged_cells: int = 0
    balance_target_miss: float = 0.0
    nu_j_drift_nodes: int = 0
    cell_iterations: int = 0
    cell_flops: float = 0.0


def cell_lse_flops(nw0: int, nw1: int, ny0, ny1):
    """Algorithmic FLOPs of one Sinkhorn iteration of a cell: the four separable
    contractions (2 per FMA) of the X and Y sweeps."""
    nx = nw0 * nw1
    return 2.0 * (ny0 * nw1 * ny1 + nx * ny0 + nw0 * ny1 * nw1 + ny0 * ny1 * nw0)


def _absorb(stats: IterationStats, batch: _Batch) -> None:
    c1, c2 = batch.stats()
    hist = batch.st.iter_hist.setdefault(batch.pt.label, np.zeros(batch.pt.ncomp))
    own = batch.owned
    hist[batch.ids[own]] = c2[own, 4]
    c1, c2 = c1[own], c2[own]
    fl = cell_lse_flops(batch.pt.nw0, batch.pt.nw1, batch.ybox[own, 1].astype(np.float64),
                        batch.ybox[own, 3].astype(np.float64))
    # roofline work counts executed iterations only (a stagnant cell's loop ends
    # early with the reference-equivalent count reported in c1)
    sums = np.array([(c2[:, 4] * fl).sum(), c1[:, 1].sum(), c1[:, 6].sum(), c1[:, 4].sum(),
                     (c1[:, 3] == 0).sum(), c2[:, 0].sum(), c1[:, 2].sum()], dtype=np.float64)
    maxs = np.array([c1[:, 5].max(initial=0), c1[:, 7].max(initial=0.0)], dtype=np.float64)
    if batch.shard is not None:
        sums = batch.shard.reduce_np(sums, "sum", batch.st.dp.device)
        maxs = batch.shard.reduce_np(maxs, "max", batch.st.dp.device)
    stats.cell_flops += float(sums[0])
    stats.entry_gap += float(sums[1])
    stats.balance_fallbacks += int(sums[2])
    stats.nu_minus_clamped += int(sums[3])
    stats.nonconverged_cells += int(sums[4])
    stats.nu_j_drift_nodes += int(sums[5])
    stats.cell_iterations += int(sums[6])
    stats.newton_clamped = max(stats.newton_clamped, int(maxs[0]))
    stats.balance_target_miss = max(stats.balance_target_miss, float(maxs[1]))


def _alpha_grid(plan: PlanState, stats: IterationStats):
    import torch
    if stats.alpha is None:
        stats.alpha = torch.zeros(plan.dp.nx, dtype=torch.float64, device=plan.dp.device)
    return stats.alpha


def _sync():
    import torch
    torch.cuda.synchronize()


def iteration_sequential(plan: PlanState, part: CompositePartition,
                         config: EngineConfig = EngineConfig(),
                         stats: IterationStats | None = None) -> PlanState:
    """Cell-by-cell pass on a running Y-marginal (engine.py:799-836)."""
    if _SHARD is not None and _SHARD.world > 1:
        raise ValueError("the sequential sweep is inherently serial; run it on one rank")
    stats = stats if stats is not None else IterationStats()
    cfg = config.cell_config()
    pt = _tables(part)
    t0 = time.perf_counter()
    y_run = plan.assemble_device(plan.buf.get("yrun", plan.dp.ny, plan.dp.mu.dtype))
    stats.assemble_time += time.perf_counter() - t0
    ag = _alpha_grid(plan, stats)
    for j in range(pt.ncomp):
        t0 = time.perf_counter()
        bt = _Batch(plan, pt, [j], y_run, cfg)
        bt.solve()
        stats.solve_time += time.perf_counter() - t0
        _absorb(stats, bt)
        t0 = time.perf_counter()
        e = bt.commit(np.ones(1), ag, y_run)
        stats.commit_time += time.perf_counter() - t0
        stats.x_err += float(e[0, 0])
        stats.y_err += float(e[0, 1])
        plan.truncated_mass += float(e[0, 2])
        stats.truncated_mass += float(e[0, 2])
    stats.action = "sequential"
    return plan


def iteration_parallel(plan: PlanState, part: CompositePartition, strategy: StrategyConfig,
                       config: EngineConfig = EngineConfig(),
                       stats: IterationStats | None = None) -> PlanState:
    """Snapshot, batch solve, weighted commit (engine.py:839-922)."""
    if strategy.kind == "sequential":
        raise ValueError("sequential updates run through iteration_sequential")
    stats = stats if stats is not None else IterationStats()
    cfg = config.cell_config()
    pt = _tables(part)
    batches = pt.batches if strategy.kind == "staggered" else [np.arange(pt.ncomp)]
    ag = _alpha_grid(plan, stats)
    shard = _SHARD if (_SHARD is not None and _SHARD.world > 1) else None
    if shard is not None:
        # this partition's slab ownership; the boundary block row's basic cells
        # (the halo) arrive from the neighbour that updated them last
        comp_owner, basic_owner = _slab_layout(plan, pt)
        shard.halo_exchange(plan, basic_owner)
        plan.comp_owner[pt.label] = comp_owner
    actions = []
    for batch in batches:
        t0 = time.perf_counter()
        snapshot = plan.assemble_device(plan.buf.get("snapshot", plan.dp.ny, plan.dp.mu.dtype))
        stats.assemble_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        bt = _Batch(plan, pt, batch, snapshot, cfg)
        bt.solve()
        _absorb(stats, bt)
        stats.solve_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        kb = bt.n
        ids = [int(j) for j in bt.ids]
        if strategy.kind == "fast":
            theta = np.ones(kb)
            actions.append("greedy")
        elif strategy.kind == "safe":
            theta = np.full(kb, 1.0 / kb)
            actions.append("safe")
        elif strategy.kind == "swift":
            scorer = BlendScorer(plan, bt, snapshot)
            w = get_weights_swift(None, ids, part, scorer).theta
            theta = np.array([w[j] for j in ids])
            actions.append("greedy" if all(t == 1.0 for t in theta) else "safe")
        elif strategy.kind == "opt":
            scorer = BlendScorer(plan, bt, snapshot)
            w = get_weights_opt(None, ids, part, scorer, strategy.opt_max_sweeps,
                                strategy.opt_tol).theta
            theta = np.array([w[j] for j in ids])
            actions.append("opt")
        else:
            scorer = BlendScorer(plan, bt, snapshot)
            e_base = scorer.energy_at(np.zeros(kb))
            e_greedy = scorer.energy_at(np.ones(kb))
            e_safe = scorer.energy_at(np.full(kb, 1.0 / kb))
            allowance = strategy.leniency * max(0.0, e_base - e_safe)
            if e_greedy <= e_base + allowance:
                theta = np.ones(kb)
                actions.append("greedy")
            else:
                theta = np.full(kb, 1.0 / kb)
                actions.append("safe-fallback")
                stats.safe_fallbacks += 1
        stats.score_time += time.perf_counter() - t0
        t0 = time.perf_counter()
        e = bt.commit(theta, ag, None)
        es = e[:, :3].sum(axis=0)
        if shard is not None:
            es = shard.reduce_np(es, "sum", plan.dp.device)
        stats.x_err += float(es[0])
        stats.y_err += float(es[1])
        added = float(es[2])
        plan.truncated_mass += added
        stats.truncated_mass += added
        stats.commit_time += time.perf_counter() - t0
    if shard is not None:
        shard.all_reduce(ag)   # stitched alpha: each rank wrote its own composites' blocks
    if len(actions) == 1:
        stats.action = actions[0]
    else:
        n_fb = actions.count("safe-fallback")
        stats.action = "greedy" if n_fb == 0 else f"safe-fallback({n_fb}/{len(actions)})"
    return plan


def _score_dict(sb: ScoreBreakdown) -> dict:
    return {"transport": sb.transport, "entropy": sb.entropy, "d1": sb.d1, "d2": sb.d2,
            "total": sb.total}


def domdec_solve(problem: TransportProblem, partitions: Decomposition,
                 strategy: StrategyConfig = StrategyConfig(), config: EngineConfig = EngineConfig(),
                 state: PlanState | None = None, evaluator: StitchedGapEvaluator | None = None):
    """Alternate composite partitions until the duality-gap certificate falls
    below lam * delta * |mu| or the iteration cap (engine.py:938-1037)."""
    if problem.mu.grid.ndim == 3:
        from .volume import domdec_solve3
        return domdec_solve3(problem, partitions, strategy, config, state, evaluator)
    if state is None:
        state = initial_plan_state(problem, partitions.basic)
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
            "strategy": strategy.kind,
            "leniency": strategy.leniency, "delta": config.delta}
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
            iteration_sequential(state, part, config, stats)
        else:
            iteration_parallel(state, part, strategy, config, stats)
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
        timings["assemble"] += stats.assemble_time
        timings["solve"] += stats.solve_time
        timings["score"] += stats.score_time
        timings["commit"] += stats.commit_time
        for key in ("balance_fallbacks", "safe_fallbacks", "nonconverged_cells",
                    "nu_minus_clamped", "nu_j_drift_nodes"):
            diag[key] += getattr(stats, key)
        diag["cell_iterations"] += stats.cell_iterations
        diag["cell_flops"] += stats.cell_flops
        diag["newton_clamped"] = max(diag["newton_clamped"], stats.newton_clamped)
        diag["balance_target_miss"] = max(diag["balance_target_miss"], stats.balance_target_miss)
        if last_gap / lam <= config.delta * mu_total:
            converged = True
            break
    if _SHARD is not None and _SHARD.world > 1:
        _SHARD.replicate(state)     # the whole plan current on every rank again
    timings["total"] = time.perf_counter() - t_all
    diag["truncated_mass"] = state.truncated_mass
    report = SolveReport(converged=converged, iterations=len(trace), final_score=_score_dict(sb),
                         rel_pd_gap=last_gap / max(abs(sb.total), 1e-300), x_err=stats.x_err,
                         y_err=stats.y_err, trace=trace, timings=timings,
                         sparsity=state.sparsity(), diagnostics=diag)
    return state, report
