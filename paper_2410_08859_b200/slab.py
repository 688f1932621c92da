"""Row-slab domain sharding of the domdec solve over a torch.distributed group.

north_star layout: the basic-cell lattice is cut into contiguous slabs of block
rows, one per rank (1-8 GPUs, one process per GPU, NCCL over NVLink).  A
composite cell belongs to the rank whose slab holds its first block row, so
every rank solves and commits only its own composites.  Slab boundaries sit on
even block rows: partition A composites (block rows 2a, 2a+1) never straddle a
boundary, and a partition B composite (rows 2a-1, 2a, shifted by one block,
ref partitions.py:183-184) that straddles boundary R belongs to the rank below
it.  The basic cells of the boundary block row R therefore change owner between
an A sweep and the following B sweep: that row is the halo, and its state (Y
box, slot values, X-marginal, fragments) moves to the neighbour with one
point-to-point exchange per partition switch.  Dual stores never move: a
composite of a given partition always has the same owner.

Everything else a rank needs is global and reduced with collectives:

* the Y-marginal snapshot of every staggered batch: each rank assembles its own
  basic cells (``dd_assemble_masked``) and one dense all-reduce sums them;
* the staggered / swift decision: the rank-local parts of the blended energy
  (``dd_blend_parts``: sum_c theta_c dy_c on a dense Y grid plus per-cell
  pieces) are summed with one dense and one 3-scalar all-reduce;
* the energy: per-cell sums over owned basic cells (``dd_energy_terms_masked``)
  plus KL of the (already global) assembled Y-marginal;
* the certificate: each rank stitches alpha on its own composites' X blocks,
  one all-reduce builds the global alpha, the dual evaluation is replicated.

The global Sinkhorn layers, the warm start and the refinement run replicated
(identical, deterministic); at the end of a domdec solve the state is made
whole on every rank again (``replicate``), so the solver API returns the full
plan everywhere.  The weight strategies that need per-cell global coordination
inside a batch (opt) and the sequential sweep are single-rank only.
"""

from __future__ import annotations

import numpy as np

__all__ = ["ShardSpec", "slab_bounds", "composite_owners", "basic_owners", "halo_sets"]


def slab_bounds(n_rows: int, world: int) -> np.ndarray:
    """Block-row boundaries R_0 = 0 < ... < R_world = n_rows, interior ones even."""
    b = [0]
    for r in range(1, world):
        x = int(round(r * n_rows / world / 2.0)) * 2
        b.append(min(max(x, b[-1]), n_rows))
    b.append(n_rows)
    return np.asarray(b, dtype=np.int64)


def composite_owners(first_rows: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    """Owner rank of each composite from its first block row (clamped onto the lattice)."""
    n_rows = int(bounds[-1])
    r = np.clip(np.asarray(first_rows, dtype=np.int64), 0, max(n_rows - 1, 0))
    return (np.searchsorted(bounds, r, side="right") - 1).astype(np.int64)


def basic_owners(members: np.ndarray, nmem: np.ndarray, comp_owner: np.ndarray,
                 n_basic: int) -> np.ndarray:
    """Owner of each basic cell under one partition (the owner of its composite)."""
    own = np.full(n_basic, -1, dtype=np.int64)
    for j in range(len(nmem)):
        m = members[j, :nmem[j]]
        own[m[m >= 0]] = comp_owner[j]
    return own


def _box_width(plan) -> int:
    """4 for the 2D path's boxes, 6 for the three-axis path's."""
    return 6 if getattr(plan, "box_width", 4) == 6 else 4


def _box_sizes(b: np.ndarray) -> np.ndarray:
    """Entries of each box row (o0, e0, o1, e1[, o2, e2])."""
    b = np.asarray(b, dtype=np.int64).reshape(len(b), -1)
    n = b[:, 1] * b[:, 3]
    return n * b[:, 5] if b.shape[1] == 6 else n


def halo_sets(prev_owner: np.ndarray, new_owner: np.ndarray, rank: int):
    """Basic cells this rank sends ({peer: ids}) and receives ({peer: ids})."""
    send, recv = {}, {}
    moved = prev_owner != new_owner
    for q in np.unique(new_owner[moved & (prev_owner == rank)]):
        send[int(q)] = np.flatnonzero(moved & (prev_owner == rank) & (new_owner == q))
    for r in np.unique(prev_owner[moved & (new_owner == rank)]):
        recv[int(r)] = np.flatnonzero(moved & (new_owner == rank) & (prev_owner == r))
    return send, recv


class ShardSpec:
    """Slab ownership and the collectives of a sharded domdec solve."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self._cache: dict = {}
        self.bytes_exchanged = 0      # halo + replicate payload sent by this rank

    # ---- collectives (NCCL on the device; gloo through host memory)
    def _global(self, r: int) -> int:
        import torch.distributed as dist
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def all_reduce(self, t, op: str = "sum") -> None:
        import torch.distributed as dist

        rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
        if self.nccl or t.device.type == "cpu":
            dist.all_reduce(t, op=rop, group=self.group)
        else:
            c = t.cpu()
            dist.all_reduce(c, op=rop, group=self.group)
            t.copy_(c)

    all_reduce_sum = all_reduce

    def reduce_np(self, arr, op: str = "sum", device=None) -> np.ndarray:
        """All-reduce a small host vector (returns the reduced copy)."""
        import torch

        t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64))
        if self.nccl:
            t = t.to(device or "cuda")
        self.all_reduce(t, op)
        return t.cpu().numpy()

    def _p2p(self, sends: dict, recvs: dict) -> dict:
        """Exchange tensors: sends {peer: tensor}, recvs {peer: preallocated tensor}."""
        import torch.distributed as dist

        if not sends and not recvs:
            return recvs
        host = not self.nccl
        ops, staged = [], {}
        for q, t in sorted(sends.items()):
            tt = t.cpu() if host else t.contiguous()
            ops.append(dist.P2POp(dist.isend, tt, self._global(q), group=self.group))
            self.bytes_exchanged += tt.numel() * tt.element_size()
        for r, t in sorted(recvs.items()):
            tt = t.cpu() if host else t
            staged[r] = tt
            ops.append(dist.P2POp(dist.irecv, tt, self._global(r), group=self.group))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if host:
            for r, t in recvs.items():
                t.copy_(staged[r])
        return recvs

    # ---- slab geometry
    def layout(self, pt, block: tuple, n_basic: int, lattice_rows: int, lattice_cols: int):
        """(composite owner, basic-cell owner) of one partition table (cached)."""
        key = (id(pt), n_basic)
        hit = self._cache.get(key)
        if hit is not None and hit[0] is pt:
            return hit[1], hit[2]
        axis = 0 if lattice_rows >= 2 * self.world or lattice_cols < 2 * self.world else 1
        n_rows = lattice_rows if axis == 0 else lattice_cols
        blk = block[0] if axis == 0 else block[1]
        off = pt.xbox[:, 0] if axis == 0 else pt.xbox[:, 2]
        first = np.floor_divide(off, blk)
        bounds = slab_bounds(n_rows, self.world)
        comp = composite_owners(first, bounds)
        basic = basic_owners(pt.mem, pt.nmem, comp, n_basic)
        self._cache[key] = (pt, comp, basic)
        return comp, basic

    # ---- state movement
    def exchange_cells(self, plan, send: dict, recv: dict) -> None:
        """Move whole basic-cell states (box, values, X-marginal, fragments)."""
        import torch

        dev = plan.ybox.device
        bw = _box_width(plan)
        boxes = plan.ybox.view(-1, bw)
        sb = {q: boxes[torch.as_tensor(ids, device=dev)].clone() for q, ids in send.items()}
        rb = {r: torch.empty((len(ids), bw), dtype=torch.int32, device=dev)
              for r, ids in recv.items()}
        self._p2p(sb, rb)
        need = 1
        for r, ids in recv.items():
            b = rb[r].cpu().numpy()
            need = max(need, int(_box_sizes(b).max(initial=1)))
        plan.ensure_cap(need)
        bs = plan.bs
        vals = plan.yval.view(plan.n_basic, plan.cap)
        xm = plan.x_marg_d.view(plan.n_basic, bs)

        def pack(ids, bx):
            parts = []
            for i, k in zip(ids, _box_sizes(bx)):
                parts.append(vals[int(i), :int(k)])
                parts.append(xm[int(i)])
            t = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.float64, device=dev)
            frag = torch.stack([plan.transport_d[torch.as_tensor(ids, device=dev)],
                                plan.kl_d[torch.as_tensor(ids, device=dev)]], 1).reshape(-1)
            return torch.cat([t, frag])

        sp = {q: pack(ids, sb[q].cpu().numpy()) for q, ids in send.items()}
        rp = {}
        for r, ids in recv.items():
            b = rb[r].cpu().numpy()
            n = int(_box_sizes(b).sum()) + len(ids) * bs + 2 * len(ids)
            rp[r] = torch.empty(n, dtype=torch.float64, device=dev)
        self._p2p(sp, rp)
        for r, ids in recv.items():
            b = rb[r].cpu().numpy()
            buf, o = rp[r], 0
            for i, k in zip(ids, _box_sizes(b)):
                k = int(k)
                vals[int(i), :k] = buf[o:o + k]
                o += k
                xm[int(i)] = buf[o:o + bs]
                o += bs
            fr = buf[o:].view(-1, 2)
            idx = torch.as_tensor(ids, device=dev)
            plan.transport_d[idx] = fr[:, 0]
            plan.kl_d[idx] = fr[:, 1]
            boxes[idx] = rb[r]
            plan.ybox_h[ids] = b

    def halo_exchange(self, plan, new_owner: np.ndarray) -> None:
        """Before a partition sweep: receive the basic cells this rank now owns."""
        prev = plan.owner
        if prev is not None:
            send, recv = halo_sets(prev, new_owner, self.rank)
            self.exchange_cells(plan, send, recv)
        plan.set_owner(new_owner)

    def replicate(self, plan) -> None:
        """Make the whole state current on every rank (end of a sharded solve):
        basic-cell states from their owners, and every partition's dual store
        (each composite's entry from its owner: rows of other owners are zeroed
        and the stores summed, which is exact)."""
        import torch

        for label, store in plan.stores.items():
            comp = plan.comp_owner.get(label)
            if comp is None:
                continue
            dcap = int(self.reduce_np([store.dcap], "max", plan.ybox.device)[0])
            store.resize(dcap)        # the same size on every rank before the sums
            keep = torch.from_numpy(comp == self.rank).to(store.alpha.device)
            a = store.alpha.view(store.ncomp, store.nx)
            bt = store.beta.view(store.ncomp, store.dcap)
            a.mul_(keep[:, None].to(a.dtype))
            bt.mul_(keep[:, None].to(bt.dtype))
            store.has.mul_(keep.to(store.has.dtype))
            store.box.view(store.ncomp, -1).mul_(keep[:, None].to(store.box.dtype))
            for t in (store.alpha, store.beta, store.has, store.box):
                self.all_reduce(t)
        own = plan.owner
        if own is None:
            return
        for src in range(self.world):
            ids = np.flatnonzero(own == src)
            send = {q: ids for q in range(self.world) if q != src} if self.rank == src else {}
            recv = {src: ids} if self.rank != src else {}
            self.exchange_cells(plan, send, recv)
        plan.set_owner(None)
