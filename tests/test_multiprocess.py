"""World-size-2 gloo run of the bench's replica path host logic (CPU).

Round 1 runs N independent replicas (DESIGN.md §(e)); the only cross-rank
step is the max-over-ranks of the device time, exercised here over gloo.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2410_08859_b200.multiscale import build_pyramid, eps_schedule
    prob, cfg, eps_start = bench.problem("ms_256", seed=rank)
    levels = build_pyramid(prob.mu, prob.nu, cfg["coarsest"])
    sched = eps_schedule(levels, eps_start, prob.eps)
    t = bench.max_over_ranks(1.0 + rank)
    q.put((rank, t, len(levels), sum(len(r) for r in sched)))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_reduction_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == [2.0, 2.0]
    assert out[0][2:] == out[1][2:] == (4, 6)


class _FakePlan:
    """Host stand-in for PlanState's per-basic-cell arrays (what the slab layer moves)."""

    def __init__(self, n_basic, bs, cap):
        self.n_basic, self.bs, self.cap = n_basic, bs, cap
        self.ybox = torch.zeros(n_basic * 4, dtype=torch.int32)
        self.yval = torch.zeros(n_basic * cap, dtype=torch.float64)
        self.x_marg_d = torch.zeros(n_basic * bs, dtype=torch.float64)
        self.transport_d = torch.zeros(n_basic, dtype=torch.float64)
        self.kl_d = torch.zeros(n_basic, dtype=torch.float64)
        self.ybox_h = self.ybox.view(-1, 4).numpy().copy()
        self.owner = None
        self.stores, self.comp_owner = {}, {}

    def ensure_cap(self, need):
        if need <= self.cap:
            return
        nv = torch.zeros(self.n_basic * need, dtype=torch.float64)
        nv.view(self.n_basic, need)[:, :self.cap] = self.yval.view(self.n_basic, self.cap)
        self.yval, self.cap = nv, need

    def set_owner(self, owner):
        self.owner = None if owner is None else owner.copy()


def _cell_state(i, gen):
    """Deterministic per-(cell, generation) content: box extents vary with i."""
    e0, e1 = 1 + i % 3, 2 + i % 4
    box = np.array([i % 7, e0, i % 5, e1], dtype=np.int32)
    vals = np.arange(e0 * e1, dtype=np.float64) + 1000.0 * i + 0.5 * gen
    return box, vals


def _write(plan, ids, gen):
    bs = plan.bs
    for i in ids:
        box, vals = _cell_state(int(i), gen)
        plan.ensure_cap(len(vals))
        plan.ybox.view(-1, 4)[int(i)] = torch.from_numpy(box)
        plan.yval.view(plan.n_basic, plan.cap)[int(i), :len(vals)] = torch.from_numpy(vals)
        plan.x_marg_d.view(plan.n_basic, bs)[int(i)] = float(i) + gen
        plan.transport_d[int(i)] = 2.0 * i + gen
        plan.kl_d[int(i)] = 3.0 * i + gen
        plan.ybox_h[int(i)] = box


def _check(plan, ids, gen):
    bs = plan.bs
    for i in ids:
        box, vals = _cell_state(int(i), gen)
        assert np.array_equal(plan.ybox.view(-1, 4)[int(i)].numpy(), box), i
        got = plan.yval.view(plan.n_basic, plan.cap)[int(i), :len(vals)].numpy()
        assert np.array_equal(got, vals), i
        assert np.all(plan.x_marg_d.view(plan.n_basic, bs)[int(i)].numpy() == float(i) + gen)
        assert float(plan.transport_d[int(i)]) == 2.0 * i + gen
        assert float(plan.kl_d[int(i)]) == 3.0 * i + gen
        assert np.array_equal(plan.ybox_h[int(i)], box)


def _slab_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import warnings
    import numpy as np
    from paper_2410_08859_b200 import Grid, GridMeasure, make_decomposition
    from paper_2410_08859_b200.engine import _tables
    from paper_2410_08859_b200.slab import ShardSpec, halo_sets

    n, s_ = 64, 4
    g = Grid((n, n), 1.0 / n, (0.5 / n, 0.5 / n))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dec = make_decomposition(GridMeasure(g, np.ones((n, n))), s_)
    sp = ShardSpec()
    nb = dec.basic.n_cells
    lat = dec.basic.lattice_to_cell.shape
    pa, pb = (_tables(p) for p in dec.composites)
    ca, ba = sp.layout(pa, (s_, s_), nb, lat[0], lat[1])
    cb, bb = sp.layout(pb, (s_, s_), nb, lat[0], lat[1])
    rows = dec.basic.positions[:, 0]
    # owned rows are contiguous slabs; A and B ownership differ exactly on the
    # boundary block rows (the halo)
    diff_rows = sorted(set(rows[ba != bb].tolist()))
    send, recv = halo_sets(ba, bb, rank)
    plan = _FakePlan(nb, s_ * s_, 4)
    # generation 0: everything valid (replicated start); the A sweep updates owned cells
    _write(plan, np.arange(nb), 0)
    plan.set_owner(None)
    sp.halo_exchange(plan, ba)
    _write(plan, np.flatnonzero(ba == rank), 1)            # this rank's A sweep
    sp.halo_exchange(plan, bb)                              # switch to B: halo arrives
    _check(plan, np.flatnonzero(bb == rank), 1)
    _write(plan, np.flatnonzero(bb == rank), 2)            # this rank's B sweep
    sp.replicate(plan)                                      # whole plan on every rank
    _check(plan, np.arange(nb), 2)
    q.put((rank, ca.tolist(), cb.tolist(), diff_rows,
           {k: v.tolist() for k, v in send.items()}, {k: v.tolist() for k, v in recv.items()},
           [int(r) for r in rows[ba == rank].min(initial=-1).reshape(-1)],
           sp.bytes_exchanged))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_layout_halo_exchange_gloo_world2():
    """Row slabs over 2 ranks (gloo, CPU): composite ownership, the boundary block
    row as the only halo between A and B, and the halo exchange / replicate moving
    whole basic-cell states (box, values, X-marginal, fragments) exactly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = out
    assert r0[1] == r1[1] and r0[2] == r1[2]        # same layout on every rank
    assert set(r0[1]) == {0, 1} and set(r0[2]) == {0, 1}
    assert r0[3] == [8]                              # 16 block rows -> boundary row 8
    # rank 0 hands row 8 to rank 1?  No: B composites on rows (7, 8) stay with rank 0,
    # so rank 1 sends its row-8 cells to rank 0 at the A -> B switch
    assert not r0[4] and len(r0[5][1]) == 16 and len(r1[4][0]) == 16 and not r1[5]
    assert r0[7] > 0 and r1[7] > 0
