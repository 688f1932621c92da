"""World-size-2 gloo run of the bench's replica path host logic (CPU).

Round 1 runs N independent replicas (DESIGN.md §(e)); the only cross-rank
step is the max-over-ranks of the device time, exercised here over gloo.
"""

import os
import socket

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


def _owner_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    from paper_2410_08859_b200.engine import ShardSpec
    sp = ShardSpec()
    cost = np.random.default_rng(0).uniform(1, 100, 257)
    own = sp.owners(cost)
    t = torch.zeros(257, dtype=torch.float64)
    t[torch.from_numpy(own == rank)] = 1.0
    sp.all_reduce_sum(t)     # every cell owned exactly once across ranks
    loads = [float(cost[own == r].sum()) for r in range(world)]
    q.put((rank, own.tolist(), bool((t == 1.0).all()), max(loads) / min(loads)))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ownership_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_owner_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] == out[1][1]          # identical assignment on every rank
    assert out[0][2] and out[1][2]         # exact cover
    assert out[0][3] < 1.05                # balanced
