"""Cell-sharded solve over 2 ranks (gloo, both on cuda:0) equals the reference fixtures.

The ranks exchange data only through host-side gloo collectives; no kernel
waits on another rank.  Sharding is exact (owned cells write, others are
zero, arenas are summed), so both ranks must reproduce the single-GPU
parity bounds and agree with each other bitwise.
"""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_08859_b200.engine import set_shard
    from _engine_run import run_device
    from _golden import load
    set_shard()
    g = load(name)
    prob, dec, st, rep = run_device(g)
    vals = st.yval.view(st.n_basic, st.cap).cpu().numpy()
    q.put((rank, rep.iterations, [r.total for r in rep.trace], st.ybox.cpu().numpy().tolist(),
           float(vals.sum()), float(g["score"][-1]), int(g["iterations"]),
           [float(t) for t in g["trace_total"]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["mix16_staggered", "mix32_staggered", "toy1d_swift"])
def test_sharded_solve_matches_reference(name):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, it0, tr0, bx0, v0, ref_total, ref_iters, ref_trace), (_, it1, tr1, bx1, v1, *_rest) = out
    assert it0 == it1 == ref_iters
    assert tr0 == tr1                      # ranks agree bitwise
    assert bx0 == bx1 and v0 == v1
    np.testing.assert_allclose(tr0, ref_trace, rtol=1e-10)
