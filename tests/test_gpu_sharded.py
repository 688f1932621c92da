"""Row-slab sharded solve over 2 ranks (gloo, both on cuda:0) against the reference.

Each rank solves and commits the composites of its slab; the Y-marginal
snapshot and the blend energies are summed over the ranks, the boundary
block row's basic cells move between the ranks at every A/B switch (halo
exchange) and the plan is made whole again at the end (slab.py).  The ranks
exchange data only through host-side gloo collectives / point-to-point
messages; no kernel waits on another rank.  Both ranks must reproduce the
reference's iteration counts, actions and scores within the fp64 tolerances,
and hold identical final plans.
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
    from _golden import dense, ref_marginals, rel_err
    from _engine_run import box4
    shape = prob.nu.mass.reshape(1, -1).shape if prob.nu.grid.ndim == 1 else prob.nu.mass.shape
    nu_i = st.nu_i
    worst = 0.0
    for i, (box, v) in enumerate(ref_marginals(g)):
        b = box4(nu_i[i].box)
        mine = dense(b, nu_i[i].values.reshape(b[1], b[3]) if b[1] else np.zeros((0, 0)), shape)
        worst = max(worst, rel_err(mine, dense(box, v, shape)))
    vals = st.yval.view(st.n_basic, st.cap).cpu().numpy()
    sizes = (st.ybox.view(-1, 4).cpu().numpy()[:, 1] * st.ybox.view(-1, 4).cpu().numpy()[:, 3])
    vsum = float(sum(vals[i, :sizes[i]].sum() for i in range(st.n_basic)))
    q.put((rank, rep.iterations, [r.total for r in rep.trace], st.ybox.cpu().numpy().tolist(),
           vsum, float(g["score"][-1]), int(g["iterations"]),
           [float(t) for t in g["trace_total"]], [r.action for r in rep.trace],
           [str(a) for a in g["trace_action"]], worst))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["mix16_staggered", "mix32_staggered", "mix16_warm",
                                  "toy1d_staggered", "toy1d_swift", "mix16_zeros"])
def test_slab_sharded_solve_matches_reference(name):
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
    r0, r1 = out
    (_, it0, tr0, bx0, v0, ref_total, ref_iters, ref_trace, act0, ref_act, w0) = r0
    (_, it1, tr1, bx1, v1, _, _, _, act1, _, w1) = r1
    assert it0 == it1 == ref_iters
    assert act0 == act1 == ref_act
    assert tr0 == tr1                      # both ranks run the same reductions
    assert bx0 == bx1 and v0 == v1         # the replicated plan is identical everywhere
    np.testing.assert_allclose(tr0, ref_trace, rtol=1e-10)
    assert w0 < 1e-9 and w1 < 1e-9         # basic-cell marginals vs the reference
