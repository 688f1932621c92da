"""z-slab sharded three-axis solve over 2 ranks (gloo, both on cuda:0) against the reference.

The three-axis path under ``engine.set_shard()``: each rank solves and commits the
composites of its slab of the first real axis (z for 3D, configs[4]); snapshots,
blend energies, residuals and the stitched alpha are reduced over the ranks and the
boundary layer's basic cells move at every A/B switch (slab.py).  The ranks exchange
data only through host-side gloo collectives / point-to-point messages; no kernel
waits on another rank.  Both ranks must reproduce the reference's iterations,
actions, scores and marginals, and hold identical final plans.
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
    from _golden import load, rel_err
    from test_gpu_volume import _box6, _dense, _run
    set_shard()
    g = load(name)
    prob, st, rep = _run(g)
    shape3 = st.dp.shape_y
    nu_i = st.nu_i
    offs = g["nu_i_off"]
    worst = 0.0
    for i, rb in enumerate(g["nu_i_box"]):
        wb = _box6(rb)
        mb = _box6([c for ax in nu_i[i].box for c in ax])
        if mb != wb:
            worst = float("inf")
            continue
        worst = max(worst, rel_err(_dense(mb, nu_i[i].values, shape3),
                                   _dense(wb, g["nu_i_val"][offs[i]:offs[i + 1]], shape3)))
    vals = st.yval.view(st.n_basic, st.cap).cpu().numpy()
    b = st.ybox.view(-1, 6).cpu().numpy().astype(np.int64)
    sizes = b[:, 1] * b[:, 3] * b[:, 5]
    vsum = float(sum(vals[i, :sizes[i]].sum() for i in range(st.n_basic)))
    q.put((rank, rep.iterations, [r.total for r in rep.trace], b.tolist(), vsum,
           int(g["iterations"]), [float(t) for t in g["trace_total"]],
           [r.action for r in rep.trace], [str(a) for a in g["trace_action"]], worst))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["vol8_staggered", "vol16_cold", "vol32_warm", "mix16_staggered",
                                  "toy1d_staggered"])
def test_zslab_sharded_volume_solve_matches_reference(name):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0, r1 = out
    (_, it0, tr0, bx0, v0, ref_iters, ref_trace, act0, ref_act, w0) = r0
    (_, it1, tr1, bx1, v1, _, _, act1, _, w1) = r1
    assert it0 == it1 == ref_iters
    assert act0 == act1 == ref_act
    assert tr0 == tr1                      # both ranks run the same reductions
    assert bx0 == bx1 and v0 == v1         # the replicated plan is identical everywhere
    np.testing.assert_allclose(tr0, ref_trace, rtol=1e-10)
    assert w0 < 1e-9 and w1 < 1e-9         # basic-cell marginals vs the reference
