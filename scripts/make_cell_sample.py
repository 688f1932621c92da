"""Record the CPU-baseline cell sample of the ms_1024 workload (run on a GPU box).

The SPEC multiscale driver solves BASELINE configs[2] (1024^2) on the GPU; at
the start of the 1024^2 stage the first staggered batch of partition A is
windowed exactly as the reference's make_cell_problems does (the oracle's
``prepare`` on the device state), and every 16th composite cell of that batch
is saved with its complete subproblem inputs (X/Y windows, mu, nu, background
density, warm duals, member rows and masses, coordinates).  The file also
records the GPU's iteration count for each saved cell at the full cap and the
algorithmic cell-sweep work of one whole converged solve, so the bench can put
the CPU sample next to the full workload.

    python scripts/make_cell_sample.py        # writes tests/golden/ms1024_cells.npz
"""
import os
import sys
import warnings
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from test_gpu_baseline_parity import _capture_1024_stage
    from paper_2410_08859_b200.engine import CellSolverConfig, _Batch, _tables, cell_lse_flops
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.multiscale import multiscale_solve
    from oracle.ref_cell import prepare
    from oracle.ref_problem import make_ctx

    cap, mu, nu, dx, org, cfg = _capture_1024_stage()
    st, prob, dec = cap["state"], cap["problem"], cap["dec"]
    part = dec.composites[0]
    pt = _tables(part)
    ids = np.asarray(pt.batches[0])
    delta = 2e-5 * 0.25
    snap = st.assemble_device()
    boxes = [tuple(int(x) for x in b) for b in st.ybox.view(-1, 4).cpu().numpy()]
    vals_all = st.yval.view(st.n_basic, st.cap).cpu().numpy()
    duals = {}
    for (label, j), d in st.duals.items():
        if label == part.label:
            b = [c for ax in d.beta_box for c in ax]
            duals[(label, j)] = (d.alpha.copy(), tuple(int(x) for x in b), d.beta.copy())
    snap_h = snap.cpu().numpy().reshape(nu.shape)
    bt = _Batch(st, pt, ids, snap, CellSolverConfig(delta=delta))
    bt.solve()
    c1, _ = bt.stats()
    torch.cuda.synchronize()
    ctx = make_ctx(mu, nu, dx, org, cfg["lam"], prob.eps, cfg["cell"])
    opart = [p for p in ctx.parts if p["label"] == part.label][0]
    vals = [vals_all[i, :b[1] * b[3]].reshape(b[1], b[3]) if b[1] and b[3] else np.zeros((0, 0))
            for i, b in enumerate(boxes)]
    ost = SimpleNamespace(box=[b if b[1] and b[3] else (0, 0, 0, 0) for b in boxes], vals=vals,
                          duals=duals)
    sel = np.arange(0, len(ids), 16)
    probs = prepare(ctx, opart, [int(ids[k]) for k in sel], ost, snap_h)
    out = {}
    for q, (k, p) in enumerate(zip(sel, probs)):
        pre = f"c{q}_"
        out[pre + "j"] = p.j
        out[pre + "xbox"] = np.array(p.xbox)
        out[pre + "ybox"] = np.array(p.ybox)
        out[pre + "mu_win"] = p.mu_win
        out[pre + "nu_win"] = p.nu_win
        out[pre + "m_win"] = p.m_win if p.m_win is not None else np.zeros(0)
        out[pre + "alpha0"] = p.alpha0
        out[pre + "beta0"] = p.beta0
        out[pre + "members"] = np.array(p.members)
        out[pre + "rows"] = np.stack(p.rows)
        out[pre + "masses"] = p.masses
        out[pre + "xc0"], out[pre + "xc1"] = p.xc
        out[pre + "yc0"], out[pre + "yc1"] = p.yc
        out[pre + "gpu_iters"] = int(c1[k, 2])
    # work of one complete converged solve (GPU run, same protocol as the bench)
    h2 = dx * dx
    grid = Grid(mu.shape, dx, org)
    fprob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu),
                             DivergenceSpec(cfg["lam"]), 2 * h2)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, rep = multiscale_solve(fprob, cfg["cell"], cfg["coarsest"], cfg["eps_start_h2"] * h2)
    full_flops = sum(r.diagnostics.get("cell_flops", 0.0) for _, _, r in rep.stages)
    full_iters = sum(r.diagnostics.get("cell_iterations", 0) for _, _, r in rep.stages)
    batch_flops = float((c1[:, 2] * cell_lse_flops(pt.nw0, pt.nw1, bt.ybox[:, 1].astype(float),
                                                    bt.ybox[:, 3].astype(float))).sum())
    out.update(n_cells=len(sel), eps=prob.eps, lam=cfg["lam"], nu_total=float(nu.sum()),
               delta=delta, nw0=pt.nw0, nw1=pt.nw1, batch_cells=len(ids),
               full_solve_cell_flops=full_flops, full_solve_cell_iterations=full_iters,
               batch_cell_flops=batch_flops, converged=rep.converged)
    path = os.path.join(ROOT, "tests", "golden", "ms1024_cells.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes;", len(sel), "cells; gpu iters",
          [int(c1[k, 2]) for k in sel][:16], "full flops", full_flops)


if __name__ == "__main__":
    main()
