"""Probe: single-CTA vs 2-CTA-cluster cell solves on the first 1024^2 batch at the full
cap (10000 iterations): iteration counts and duals must agree to rounding."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from test_gpu_baseline_parity import _capture_1024_stage
    from paper_2410_08859_b200.engine import CellSolverConfig, _Batch, _tables, set_exec_mode

    cap, mu, nu, dx, org, cfg = _capture_1024_stage()
    st, prob, dec = cap["state"], cap["problem"], cap["dec"]
    pt = _tables(dec.composites[0])
    ids = np.asarray(pt.batches[0])
    snap = st.assemble_device()
    ccfg = CellSolverConfig(delta=2e-5 * 0.25)
    res = {}
    for mode in ("default", "cluster2", "cluster4"):
        prev = set_exec_mode(force_cluster={"default": 0, "cluster2": 2, "cluster4": 4}[mode])
        try:
            bt = _Batch(st, pt, ids, snap, ccfg)
            bt.solve()
            torch.cuda.synchronize()
            c1, c2 = bt.stats()
            nx = pt.nw0 * pt.nw1
            res[mode] = (c1.copy(), c2.copy(), bt.alpha[:bt.n * nx].cpu().numpy().copy(),
                         bt.beta[:int(bt.ny.sum())].cpu().numpy().copy(), bt.ny.copy())
        finally:
            set_exec_mode(prev)
    c1d, c2d, ad, bd, ny = res["default"]
    print("cells", len(ids), "capped", int((c1d[:, 2] >= 10000).sum()))
    for mode in ("cluster2", "cluster4"):
        c1, c2, a, b, _ = res[mode]
        same_it = (c1[:, 2] == c1d[:, 2])
        print(mode, "iterations equal:", int(same_it.sum()), "/", len(same_it),
              "conv equal:", int((c1[:, 3] == c1d[:, 3]).sum()),
              "alpha rel", float(np.abs(a - ad).max() / np.abs(ad).max()),
              "beta rel", float(np.abs(b - bd).max() / np.abs(bd).max()))
        bad = np.flatnonzero(~same_it)[:10]
        for k in bad:
            print("   cell", k, "iters", int(c1d[k, 2]), int(c1[k, 2]), "ny", int(ny[k]),
                  "exec", int(c2d[k, 4]), int(c2[k, 4]))


if __name__ == "__main__":
    main()
