"""Compare one batch solved by the cluster kernel against the single-CTA kernel."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, warnings
import paper_2410_08859_b200.engine as E
from paper_2410_08859_b200.decomposition import make_decomposition
from _golden import load
from _engine_run import problem_from_golden
g = load(sys.argv[1] if len(sys.argv) > 1 else "mix16_staggered")
prob = problem_from_golden(g)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    dec = make_decomposition(prob.mu, int(g["s"]))
out = {}
for mode in (0, 2):
    E._FORCE_CLUSTER = mode
    st = E.initial_plan_state(prob, dec.basic)
    pt = E._tables(dec.composites[0])
    snap = st.assemble_device()
    bt = E._Batch(st, pt, pt.batches[0], snap, E.EngineConfig(delta=float(g["delta"])).cell_config())
    print("mode", mode, "n_clu", bt.n_clu, "groups", [(C, len(sel)) for C, sel, _ in bt.clu_groups], "n_big", bt.n_big, "smem", bt.batch.smem_mode)
    bt.solve()
    torch.cuda.synchronize()
    c1, c2 = bt.stats()
    nx = pt.nw0 * pt.nw1
    out[mode] = dict(c1=c1.copy(), alpha=bt.alpha[:bt.n * nx].cpu().numpy().copy(),
                     beta=bt.beta[:int(bt.ny.sum())].cpu().numpy().copy(),
                     lout=bt.lout[:bt.n * nx].cpu().numpy().copy(),
                     mstat=bt.mstat[:int(bt.nmem.sum()) * 4].cpu().numpy().copy())
a, b = out[0], out[2]
print("iters", a["c1"][:, 2], b["c1"][:, 2])
print("gap", a["c1"][:, 0], b["c1"][:, 0])
print("first_gap", a["c1"][:, 1], b["c1"][:, 1])
print("alpha maxdiff", np.abs(a["alpha"] - b["alpha"]).max(), "beta maxdiff", np.abs(a["beta"] - b["beta"]).max())
print("mstat", np.abs(a["mstat"] - b["mstat"]).max())
