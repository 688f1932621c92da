"""Golden-fixture loading shared by the oracle (CPU) and parity (GPU) tests."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

ENGINE_CASES = ["toy1d_staggered", "toy1d_safe", "toy1d_swift", "toy1d_opt", "toy1d_sequential",
                "toy1d_fast", "mix16_staggered", "mix16_warm", "mix32_staggered", "mix16_cellcap",
                "toy1d_cellcap_swift", "mix16_zeros", "mix16_zeros_warm_opt"]


def cell_cap(g) -> int:
    return int(g["cell_max_iters"]) if "cell_max_iters" in g else 10_000


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as f:
        return {k: f[k] for k in f.files}


def scalar(g, k):
    v = g[k]
    return v.item() if hasattr(v, "item") else v


def ref_marginals(g):
    """[(box (o0,e0,o1,e1), values 2D)] per basic cell."""
    out = []
    for i, b in enumerate(g["nu_i_box"]):
        lo, hi = g["nu_i_off"][i], g["nu_i_off"][i + 1]
        b = tuple(int(x) for x in b)
        out.append((b, g["nu_i_val"][lo:hi].reshape(b[1], b[3]) if hi > lo else np.zeros((0, 0))))
    return out


def ref_duals(g):
    out = {}
    for k, key in enumerate(g["dual_keys"]):
        label, j = str(key).split(":")
        a = g["dual_alpha"][g["dual_alpha_off"][k]:g["dual_alpha_off"][k + 1]]
        b = g["dual_beta"][g["dual_beta_off"][k]:g["dual_beta_off"][k + 1]]
        out[(label, int(j))] = (a, tuple(int(x) for x in g["dual_beta_box"][k]), b)
    return out


def dense(box, vals, shape):
    out = np.zeros(shape)
    if box[1] and box[3]:
        out[box[0]:box[0] + box[1], box[2]:box[2] + box[3]] = vals.reshape(box[1], box[3])
    return out


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0
