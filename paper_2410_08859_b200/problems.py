"""Seeded synthetic problem generators for the BASELINE.json configurations.

The reference benchmarks on Gaussian-mixture images (paper §4.3.1, "Gaussian
mixtures supported on X = [0,1]^2 with random variances, means, and
magnitudes"); no image files travel, so every config is regenerated from a
seed.  The generator is host-side setup used by bench.py (both arms), the
BASELINE-config parity tests and the configs[0] golden fixture
(scripts/make_golden.py ``pr1_64``), so those comparisons see bit-identical
inputs.  The small hand-made golden cases (toy1d_*, mix16_*, mix32_*) use
make_golden.py's own mixture helper instead.

Density recipe (documented in DESIGN.md §Data):
    dens = sum_k w_k exp(-|x - c_k|^2 / (2 sigma_k^2))      (isotropic)
    dens = dens / dens.sum() + floor                         (floor per pixel)
    mass = total * dens / dens.sum()
with c_k ~ U[0.2, 0.8]^d, sigma_k ~ U[0.05, 0.15], w_k ~ U[0.5, 1].
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["MixtureSpec", "gaussian_mixture", "BASELINE_CONFIGS", "config_problem_arrays"]


@dataclass(frozen=True)
class MixtureSpec:
    n_bumps: int
    floor: float
    total: float
    centre_lo: float = 0.2
    centre_hi: float = 0.8
    sigma_lo: float = 0.05
    sigma_hi: float = 0.15
    w_lo: float = 0.5
    w_hi: float = 1.0
    anisotropic: bool = False   # one sigma per axis (BASELINE configs[4]) instead of one per bump


def gaussian_mixture(dims: tuple, dx: float, origin: tuple, spec: MixtureSpec,
                     rng: np.random.Generator) -> np.ndarray:
    """Floored, normalised Gaussian mixture (isotropic, or diagonal with
    ``spec.anisotropic``) on a regular grid."""
    d = len(dims)
    axes = [origin[a] + dx * np.arange(dims[a], dtype=np.float64) for a in range(d)]
    dens = np.zeros(dims, dtype=np.float64)
    for _ in range(spec.n_bumps):
        c = rng.uniform(spec.centre_lo, spec.centre_hi, size=d)
        if spec.anisotropic:
            sig = rng.uniform(spec.sigma_lo, spec.sigma_hi, size=d)
            w = rng.uniform(spec.w_lo, spec.w_hi)
            q = np.zeros(dims, dtype=np.float64)
            for a in range(d):
                shape = [1] * d
                shape[a] = dims[a]
                q = q + (((axes[a] - c[a]) ** 2) / (2.0 * sig[a] * sig[a])).reshape(shape)
            dens += w * np.exp(-q)
            continue
        sig = rng.uniform(spec.sigma_lo, spec.sigma_hi)
        w = rng.uniform(spec.w_lo, spec.w_hi)
        q = np.zeros(dims, dtype=np.float64)
        for a in range(d):
            shape = [1] * d
            shape[a] = dims[a]
            q = q + ((axes[a] - c[a]) ** 2).reshape(shape)
        dens += w * np.exp(-q / (2.0 * sig * sig))
    dens = dens / dens.sum() + spec.floor
    return dens * (spec.total / dens.sum())


# BASELINE.json "configs", index-aligned.  Only the fields the solver needs.
BASELINE_CONFIGS = [
    dict(name="pr1_64", n=64, mu=MixtureSpec(3, 1e-4, 1.0), nu=MixtureSpec(3, 1e-4, 1.3),
         lam=1.0, eps_final_h2=2.0, eps_start_h2=2.0, coarsest=64, cell=4, domdec_sweeps=30,
         inner_tol=1e-7),
    dict(name="ms_256", n=256, mu=MixtureSpec(5, 1e-4, 1.0), nu=MixtureSpec(5, 1e-4, 0.8),
         lam=0.5, eps_final_h2=2.0, eps_start_h2=64.0, coarsest=32, cell=4),
    dict(name="ms_1024", n=1024, mu=MixtureSpec(8, 1e-5, 1.0), nu=MixtureSpec(8, 1e-5, 1.5),
         lam=1.0, eps_final_h2=2.0, eps_start_h2=256.0, coarsest=64, cell=8),
    # configs[3] names only the final eps (2h^2) and the pyramid 128^2 -> 2048^2; the
    # ladder starts at the coarsest layer's 2 dx^2 = 2 (16 h)^2 = 512 h^2 (SPEC eps_schedule)
    dict(name="ms_2048", n=2048, mu=MixtureSpec(16, 1e-5, 1.0), nu=MixtureSpec(16, 1e-5, 0.7),
         lam=2.0, eps_final_h2=2.0, eps_start_h2=512.0, coarsest=128, cell=8),
    # configs[4]: 3D 128^3, 4 anisotropic Gaussians (diagonal sigma in [0.05, 0.2]) + 1e-5
    # floor, masses 1.0 / 1.2, lam 1, eps 32h^2 -> 2h^2, levels 16^3 -> 128^3, 4^3 cells
    dict(name="vol_128", n=128, dim=3,
         mu=MixtureSpec(4, 1e-5, 1.0, sigma_lo=0.05, sigma_hi=0.2, anisotropic=True),
         nu=MixtureSpec(4, 1e-5, 1.2, sigma_lo=0.05, sigma_hi=0.2, anisotropic=True),
         lam=1.0, eps_final_h2=2.0, eps_start_h2=32.0, coarsest=16, cell=4),
]


def config_problem_arrays(index: int, seed: int = 0, n: int | None = None):
    """(mu, nu, dx, origin, cfg) for a BASELINE config; ``n`` overrides the size."""
    cfg = dict(BASELINE_CONFIGS[index])
    n = int(n or cfg["n"])
    dx = 1.0 / n
    d = int(cfg.get("dim", 2))
    origin = (0.5 * dx,) * d
    rng = np.random.default_rng(seed)
    mu = gaussian_mixture((n,) * d, dx, origin, cfg["mu"], rng)
    nu = gaussian_mixture((n,) * d, dx, origin, cfg["nu"], rng)
    cfg["n"] = n
    return mu, nu, dx, origin, cfg
