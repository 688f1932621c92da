"""Oracle kernels: log-sum-exp sweeps, the Newton Y-step, the global solve.

Restates /root/reference/pkg/src/domdec/sinkhorn.py (numpy, CPU, test-only):
  _lse :57, DenseKernel :91-130, SeparableKernel :133-175 (+ its three-axis
  extension GridKernel3, the same pattern over one more axis),
  y_halfstep_newton :230-333, gap_kl_terms :336-351, sinkhorn_solve :361-432.
"""

from __future__ import annotations

import math

import numpy as np

DEGENERATE_BETA_SCALE = 700.0  # sinkhorn.py:54


def lse(v: np.ndarray, axis: int) -> np.ndarray:
    """Max-shifted log-sum-exp; an all -inf slice gives -inf (sinkhorn.py:57-67)."""
    m = np.max(v, axis=axis, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore"):
        return np.log(np.sum(np.exp(v - m), axis=axis)) + np.squeeze(m, axis=axis)


class WindowKernel:
    """Explicit -c/eps over stacked cell windows, shape (B, nx, ny) (sinkhorn.py:91-130).

    When every exponent stays above -700 the kernel matrix is exponentiated
    once and a sweep is one shifted exponential of the dual vector plus a
    matrix product; otherwise the sweep is the fully shifted log-domain sum.
    """

    def __init__(self, negc: np.ndarray):
        self.negc = negc
        self.mat = np.exp(negc) if negc.min() > -700.0 else None

    @staticmethod
    def _shift(v):
        m = np.max(v, axis=-1, keepdims=True)
        m = np.where(np.isfinite(m), m, 0.0)
        return np.exp(v - m), m

    def lse_x(self, b: np.ndarray) -> np.ndarray:
        if self.mat is not None:
            w, m = self._shift(b)
            with np.errstate(divide="ignore"):
                return np.log(np.einsum("bxy,by->bx", self.mat, w)) + m
        return lse(b[:, None, :] + self.negc, axis=-1)

    def lse_y(self, a: np.ndarray) -> np.ndarray:
        if self.mat is not None:
            w, m = self._shift(a)
            with np.errstate(divide="ignore"):
                return np.log(np.einsum("bxy,bx->by", self.mat, w)) + m
        return lse(a[:, :, None] + self.negc, axis=-2)


class GridKernel:
    """Axis-separable sweeps over full 2D grids (sinkhorn.py:133-175).

    x_axes / y_axes: two coordinate arrays each (1D problems use a 1-node
    axis 0).  lse_x maps a Y-grid array to the X grid, lse_y the reverse.
    """

    def __init__(self, x_axes, y_axes, eps: float, chunk: int = 32):
        self.eps = float(eps)
        self.chunk = chunk
        self.t = [-np.subtract.outer(xa, ya) ** 2 / self.eps for xa, ya in zip(x_axes, y_axes)]

    def _sweep(self, v, t0, t1):
        m1 = v.shape[0]
        n1, n2 = t0.shape[0], t1.shape[0]
        mid = np.empty((m1, n2))
        for lo in range(0, m1, self.chunk):
            hi = min(lo + self.chunk, m1)
            mid[lo:hi] = lse(v[lo:hi, None, :] + t1[None, :, :], axis=2)
        out = np.empty((n1, n2))
        for lo in range(0, n1, self.chunk):
            hi = min(lo + self.chunk, n1)
            out[lo:hi] = lse(mid[None, :, :] + t0[lo:hi, :, None], axis=1)
        return out

    def lse_x(self, b):
        return self._sweep(np.asarray(b, dtype=np.float64), self.t[0], self.t[1])

    def lse_y(self, a):
        return self._sweep(np.asarray(a, dtype=np.float64), self.t[0].T, self.t[1].T)


class GridKernel3:
    """Axis-separable sweeps over full 3D grids: the reference's SeparableKernel._sweep
    (sinkhorn.py:159-175, two axes: last axis first, one _lse per axis) extended by one
    axis in the same pattern -- the sweep scripts/make_golden.py installs in the
    reference to produce the 3D fixtures."""

    def __init__(self, x_axes, y_axes, eps: float):
        self.eps = float(eps)
        self.t = [-np.subtract.outer(xa, ya) ** 2 / self.eps for xa, ya in zip(x_axes, y_axes)]

    @staticmethod
    def _sweep(v, t0, t1, t2):
        a = lse(v[:, :, None, :] + t2[None, None, :, :], axis=3)       # (m0, m1, n2)
        b = lse(a[:, None, :, :] + t1[None, :, :, None], axis=2)       # (m0, n1, n2)
        return lse(b[None, :, :, :] + t0[:, :, None, None], axis=1)    # (n0, n1, n2)

    def lse_x(self, b):
        return self._sweep(np.asarray(b, dtype=np.float64), *self.t)

    def lse_y(self, a):
        return self._sweep(np.asarray(a, dtype=np.float64), *[t.T for t in self.t])


def newton_y(z, m, eps: float, lam: float, beta0, tol: float = 1e-12, max_iters: int = 100):
    """Per node root of g(b) = log(m + exp(b/eps + z)) + b/lam (sinkhorn.py:230-333).

    Closed forms: m = 0 -> b = -z eps lam/(eps+lam); z = -inf, m > 0 ->
    b = -lam log m; both -> b = 700 lam (degenerate, counted).  General nodes
    run Newton from the clipped warm start inside the bracket spanned by the
    two closed forms widened by +-lam, bisecting whenever a node's step
    leaves its bracket.  ``m=None`` means an identically zero background.
    Returns (beta, n_degenerate).
    """
    z = np.asarray(z, dtype=np.float64)
    ratio = eps * lam / (eps + lam)
    if m is None:
        fin = z > -np.inf
        return np.where(fin, -ratio * z, lam * DEGENERATE_BETA_SCALE), int((~fin).sum())
    shape = np.broadcast_shapes(z.shape, np.shape(m), np.shape(beta0))
    z = np.broadcast_to(z, shape).ravel()
    m = np.broadcast_to(np.asarray(m, dtype=np.float64), shape).ravel()
    beta = np.array(np.broadcast_to(np.asarray(beta0, dtype=np.float64), shape)).ravel()
    fz = z > -np.inf
    pm = m > 0
    deg = ~fz & ~pm
    beta[fz & ~pm] = -ratio * z[fz & ~pm]
    beta[~fz & pm] = -lam * np.log(m[~fz & pm])
    beta[deg] = lam * DEGENERATE_BETA_SCALE
    idx = np.flatnonzero(fz & pm)
    if idx.size:
        zg, lm = z[idx], np.log(m[idx])
        c1 = -lam * np.logaddexp(lm, zg)
        c2 = -ratio * zg
        lo = np.minimum(c1, c2) - lam
        hi = np.maximum(c1, c2) + lam
        b = np.clip(beta[idx], lo, hi)
        for _ in range(max_iters):
            w = b / eps + zg
            g = np.logaddexp(lm, w) + b / lam
            gp = 1.0 / (1.0 + np.exp(lm - w)) / eps + 1.0 / lam
            step = g / gp
            act = (np.abs(g) > tol) | (np.abs(step) > 4e-16 * (1.0 + np.abs(b)))
            if not act.any():
                break
            nb = b - step
            out = act & ~((nb > lo) & (nb < hi))
            if out.any():
                pos = g > 0
                hi = np.where(out & pos, np.minimum(hi, b), hi)
                lo = np.where(out & ~pos, np.maximum(lo, b), lo)
                nb = np.where(out & ((nb <= lo) | (nb >= hi)), 0.5 * (lo + hi), nb)
            b = np.where(act, nb, b)
        beta[idx] = b
    return beta.reshape(shape), int(deg.sum())


def gap_terms(alpha, L, mu, eps: float, lam: float):
    """Per-node lam-free terms of KL(P_X pi | e^{-alpha/lam} mu) and P_X pi (sinkhorn.py:336-351)."""
    pos = mu > 0
    lr = alpha / eps + L
    with np.errstate(over="ignore", invalid="ignore"):
        px = np.where(pos, mu * np.exp(lr), 0.0)
        ref = np.where(pos, mu * np.exp(-alpha / lam), 0.0)
        t = np.where(pos, px * (lr + alpha / lam) - px + ref, 0.0)
    return t, px


def global_sinkhorn(kernel: GridKernel, mu, nu, m, alpha0, beta0, lam: float, delta: float,
                    max_iters: int = 10_000, newton_tol: float = 1e-12, newton_iters: int = 100,
                    stop_mass: float | None = None, trace: bool = False) -> dict:
    """Full-grid unbalanced Sinkhorn, gap checked at the top of every iteration
    (reusing the X sweep) and always ending after a Y half-step
    (sinkhorn.py:361-432)."""
    eps = kernel.eps
    ratio = eps * lam / (eps + lam)
    alpha = np.array(alpha0, dtype=np.float64)
    beta = np.array(beta0, dtype=np.float64)
    thr = delta * (float(np.sum(mu)) if stop_mass is None else stop_mass)
    with np.errstate(divide="ignore"):
        log_mu, log_nu = np.log(mu), np.log(nu)
    gap, px, z = math.inf, np.zeros_like(mu), np.full_like(nu, -np.inf)
    iters, converged, clamped, gaps = 0, False, 0, []
    for k in range(1, max_iters + 1):
        L = kernel.lse_x(beta / eps + log_nu)
        if k >= 2:
            t, px = gap_terms(alpha, L, mu, eps, lam)
            gap = lam * float(t.sum())
            gaps.append(gap)
            if gap / lam <= thr:
                converged = True
                break
        alpha = -ratio * L
        z = kernel.lse_y(alpha / eps + log_mu)
        beta, nd = newton_y(z, m, eps, lam, beta, newton_tol, newton_iters)
        clamped = max(clamped, nd)
        iters = k
    if not converged:
        L = kernel.lse_x(beta / eps + log_nu)
        t, px = gap_terms(alpha, L, mu, eps, lam)
        gap = lam * float(t.sum())
        converged = gap / lam <= thr
    return dict(alpha=alpha, beta=beta, gap=gap, iterations=iters, converged=converged,
                x_marginal=px, z=z, newton_clamped=clamped, gap_trace=gaps if trace else [])
