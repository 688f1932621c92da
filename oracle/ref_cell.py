"""Oracle cell pipeline: window assembly, stacked solves, balancing, fragments.

Restates /root/reference/pkg/src/domdec/cells.py (numpy, CPU, test-only):
  compute_nu_minus :144, make_cell_problems :165, solve_cell_batch :235,
  _solve_chunk :283, _finalize :396, balance_cell_masses :446,
  _move_mass :488, _restore_columns :510, _fix_column :529, _walk_entry :552,
  product_plan_fragments :566.

Everything is 2D-embedded: a box is (off0, ext0, off1, ext1).
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field

import numpy as np

from .ref_lse import WindowKernel, gap_terms, newton_y

log = logging.getLogger(__name__)


# -- box helpers (2D embedded) -------------------------------------------------

def bshape(b):
    return (b[1], b[3])


def bempty(b):
    return b[1] == 0 or b[3] == 0


def bunion(boxes):
    lo0 = min(b[0] for b in boxes)
    hi0 = max(b[0] + b[1] for b in boxes)
    lo1 = min(b[2] for b in boxes)
    hi1 = max(b[2] + b[3] for b in boxes)
    return (lo0, hi0 - lo0, lo1, hi1 - lo1)


def rewindow(vals, src, dst):
    """Values boxed on ``src`` re-read on ``dst`` (zero fill)."""
    out = np.zeros(bshape(dst))
    if vals is None or bempty(src):
        return out
    l0, h0 = max(src[0], dst[0]), min(src[0] + src[1], dst[0] + dst[1])
    l1, h1 = max(src[2], dst[2]), min(src[2] + src[3], dst[2] + dst[3])
    if l0 < h0 and l1 < h1:
        out[l0 - dst[0]:h0 - dst[0], l1 - dst[2]:h1 - dst[2]] = \
            vals.reshape(bshape(src))[l0 - src[0]:h0 - src[0], l1 - src[2]:h1 - src[2]]
    return out


def grid_window(arr2d, b):
    return rewindow(arr2d, (0, arr2d.shape[0], 0, arr2d.shape[1]), b)


def truncate(vals2d, box, thr):
    """Drop entries < thr, shrink box; (values, box, removed) (measures.py:383-407)."""
    if bempty(box):
        return vals2d, box, 0.0
    keep = vals2d >= thr
    removed = float(vals2d[~keep].sum())
    if not keep.any():
        return np.zeros((0, 0)), (0, 0, 0, 0), removed
    r = np.nonzero(keep.any(axis=1))[0]
    c = np.nonzero(keep.any(axis=0))[0]
    r0, r1, c0, c1 = int(r[0]), int(r[-1]) + 1, int(c[0]), int(c[-1]) + 1
    v = np.where(keep, vals2d, 0.0)[r0:r1, c0:c1]
    return v, (box[0] + r0, r1 - r0, box[2] + c0, c1 - c0), removed


def xlogy(x, y):
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(x == 0.0, 0.0, x * np.log(np.where(x == 0.0, 1.0, y)))


# -- problem context -----------------------------------------------------------

@dataclass
class Ctx:
    """Problem data in 2D embedding plus partition tables."""

    mu: np.ndarray          # X grid masses (2D)
    nu: np.ndarray          # Y grid masses (2D)
    x_dx: float
    x_org: tuple
    y_dx: float
    y_org: tuple
    lam: float
    eps: float
    basic_box: list         # per basic cell (o0, e0, o1, e1)
    basic_mass: np.ndarray
    parts: list             # dicts: label, xbox (list of boxes), members (lists), batches
    nu_total: float = 0.0

    def __post_init__(self):
        self.nu_total = float(self.nu.sum())

    def xcoords(self, b):
        return [self.x_org[0] + self.x_dx * np.arange(b[0], b[0] + b[1], dtype=np.float64),
                self.x_org[1] + self.x_dx * np.arange(b[2], b[2] + b[3], dtype=np.float64)]

    def ycoords(self, b):
        return [self.y_org[0] + self.y_dx * np.arange(b[0], b[0] + b[1], dtype=np.float64),
                self.y_org[1] + self.y_dx * np.arange(b[2], b[2] + b[3], dtype=np.float64)]

    @property
    def yfull(self):
        return (0, self.nu.shape[0], 0, self.nu.shape[1])


def cost_block(xc, yc):
    """|x - y|^2 between flattened window enumerations (scores.py:86-91)."""
    x = np.stack([g.ravel() for g in np.meshgrid(xc[0], xc[1], indexing="ij")], axis=-1)
    y = np.stack([g.ravel() for g in np.meshgrid(yc[0], yc[1], indexing="ij")], axis=-1)
    d = x[:, None, :] - y[None, :, :]
    return np.einsum("ijk,ijk->ij", d, d)


@dataclass
class CellProb:
    j: int
    xbox: tuple
    mu_win: np.ndarray
    ybox: tuple
    nu_win: np.ndarray
    m_win: np.ndarray | None
    alpha0: np.ndarray
    beta0: np.ndarray
    members: list
    rows: list
    masses: np.ndarray
    xc: list
    yc: list
    n_clamped: int
    cell_sum: np.ndarray


@dataclass
class CellSol:
    j: int
    members: list
    rows: list
    ybox: tuple
    alpha: np.ndarray
    beta: np.ndarray
    vals: np.ndarray         # (n_mem, ny) balanced member marginals
    raw: np.ndarray          # pre-balancing split
    converged: bool
    iterations: int
    gap: float
    first_gap: float = 0.0
    new_box: list = field(default_factory=list)
    new_vals: list = field(default_factory=list)
    x_marg: list = field(default_factory=list)
    transport: np.ndarray | None = None
    kl: np.ndarray | None = None
    balance_fallbacks: int = 0
    truncated_mass: float = 0.0
    newton_clamped: int = 0
    n_clamped: int = 0
    targets: np.ndarray | None = None
    target_miss: float = 0.0
    drift_nodes: int = 0


def prepare(ctx: Ctx, part: dict, ids, st, snap: np.ndarray) -> list:
    """Window up composite cells against a Y-marginal snapshot (cells.py:144-232)."""
    out = []
    for j in ids:
        xb = part["xbox"][j]
        mem = part["members"][j]
        mu_win = grid_window(ctx.mu, xb).ravel()
        flat = np.arange(xb[1] * xb[3]).reshape(xb[1], xb[3])
        rows = []
        for i in mem:
            bb = ctx.basic_box[i]
            rows.append(flat[bb[0] - xb[0]:bb[0] - xb[0] + bb[1],
                             bb[2] - xb[2]:bb[2] - xb[2] + bb[3]].ravel())
        live = [st.box[i] for i in mem if not bempty(st.box[i])]
        yb = bunion(live) if live else ctx.yfull
        csum = np.zeros(bshape(yb))
        for i in mem:
            csum += rewindow(st.vals[i], st.box[i], yb)
        pw = grid_window(snap, yb)
        nw = grid_window(ctx.nu, yb)
        if (nw <= 0).any():
            raise ValueError("nu must be positive on the cell window")
        diff = pw - csum
        n_cl = int(np.count_nonzero(diff < -1e-12 * np.maximum(pw, csum)))
        m = (np.clip(diff, 0.0, None) / nw).ravel()
        dual = st.duals.get((part["label"], j))
        if dual is None:
            a0, b0 = np.zeros(mu_win.size), np.zeros(csum.size)
        else:
            a0 = dual[0]
            b0 = rewindow(dual[2], dual[1], yb).ravel()
        out.append(CellProb(j=j, xbox=xb, mu_win=mu_win, ybox=yb, nu_win=nw.ravel(),
                            m_win=m if m.any() else None, alpha0=a0, beta0=b0, members=list(mem),
                            rows=rows, masses=ctx.basic_mass[list(mem)], xc=ctx.xcoords(xb),
                            yc=ctx.ycoords(yb), n_clamped=n_cl, cell_sum=csum.ravel()))
    return out


def solve_batch(probs: list, ctx: Ctx, cfg) -> list:
    """Zero-mass cells pass through; live cells solve in stacked chunks (cells.py:235-280)."""
    sols = [None] * len(probs)
    live = []
    for k, p in enumerate(probs):
        if p.mu_win.sum() > 0:
            live.append(k)
            continue
        nm = len(p.members)
        sols[k] = CellSol(j=p.j, members=p.members, rows=p.rows, ybox=p.ybox,
                          alpha=p.alpha0.copy(), beta=p.beta0.copy(),
                          vals=np.zeros((nm, p.nu_win.size)), raw=np.zeros((nm, p.nu_win.size)),
                          converged=True, iterations=0, gap=0.0,
                          new_box=[(0, 0, 0, 0)] * nm, new_vals=[np.zeros((0, 0))] * nm,
                          x_marg=[np.zeros(0)] * nm, transport=np.zeros(nm), kl=np.zeros(nm))
    if not live:
        return sols
    nx = probs[live[0]].mu_win.size
    if any(probs[k].mu_win.size != nx for k in live):
        raise ValueError("cells of one batch must share the X-window shape")
    ny_max = max(probs[k].nu_win.size for k in live)
    per = max(1, cfg.chunk_entries // max(nx * ny_max, 1))
    for lo in range(0, len(live), per):
        grp = live[lo:lo + per]
        for k, s in zip(grp, _solve_stack([probs[k] for k in grp], ctx, cfg)):
            sols[k] = s
    return sols


def _solve_stack(probs, ctx: Ctx, cfg) -> list:
    """One stacked Sinkhorn run with per-cell freezing (cells.py:283-393)."""
    B, nx = len(probs), probs[0].mu_win.size
    ny = max(p.nu_win.size for p in probs)
    eps, lam = ctx.eps, ctx.lam
    ratio = eps * lam / (eps + lam)
    cost = np.zeros((B, nx, ny))
    mu = np.zeros((B, nx))
    nu = np.zeros((B, ny))
    m = np.zeros((B, ny))
    alpha = np.zeros((B, nx))
    beta = np.zeros((B, ny))
    any_m = False
    for b, p in enumerate(probs):
        n = p.nu_win.size
        cost[b, :, :n] = cost_block(p.xc, p.yc)
        mu[b], nu[b, :n] = p.mu_win, p.nu_win
        if p.m_win is not None:
            m[b, :n] = p.m_win
            any_m = True
        alpha[b], beta[b, :n] = p.alpha0, p.beta0
    negc = -cost / eps
    ker = WindowKernel(negc)
    with np.errstate(divide="ignore"):
        lmu, lnu = np.log(mu), np.log(nu)
    thr = cfg.delta * mu.sum(axis=1)
    frozen = np.zeros(B, dtype=bool)
    gaps = np.full(B, np.inf)
    first = None
    iters = np.zeros(B, dtype=int)
    clamped = 0
    for k in range(1, cfg.max_iters + 1):
        L = ker.lse_x(beta / eps + lnu)
        if k >= 2:
            g = lam * gap_terms(alpha, L, mu, eps, lam)[0].sum(axis=1)
            if first is None:
                first = g.copy()
            new = ~frozen & (g / lam <= thr)
            gaps = np.where(new, g, gaps)
            frozen |= new
            if frozen.all():
                break
        alpha = np.where(frozen[:, None], alpha, -ratio * L)
        z = ker.lse_y(alpha / eps + lmu)
        bn, nd = newton_y(z, m if any_m else None, eps, lam, beta, cfg.newton_tol,
                          cfg.newton_max_iters)
        clamped = max(clamped, nd)
        beta = np.where(frozen[:, None], beta, bn)
        iters = np.where(frozen, iters, k)
    L = ker.lse_x(beta / eps + lnu)
    if not frozen.all():
        g = lam * gap_terms(alpha, L, mu, eps, lam)[0].sum(axis=1)
        gaps = np.where(frozen, gaps, g)
        if first is None:
            first = g.copy()
    conv = gaps / lam <= thr
    mu_bar = np.exp(ratio * L / lam) * mu          # exp(-alpha_extra/lam) mu
    sc = alpha[:, :, None] / eps + beta[:, None, :] / eps + negc
    with np.errstate(over="ignore"):
        plan = np.exp(sc + lmu[:, :, None] + lnu[:, None, :])
    out = []
    for b, p in enumerate(probs):
        n = p.nu_win.size
        nm = len(p.members)
        split, tc, tl, mc = (np.empty((nm, n)) for _ in range(4))
        for i, r in enumerate(p.rows):
            pw = plan[b, r, :n]
            split[i] = pw.sum(axis=0)
            tc[i] = (pw * cost[b, r, :n]).sum(axis=0)
            tl[i] = (pw * sc[b, r, :n]).sum(axis=0)
            mc[i] = (cost[b, r, :n] * mu[b, r, None]).sum(axis=0)
        s = CellSol(j=p.j, members=p.members, rows=p.rows, ybox=p.ybox, alpha=alpha[b].copy(),
                    beta=beta[b, :n].copy(), vals=split.copy(), raw=split,
                    converged=bool(conv[b]), iterations=int(iters[b]), gap=float(gaps[b]),
                    first_gap=float(first[b]), newton_clamped=clamped, n_clamped=p.n_clamped)
        balance(s, mu_bar[b])
        finalize(s, p, ctx, plan[b, :, :n], tc, tl, mc, cfg.trunc_threshold)
        out.append(s)
    return out


def finalize(s: CellSol, p: CellProb, ctx: Ctx, plan, tc, tl, mc, thr: float) -> None:
    """Truncate balanced member marginals; exact fragments of the edited plan (cells.py:396-443)."""
    nm = len(p.members)
    s.transport, s.kl = np.empty(nm), np.empty(nm)
    for i, r in enumerate(p.rows):
        v, nb, removed = truncate(s.vals[i].reshape(bshape(p.ybox)).copy(), p.ybox, thr)
        s.truncated_mass += removed
        fin = rewindow(v, nb, p.ybox).ravel()
        raw = s.raw[i]
        pos = raw > 0
        f = np.where(pos, fin / np.where(pos, raw, 1.0), 0.0)
        extra = np.where(pos, 0.0, fin)
        mi = float(p.masses[i])
        s.transport[i] = float((f * tc[i]).sum() + (extra * mc[i]).sum() / mi)
        s.kl[i] = float((f * tl[i]).sum() + xlogy(np.where(pos, fin, 0.0), f).sum()
                        + xlogy(extra, extra / (mi * p.nu_win)).sum() - fin.sum()
                        + mi * ctx.nu_total)
        xm = plan[r] @ f
        es = float(extra.sum())
        if es:
            xm = xm + p.mu_win[r] * (es / mi)
        s.x_marg.append(xm[p.mu_win[r] > 0])
        s.new_box.append(nb)
        s.new_vals.append(v)


def balance(s: CellSol, mu_bar: np.ndarray) -> None:
    """Horizontal mass transfer to targets m_i = mbar_i |nu_J| / mbar(X_J) (cells.py:446-485)."""
    vals = s.vals
    mbar = np.array([mu_bar[r].sum() for r in s.rows])
    tot = mbar.sum()
    if not tot > 0:
        raise ValueError("balancing reference mass must be positive")
    masses = vals.sum(axis=1)
    targets = mbar * (masses.sum() / tot)
    s.targets = targets
    sur = masses - targets
    tol = 1e-13 * np.maximum(targets, 1e-300)
    donors = [i for i in range(len(targets)) if sur[i] > tol[i]]
    recips = [i for i in range(len(targets)) if sur[i] < -tol[i]]
    if donors and recips:
        col0 = vals.sum(axis=0)
        di = ri = 0
        while di < len(donors) and ri < len(recips):
            d, r = donors[di], recips[ri]
            amt = min(sur[d], -sur[r])
            s.balance_fallbacks += move_mass(vals, d, r, amt)
            sur[d] -= amt
            sur[r] += amt
            if sur[d] <= tol[d]:
                di += 1
            if sur[r] >= -tol[r]:
                ri += 1
        np.clip(vals, 0.0, None, out=vals)
        s.drift_nodes = restore_columns(vals, col0)
    miss = np.abs(vals.sum(axis=1) - targets) / np.maximum(targets, 1e-300)
    s.target_miss = float(miss.max()) if miss.size else 0.0


def move_mass(vals, d: int, r: int, amt: float) -> int:
    """Greedy front-to-back walk of donor row d into row r; 1 on fallback (cells.py:488-507)."""
    if amt <= 0:
        return 0
    row = vals[d]
    cum = np.cumsum(row)
    if not cum.size or cum[-1] < amt:
        if cum.size and cum[-1] > 0:
            vals[r] += row
            vals[d] = 0.0
        return 1
    k = int(np.searchsorted(cum, amt))
    if k:
        vals[r, :k] += row[:k]
        vals[d, :k] = 0.0
    part = amt - (cum[k - 1] if k else 0.0)
    vals[d, k] -= part
    vals[r, k] += part
    return 0


def restore_columns(vals, col0) -> int:
    """Ulp-walk one entry per drifted column until sums match bitwise (cells.py:510-526)."""
    bad = 0
    for c in np.flatnonzero(col0 - vals.sum(axis=0)):
        if not _fix_col(vals[:, c], col0[c]):
            bad += 1
            log.warning("node %d sum off after restoration", int(c))
    return bad


def _fix_col(col, target) -> bool:
    order = np.argsort(col)[::-1]
    for t in order:
        if _walk(col, t, target):
            return True
    for t in order:
        x0 = col[t]
        for toward in (np.inf, -np.inf):
            x1 = np.nextafter(x0, toward)
            if x1 < 0:
                continue
            col[t] = x1
            for u in order:
                if u != t and _walk(col, u, target):
                    return True
            col[t] = x0
    return bool(col.sum() == target)


def _walk(col, t, target, cap: int = 256) -> bool:
    x0 = x = col[t]
    for _ in range(cap):
        s = col.sum()
        if s == target:
            return True
        x = np.nextafter(x, np.inf if s < target else -np.inf)
        if x < 0:
            break
        col[t] = x
    col[t] = x0
    return bool(col.sum() == target)


def product_fragments(mu_nodes, xnode_coords, vals, box, ctx: Ctx):
    """Exact (transport, KL) of pi_i = mu_i x nu_i / |mu_i| (cells.py:566-606)."""
    mm = float(mu_nodes.sum())
    if mm <= 0:
        raise ValueError("cell mu mass must be positive")
    if bempty(box) or float(vals.sum()) == 0.0:
        return 0.0, float(mm * ctx.nu_total)
    mn = float(vals.sum())
    yax = ctx.ycoords(box)
    tr = 0.0
    for a in range(2):
        yc = yax[a].reshape((-1, 1) if a == 0 else (1, -1))
        sx2 = float((mu_nodes * xnode_coords[:, a] ** 2).sum())
        sx1 = float((mu_nodes * xnode_coords[:, a]).sum())
        sy2 = float((vals * yc ** 2).sum())
        sy1 = float((vals * yc).sum())
        tr += sx2 * mn - 2.0 * sx1 * sy1 + mm * sy2
    tr /= mm
    nb = grid_window(ctx.nu, box)
    ent = xlogy(vals, vals / nb).sum()
    return tr, float(ent - mn * np.log(mm) - mn + mm * ctx.nu_total)
