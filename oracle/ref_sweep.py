"""Oracle driver: plan state, weight strategies, stopping certificate, solve loop.

Restates /root/reference/pkg/src/domdec/engine.py (numpy, CPU, test-only):
  StrategyConfig :94, EngineConfig :122, PlanState :157 (energy :185),
  initial_plan_state :234, warm_start_plan :260, BlendScorer :378,
  _coordinate_root :473, get_weights_safe/swift/opt :533-588,
  StitchedGapEvaluator :594, _commit_cell :726, _stitch_alpha :779,
  iteration_sequential :799, iteration_parallel :839, domdec_solve :938.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace

import numpy as np

from .ref_cell import (Ctx, bempty, bshape, grid_window, prepare, product_fragments, rewindow,
                       solve_batch, truncate)
from .ref_lse import GridKernel, global_sinkhorn

STRATEGIES = ("sequential", "safe", "fast", "swift", "opt", "staggered")


def kl_sum(rho, sigma) -> float:
    """KL(rho | sigma) summed (measures.py:337-377)."""
    rho = np.asarray(rho, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    pos = sigma > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(pos, rho, 0.0) / np.where(pos, sigma, 1.0)
        lg = np.where(rho == 0.0, 0.0, rho * np.log(np.where(rho == 0.0, 1.0, r)))
        t = np.where(pos, lg - rho + sigma, 0.0)
    t = np.where(~pos & (rho > 0), np.inf, t)
    return float(t.sum())


@dataclass(frozen=True)
class CellCfg:
    delta: float = 2e-5
    max_iters: int = 10_000
    newton_tol: float = 1e-12
    newton_max_iters: int = 100
    trunc_threshold: float = 1e-15
    chunk_entries: int = 4_000_000


@dataclass(frozen=True)
class EngCfg:
    delta: float = 2e-5
    max_iters: int = 2000
    gap_check_every: int = 1
    cell_delta_factor: float = 0.25
    cell: CellCfg = CellCfg()

    def cell_cfg(self) -> CellCfg:
        return replace(self.cell, delta=self.delta * self.cell_delta_factor)


@dataclass(frozen=True)
class StratCfg:
    kind: str = "staggered"
    leniency: float = 0.005
    opt_max_sweeps: int = 50
    opt_tol: float = 1e-9


@dataclass
class OState:
    box: list
    vals: list
    x_marg: list
    mu_nodes: list
    transport: np.ndarray
    kl: np.ndarray
    duals: dict = field(default_factory=dict)
    truncated_mass: float = 0.0
    global_duals: tuple | None = None

    def clone(self):
        return OState(list(self.box), list(self.vals), list(self.x_marg), self.mu_nodes,
                      self.transport.copy(), self.kl.copy(), dict(self.duals),
                      self.truncated_mass, self.global_duals)


def assemble(ctx: Ctx, st: OState) -> np.ndarray:
    tot = np.zeros(ctx.nu.shape)
    for b, v in zip(st.box, st.vals):
        if not bempty(b):
            tot[b[0]:b[0] + b[1], b[2]:b[2] + b[3]] += v
    return tot


def energy(ctx: Ctx, st: OState) -> dict:
    d1 = 0.0
    for x, mn in zip(st.x_marg, st.mu_nodes):
        d1 += kl_sum(x, mn)
    d2 = kl_sum(assemble(ctx, st), ctx.nu)
    t = float(st.transport.sum())
    e = ctx.eps * float(st.kl.sum())
    r = dict(transport=t, entropy=e, d1=ctx.lam * d1, d2=ctx.lam * d2)
    r["total"] = r["transport"] + r["entropy"] + r["d1"] + r["d2"]
    return r


def cell_nodes(ctx: Ctx, i: int):
    """Retained (mu > 0) flat node ids of basic cell i and their (n, 2) coordinates."""
    b = ctx.basic_box[i]
    n1 = ctx.mu.shape[1]
    r, c = np.meshgrid(np.arange(b[0], b[0] + b[1]), np.arange(b[2], b[2] + b[3]), indexing="ij")
    flat = (r * n1 + c).ravel()
    keep = ctx.mu.ravel()[flat] > 0
    flat = flat[keep]
    xy = np.stack([ctx.x_org[0] + ctx.x_dx * r.ravel()[keep].astype(np.float64),
                   ctx.x_org[1] + ctx.x_dx * c.ravel()[keep].astype(np.float64)], axis=-1)
    return flat, xy


def product_state(ctx: Ctx) -> OState:
    """nu_i = (|mu_i|/|mu|) nu on the full box, exact fragments (engine.py:234-257)."""
    mu_tot = float(ctx.mu.sum())
    ratio = ctx.nu_total / mu_tot
    full = ctx.yfull
    boxes, vals, xm, mns, tr, kl = [], [], [], [], [], []
    for i in range(len(ctx.basic_box)):
        flat, xy = cell_nodes(ctx, i)
        mn = ctx.mu.ravel()[flat]
        v = ctx.nu * (ctx.basic_mass[i] / mu_tot)
        t, k = product_fragments(mn, xy, v, full, ctx)
        boxes.append(full)
        vals.append(v)
        xm.append(mn * ratio)
        mns.append(mn)
        tr.append(t)
        kl.append(k)
    return OState(boxes, vals, xm, mns, np.array(tr), np.array(kl))


def grid_kernel(ctx: Ctx) -> GridKernel:
    xa = ctx.xcoords((0, ctx.mu.shape[0], 0, ctx.mu.shape[1]))
    ya = ctx.ycoords(ctx.yfull)
    return GridKernel(xa, ya, ctx.eps)


def warm_state(ctx: Ctx, delta: float = 1e-3, max_iters: int = 20_000,
               trunc: float = 1e-15) -> OState:
    """Loose global presolve, plan cut along basic cells (engine.py:260-345)."""
    ker = grid_kernel(ctx)
    res = global_sinkhorn(ker, ctx.mu, ctx.nu, None, np.zeros(ctx.mu.shape),
                          np.zeros(ctx.nu.shape), ctx.lam, delta, max_iters)
    return cut_plan(ctx, res["alpha"], res["beta"], trunc)


def cut_plan(ctx: Ctx, alpha_g, beta_g, trunc: float = 1e-15) -> OState:
    alpha = alpha_g.ravel()
    beta = beta_g.ravel()
    eps = ctx.eps
    yc = ctx.ycoords(ctx.yfull)
    Y = np.stack([g.ravel() for g in np.meshgrid(yc[0], yc[1], indexing="ij")], axis=-1)
    nuf = ctx.nu.ravel()
    boxes, vals, xm, mns, tr, kl = [], [], [], [], [], []
    truncated = 0.0
    for i in range(len(ctx.basic_box)):
        flat, xy = cell_nodes(ctx, i)
        mn = ctx.mu.ravel()[flat]
        cost = np.sum((xy[:, None, :] - Y[None, :, :]) ** 2, axis=-1)
        lr = (alpha[flat][:, None] + beta[None, :] - cost) / eps
        blk = np.exp(lr) * mn[:, None] * nuf[None, :]
        mass = float(blk.sum())
        v, b, rem = truncate(blk.sum(axis=0).reshape(ctx.nu.shape), ctx.yfull, trunc)
        truncated += rem
        boxes.append(b)
        vals.append(v)
        xm.append(blk.sum(axis=1))
        mns.append(mn)
        tr.append(float((cost * blk).sum()))
        kl.append(float((blk * lr).sum()) - mass + float(mn.sum()) * ctx.nu_total)
    st = OState(boxes, vals, xm, mns, np.array(tr), np.array(kl), truncated_mass=truncated,
                global_duals=(alpha_g.copy(), beta_g.copy()))
    for part in ctx.parts:
        for j, mem in enumerate(part["members"]):
            live = [st.box[i] for i in mem if not bempty(st.box[i])]
            from .ref_cell import bunion
            yb = bunion(live) if live else ctx.yfull
            st.duals[(part["label"], j)] = (grid_window(alpha_g, part["xbox"][j]).ravel(), yb,
                                            grid_window(beta_g, yb).ravel())
    return st


# -- blend scoring ---------------------------------------------------------------

class Scorer:
    """Tracked energy of theta-blended batch updates (engine.py:378-470)."""

    def __init__(self, ctx: Ctx, st: OState, sols, snap):
        self.ctx = ctx
        self.lam, self.eps = ctx.lam, ctx.eps
        self.nu = ctx.nu.ravel()
        self.y0 = snap.ravel().copy()
        self.t0 = float(st.transport.sum())
        self.k0 = float(st.kl.sum())
        d1e = np.array([kl_sum(x, mn) for x, mn in zip(st.x_marg, st.mu_nodes)])
        self.d10 = self.lam * float(d1e.sum())
        n1 = ctx.nu.shape[1]
        self.upd = []
        for s in sols:
            b = s.ybox
            r, c = np.meshgrid(np.arange(b[0], b[0] + b[1]), np.arange(b[2], b[2] + b[3]),
                               indexing="ij")
            ids = (r * n1 + c).ravel()
            yo = np.zeros(ids.size)
            yn = np.zeros(ids.size)
            for k, i in enumerate(s.members):
                yo += rewindow(st.vals[i], st.box[i], b).ravel()
                yn += rewindow(s.new_vals[k], s.new_box[k], b).ravel()
            to = float(st.transport[s.members].sum())
            ko = float(st.kl[s.members].sum())
            self.upd.append(dict(ids=ids, dy=yn - yo, dt=float(s.transport.sum()) - to,
                                 dk=float(s.kl.sum()) - ko,
                                 xo=[st.x_marg[i] for i in s.members], xn=list(s.x_marg),
                                 mn=[st.mu_nodes[i] for i in s.members],
                                 d1o=self.lam * float(d1e[s.members].sum())))
        self.theta = np.zeros(len(self.upd))
        self.ycur = self.y0.copy()

    def _d1(self, u, th):
        return self.lam * sum(kl_sum((1.0 - th) * a + th * b, m)
                              for a, b, m in zip(u["xo"], u["xn"], u["mn"]))

    def energy_at(self, theta) -> float:
        y = self.y0.copy()
        t, k, d1 = self.t0, self.k0, self.d10
        for u, th in zip(self.upd, np.asarray(theta, dtype=np.float64)):
            th = float(th)
            if th:
                y[u["ids"]] += th * u["dy"]
                t += th * u["dt"]
                k += th * u["dk"]
                d1 += self._d1(u, th) - u["d1o"]
        np.clip(y, 0.0, None, out=y)
        return t + self.eps * k + d1 + self.lam * kl_sum(y, self.nu)

    def set_theta(self, i, th):
        u = self.upd[i]
        d = th - self.theta[i]
        if d:
            self.ycur[u["ids"]] = np.clip(self.ycur[u["ids"]] + d * u["dy"], 0.0, None)
        self.theta[i] = th

    def minimize_coordinate(self, i, tol):
        u = self.upd[i]
        yb = np.clip(self.ycur[u["ids"]] - self.theta[i] * u["dy"], 0.0, None)
        return coord_root(u, yb, self.nu[u["ids"]], u["dt"] + self.eps * u["dk"], self.lam, tol)


def coord_root(u, yb, nuw, lin, lam, tol, max_iters=60) -> float:
    """Safeguarded Newton on the blend derivative over [0, 1] (engine.py:473-527)."""

    def gh(th):
        g, h = lin, 0.0
        for xo, xn, mn in zip(u["xo"], u["xn"], u["mn"]):
            d = xn - xo
            x = (1.0 - th) * xo + th * xn
            with np.errstate(divide="ignore", invalid="ignore"):
                g += lam * float(np.where(d == 0.0, 0.0, d * np.log(x / mn)).sum())
                h += lam * float(np.where(d == 0.0, 0.0, d * d / x).sum())
        y = np.clip(yb + th * u["dy"], 0.0, None)
        d = u["dy"]
        with np.errstate(divide="ignore", invalid="ignore"):
            g += lam * float(np.where(d == 0.0, 0.0, d * np.log(y / nuw)).sum())
            h += lam * float(np.where(d == 0.0, 0.0, d * d / y).sum())
        return g, h

    if gh(0.0)[0] >= 0.0:
        return 0.0
    if gh(1.0)[0] <= 0.0:
        return 1.0
    lo, hi, th = 0.0, 1.0, 0.5
    for _ in range(max_iters):
        g, h = gh(th)
        if g == 0.0:
            break
        if g > 0.0:
            hi = th
        else:
            lo = th
        cand = th - g / h if (np.isfinite(g) and np.isfinite(h) and h > 0.0) else 0.5 * (lo + hi)
        if not lo < cand < hi:
            cand = 0.5 * (lo + hi)
        if abs(cand - th) <= tol * max(1.0, abs(th)):
            th = cand
            break
        th = cand
    return min(max(th, 0.0), 1.0)


def weights_opt(sc: Scorer, k: int, sweeps: int, tol: float) -> np.ndarray:
    ones, safe = np.ones(k), np.full(k, 1.0 / k)
    start = ones if sc.energy_at(ones) <= sc.energy_at(safe) else safe
    for i in range(k):
        sc.set_theta(i, float(start[i]))
    for _ in range(sweeps):
        moved = 0.0
        for i in range(k):
            th = sc.minimize_coordinate(i, tol)
            moved = max(moved, abs(th - sc.theta[i]))
            sc.set_theta(i, th)
        if moved <= tol:
            break
    cands = [sc.theta.copy(), ones, safe]
    es = [sc.energy_at(v) for v in cands]
    return cands[int(np.argmin(es))]


# -- stopping certificate ----------------------------------------------------------

class GapEval:
    """E(state) - D(stitched alpha, best beta) with 2 polish sweeps and a persistent
    best pair (engine.py:594-682)."""

    def __init__(self, ctx: Ctx, polish: int = 2):
        self.ker = grid_kernel(ctx)
        self.eps, self.lam = ctx.eps, ctx.lam
        self.polish = polish
        self.mu, self.nu = ctx.mu, ctx.nu
        self.mp = float(self.mu.sum()) * float(self.nu.sum())
        with np.errstate(divide="ignore"):
            self.lmu, self.lnu = np.log(self.mu), np.log(self.nu)
        self.best = None
        self.sweeps = 0

    def seed(self, a, b):
        a = np.asarray(a, dtype=np.float64).reshape(self.mu.shape)
        b = np.asarray(b, dtype=np.float64).reshape(self.nu.shape)
        self.best = (a, b, self._dual(a, b))

    def _ascend(self, beta):
        sc = self.eps * self.lam / (self.eps + self.lam)
        a = bn = None
        for _ in range(max(1, self.polish)):
            a = -sc * self.ker.lse_x(beta / self.eps + self.lnu)
            bn = -sc * self.ker.lse_y(a / self.eps + self.lmu)
            beta = bn
            self.sweeps += 2
        return a, bn

    def _dual(self, a, b):
        eps, lam = self.eps, self.lam
        z = self.ker.lse_y(a / eps + self.lmu)
        self.sweeps += 1
        with np.errstate(over="ignore", under="ignore"):
            cpl = float(np.sum(self.nu * np.exp(b / eps + z)))
            dx = lam * float(np.sum(self.mu * (1.0 - np.exp(-a / lam))))
            dy = lam * float(np.sum(self.nu * (1.0 - np.exp(-b / lam))))
        return dx + dy - eps * (cpl - self.mp)

    def dual_value(self, alpha_flat):
        sc = self.eps * self.lam / (self.eps + self.lam)
        st = alpha_flat.reshape(self.mu.shape)
        b0 = -sc * self.ker.lse_y(st / self.eps + self.lmu)
        self.sweeps += 1
        a1, b1 = self._ascend(b0)
        d1 = self._dual(a1, b1)
        if self.best is not None:
            a2, b2 = self._ascend(self.best[1])
            d2 = self._dual(a2, b2)
            if d2 > d1 or (d2 == d1 and self.best[2] > d1):
                a1, b1, d1 = a2, b2, d2
            d1 = max(d1, self.best[2])
        self.best = (a1, b1, d1)
        return d1


# -- iterations ----------------------------------------------------------------------

@dataclass
class Stats:
    k: int = 0
    label: str = ""
    action: str = ""
    gap: float = float("nan")
    entry_gap: float = 0.0
    alpha: np.ndarray | None = None
    x_err: float = 0.0
    y_err: float = 0.0
    balance_fallbacks: int = 0
    safe_fallbacks: int = 0
    truncated_mass: float = 0.0
    newton_clamped: int = 0
    nu_minus_clamped: int = 0
    nonconverged_cells: int = 0
    balance_target_miss: float = 0.0
    nu_j_drift_nodes: int = 0
    cell_iters: int = 0
    times: dict = field(default_factory=lambda: dict(assemble=0.0, solve=0.0, score=0.0,
                                                     commit=0.0))


def commit(ctx: Ctx, st: OState, p, s, theta: float, label: str, thr: float):
    """Install the theta-blend of one cell (engine.py:726-776)."""
    lam = ctx.lam
    yb = s.ybox
    old = [rewindow(st.vals[i], st.box[i], yb) for i in s.members]
    yo = np.zeros(bshape(yb))
    for w in old:
        yo += w
    yn = np.zeros(bshape(yb))
    if theta >= 1.0:
        st.truncated_mass += s.truncated_mass
        for k, i in enumerate(s.members):
            st.box[i], st.vals[i] = s.new_box[k], s.new_vals[k]
            st.x_marg[i] = s.x_marg[k]
            st.transport[i], st.kl[i] = s.transport[k], s.kl[k]
            yn += rewindow(s.new_vals[k], s.new_box[k], yb)
    elif theta > 0.0:
        st.truncated_mass += theta * s.truncated_mass
        for k, i in enumerate(s.members):
            bw = (1.0 - theta) * old[k] + theta * rewindow(s.new_vals[k], s.new_box[k], yb)
            v, b, rem = truncate(bw, yb, thr)
            st.truncated_mass += rem
            st.box[i], st.vals[i] = b, v
            st.x_marg[i] = (1.0 - theta) * st.x_marg[i] + theta * s.x_marg[k]
            st.transport[i] = (1.0 - theta) * st.transport[i] + theta * s.transport[k]
            st.kl[i] = (1.0 - theta) * st.kl[i] + theta * s.kl[k]
            yn += rewindow(v, b, yb)
    else:
        yn = yo
    st.duals[(label, s.j)] = (s.alpha.copy(), yb, s.beta.copy())
    num = p.m_win * p.nu_win if p.m_win is not None else 0.0
    y_err = float(np.abs(yn.ravel() + num - np.exp(-s.beta / lam) * p.nu_win).sum())
    x_err = 0.0
    for k, i in enumerate(s.members):
        r = p.rows[k]
        keep = p.mu_win[r] > 0
        a = s.alpha[r][keep]
        x_err += float(np.abs(st.x_marg[i] - np.exp(-a / lam) * st.mu_nodes[i]).sum())
    return x_err, y_err, yo.ravel(), yn.ravel()


def stitch(ctx: Ctx, stats: Stats, p, s):
    if stats.alpha is None:
        stats.alpha = np.zeros(ctx.mu.shape)
    for k, i in enumerate(s.members):
        b = ctx.basic_box[i]
        stats.alpha[b[0]:b[0] + b[1], b[2]:b[2] + b[3]] = s.alpha[p.rows[k]].reshape(b[1], b[3])


def _absorb(stats: Stats, sols):
    for s in sols:
        stats.entry_gap += s.first_gap
        stats.balance_fallbacks += s.balance_fallbacks
        stats.newton_clamped = max(stats.newton_clamped, s.newton_clamped)
        stats.nu_minus_clamped += s.n_clamped
        stats.nonconverged_cells += 0 if s.converged else 1
        stats.balance_target_miss = max(stats.balance_target_miss, s.target_miss)
        stats.nu_j_drift_nodes += s.drift_nodes
        stats.cell_iters += s.iterations


def iterate_sequential(ctx: Ctx, st: OState, part: dict, cfg: EngCfg, stats: Stats):
    """Cell-by-cell pass on a running Y-marginal (engine.py:799-836)."""
    cc = cfg.cell_cfg()
    y = assemble(ctx, st)
    n1 = ctx.nu.shape[1]
    for j in range(len(part["members"])):
        t0 = time.perf_counter()
        probs = prepare(ctx, part, [j], st, y)
        sols = solve_batch(probs, ctx, cc)
        stats.times["solve"] += time.perf_counter() - t0
        _absorb(stats, sols)
        xe, ye, yo, yn = commit(ctx, st, probs[0], sols[0], 1.0, part["label"], cc.trunc_threshold)
        stitch(ctx, stats, probs[0], sols[0])
        b = sols[0].ybox
        yv = y.reshape(-1)
        r, c = np.meshgrid(np.arange(b[0], b[0] + b[1]), np.arange(b[2], b[2] + b[3]),
                           indexing="ij")
        ids = (r * n1 + c).ravel()
        yv[ids] = np.clip(yv[ids] + (yn - yo), 0.0, None)
        stats.x_err += xe
        stats.y_err += ye
        stats.truncated_mass += sols[0].truncated_mass
    stats.action = "sequential"


def iterate_parallel(ctx: Ctx, st: OState, part: dict, strat: StratCfg, cfg: EngCfg,
                     stats: Stats):
    """Snapshot, batch solve, weighted commit (engine.py:839-922)."""
    if strat.kind == "sequential":
        raise ValueError("sequential updates run through iterate_sequential")
    cc = cfg.cell_cfg()
    ncomp = len(part["members"])
    batches = part["batches"] if strat.kind == "staggered" else [list(range(ncomp))]
    actions = []
    for batch in batches:
        t0 = time.perf_counter()
        snap = assemble(ctx, st)
        t1 = time.perf_counter()
        probs = prepare(ctx, part, batch, st, snap)
        sols = solve_batch(probs, ctx, cc)
        t2 = time.perf_counter()
        _absorb(stats, sols)
        kb = len(sols)
        if strat.kind == "fast":
            th = np.ones(kb)
            actions.append("greedy")
        elif strat.kind == "safe":
            th = np.full(kb, 1.0 / kb)
            actions.append("safe")
        elif strat.kind == "swift":
            sc = Scorer(ctx, st, sols, snap)
            ones, safe = np.ones(kb), np.full(kb, 1.0 / kb)
            th = ones if sc.energy_at(ones) <= sc.energy_at(safe) else safe
            actions.append("greedy" if all(t == 1.0 for t in th) else "safe")
        elif strat.kind == "opt":
            sc = Scorer(ctx, st, sols, snap)
            th = weights_opt(sc, kb, strat.opt_max_sweeps, strat.opt_tol)
            actions.append("opt")
        else:
            sc = Scorer(ctx, st, sols, snap)
            e0 = sc.energy_at(np.zeros(kb))
            eg = sc.energy_at(np.ones(kb))
            es = sc.energy_at(np.full(kb, 1.0 / kb))
            allow = strat.leniency * max(0.0, e0 - es)
            if eg <= e0 + allow:
                th = np.ones(kb)
                actions.append("greedy")
            else:
                th = np.full(kb, 1.0 / kb)
                actions.append("safe-fallback")
                stats.safe_fallbacks += 1
        t3 = time.perf_counter()
        before = st.truncated_mass
        for p, s, t in zip(probs, sols, th):
            xe, ye, _, _ = commit(ctx, st, p, s, float(t), part["label"], cc.trunc_threshold)
            stitch(ctx, stats, p, s)
            stats.x_err += xe
            stats.y_err += ye
        stats.truncated_mass += st.truncated_mass - before
        t4 = time.perf_counter()
        stats.times["assemble"] += t1 - t0
        stats.times["solve"] += t2 - t1
        stats.times["score"] += t3 - t2
        stats.times["commit"] += t4 - t3
    if len(actions) == 1:
        stats.action = actions[0]
    else:
        n = actions.count("safe-fallback")
        stats.action = "greedy" if n == 0 else f"safe-fallback({n}/{len(actions)})"


def solve(ctx: Ctx, st: OState | None, strat: StratCfg = StratCfg(), cfg: EngCfg = EngCfg(),
          single_partition: bool = False, evaluator: GapEval | None = None):
    """Alternate partitions until gap/lam <= delta |mu| or the cap (engine.py:938-1037).

    Returns (state, report dict, trace list of dicts).
    """
    if st is None:
        st = product_state(ctx)
    parts = ctx.parts[:1] if single_partition else ctx.parts
    lam = ctx.lam
    mu_tot = float(ctx.mu.sum())
    ev = evaluator if evaluator is not None else GapEval(ctx)
    if st.global_duals is not None:
        ev.seed(*st.global_duals)
    every = max(1, cfg.gap_check_every)
    trace = []
    times = dict(assemble=0.0, solve=0.0, score=0.0, commit=0.0, evaluate=0.0, total=0.0)
    diag = dict(balance_fallbacks=0, safe_fallbacks=0, nonconverged_cells=0, newton_clamped=0,
                nu_minus_clamped=0, balance_target_miss=0.0, nu_j_drift_nodes=0, cell_iters=0)
    conv = False
    last = math.inf
    stats = Stats()
    sb = energy(ctx, st)
    tall = time.perf_counter()
    for k in range(1, cfg.max_iters + 1):
        part = parts[(k - 1) % len(parts)]
        stats = Stats(k=k, label=part["label"])
        t0 = time.perf_counter()
        if strat.kind == "sequential":
            iterate_sequential(ctx, st, part, cfg, stats)
        else:
            iterate_parallel(ctx, st, part, strat, cfg, stats)
        sb = energy(ctx, st)
        if k % every == 0 or k == cfg.max_iters:
            t1 = time.perf_counter()
            stats.gap = sb["total"] - ev.dual_value(stats.alpha.ravel())
            times["evaluate"] += time.perf_counter() - t1
            last = stats.gap
        trace.append(dict(k=k, label=part["label"], action=stats.action, **sb, gap=stats.gap,
                          x_err=stats.x_err, y_err=stats.y_err,
                          wall_time=time.perf_counter() - t0))
        for key in ("assemble", "solve", "score", "commit"):
            times[key] += stats.times[key]
        for key in ("balance_fallbacks", "safe_fallbacks", "nonconverged_cells",
                    "nu_minus_clamped", "nu_j_drift_nodes", "cell_iters"):
            diag[key] += getattr(stats, key)
        diag["newton_clamped"] = max(diag["newton_clamped"], stats.newton_clamped)
        diag["balance_target_miss"] = max(diag["balance_target_miss"], stats.balance_target_miss)
        if last / lam <= cfg.delta * mu_tot:
            conv = True
            break
    times["total"] = time.perf_counter() - tall
    diag["truncated_mass"] = st.truncated_mass
    rep = dict(converged=conv, iterations=len(trace), final_score=sb,
               rel_pd_gap=last / max(abs(sb["total"]), 1e-300), x_err=stats.x_err,
               y_err=stats.y_err, timings=times, diagnostics=diag,
               sparsity=dict(stored_entries=int(sum(v.size for v in st.vals)),
                             nonzero_entries=int(sum(np.count_nonzero(v) for v in st.vals))))
    return st, rep, trace
