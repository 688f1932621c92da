// Batched composite-cell kernels: solve, blend scoring, commit.
//
// One CTA per composite cell.  The cell's X window (2s x 2s nodes) and Y
// window (union of its members' Y-marginal boxes) are staged in a per-cell
// workspace (shared memory when it fits, else a global arena), the separable
// squared-Euclidean kernel is applied one grid axis at a time, and the whole
// unbalanced Sinkhorn loop runs inside the CTA until the cell's own PD gap
// test passes.  The epilogue splits the cell plan's Y-marginal by member
// basic cells, balances member masses, truncates to fresh boxes, and forms
// the score fragments and X-marginals — the same outputs the reference
// produces in cells.py:283-443.

#include <cooperative_groups.h>

#include "common.cuh"
#include "domdec_b200.h"

// minimum resident cell CTAs per SM (2 caps registers at 64 so two 512-thread
// cell CTAs can share an SM; the host then halves the shared-memory budget)
#ifndef DD_CELL_MIN_BLOCKS
#define DD_CELL_MIN_BLOCKS 1
#endif

namespace dd {

struct CellWin {
    int xo0, xe0, xo1, xe1;  // X window
    int yo0, ye0, yo1, ye1;  // Y window
    int nx, ny;
};

// Workspace layout (doubles), identical on host and device.
struct WsLayout {
    int64_t xc0, xc1, yc0, yc1;
    int64_t alpha, u, L, mu, tx, lmu, wx;
    int64_t beta, ty, wy;
    int64_t K0, K1, mid, rmax;
    int64_t K0y, K1y, c0, c1;
    int64_t midstride;
    int64_t total;
};

// Per-cell workspace: coordinates, 7 X-window arrays, 3 Y-window arrays (beta,
// bv/z, sweep weights), the two per-axis kernel tables and the stage scratch.
// The read-only Y arrays (log nu, background density m) stay in global memory.
__host__ __device__ inline WsLayout ws_layout(int nw0, int nw1, int ny0, int ny1) {
    WsLayout w;
    const int64_t nx = (int64_t)nw0 * nw1, ny = (int64_t)ny0 * ny1;
    int64_t o = 0;
    w.xc0 = o; o += nw0;
    w.xc1 = o; o += nw1;
    w.yc0 = o; o += ny0;
    w.yc1 = o; o += ny1;
    w.alpha = o; o += nx;
    w.u = o; o += nx;
    w.L = o; o += nx;
    w.mu = o; o += nx;
    w.tx = o; o += nx;
    w.lmu = o; o += nx;
    w.wx = o; o += nx;
    w.beta = o; o += ny;
    w.ty = o; o += ny;
    w.wy = o; o += ny;
    w.K0 = o; o += (int64_t)nw0 * ny0;
    w.K1 = o; o += (int64_t)nw1 * ny1;
    int64_t ms = (int64_t)ny0 * nw1;
    const int64_t ms2 = (int64_t)nw0 * ny1;
    if (ms2 > ms) ms = ms2;
    w.midstride = ms;
    w.mid = o; o += 5 * ms;
    int64_t rm = ny0 > ny1 ? ny0 : ny1;
    if (nw0 > rm) rm = nw0;
    if (nw1 > rm) rm = nw1;
    w.rmax = o; o += rm;
    // Y-sweep tables normalised per Y coordinate (column max 1) and the removed
    // log factors c_a[y_a] = max_x -(x_a - y_a)^2 / eps
    w.K0y = o; o += (int64_t)nw0 * ny0;
    w.K1y = o; o += (int64_t)nw1 * ny1;
    w.c0 = o; o += ny0;
    w.c1 = o; o += ny1;
    w.total = o;
    return w;
}

struct Ws {
    double *xc0, *xc1, *yc0, *yc1;
    double *alpha, *u, *L, *mu, *tx, *lmu, *wx;
    double *beta, *ty, *wy;
    double *K0, *K1, *mid, *rmax;
    double *K0y, *K1y, *c0, *c1;
    const double* lnu;   // global: log nu on the window (contiguous copy)
    double* m;           // global: background density on the window
    int64_t ms;
};

__device__ inline Ws ws_bind(double* base, const WsLayout& l) {
    Ws w;
    w.xc0 = base + l.xc0; w.xc1 = base + l.xc1; w.yc0 = base + l.yc0; w.yc1 = base + l.yc1;
    w.alpha = base + l.alpha; w.u = base + l.u; w.L = base + l.L; w.mu = base + l.mu;
    w.tx = base + l.tx; w.lmu = base + l.lmu; w.wx = base + l.wx;
    w.beta = base + l.beta; w.ty = base + l.ty; w.wy = base + l.wy;
    w.K0 = base + l.K0; w.K1 = base + l.K1;
    w.mid = base + l.mid; w.rmax = base + l.rmax;
    w.K0y = base + l.K0y; w.K1y = base + l.K1y; w.c0 = base + l.c0; w.c1 = base + l.c1;
    w.lnu = nullptr;
    w.m = nullptr;
    w.ms = l.midstride;
    return w;
}

__device__ inline CellWin load_win(const int32_t* d, int nw0, int nw1) {
    CellWin c;
    c.xo0 = d[1]; c.xe0 = d[2]; c.xo1 = d[3]; c.xe1 = d[4];
    c.yo0 = d[5]; c.ye0 = d[6]; c.yo1 = d[7]; c.ye1 = d[8];
    c.nx = nw0 * nw1;
    c.ny = c.ye0 * c.ye1;
    return c;
}

__device__ __forceinline__ double negsq(double a, double b, double eps) {
    const double d = a - b;
    return -(d * d) / eps;
}

// Two-pass log-sum-exp with exact skipping of terms that underflow to zero.
// Used by the log-domain (wide-window) path.

// ---- separable sweeps ------------------------------------------------------
//
// Both sweeps use the factorised kernel K(x,y) = K0[x0,y0] K1[x1,y1] with
// K_a = exp(-(x_a - y_a)^2 / eps) and one global max shift of the input
// vector (the reference's DenseKernel "matrix" form, cells.py via
// sinkhorn.py:91-130), i.e. FMA contractions instead of per-term exp.  An
// output whose shifted sum falls below kTiny may have lost its dominant
// terms to underflow, so it is recomputed exactly in the log domain; every
// other output carries all terms above 1e-308 and hence equals the
// log-domain value to rounding.  This makes the result independent of the
// window size (the reference switches to a fully log-domain sweep when
// min(-c/eps) <= -700; both of its modes agree with this one to rounding).

constexpr double kTiny = 1e-290;

// Exact 1D log-sum-exp  log sum_k exp(v[k*stride] - (p - q[k])^2 / eps)  (two passes).
__device__ __forceinline__ double lse1d(const double* v, int64_t stride, int n, double p,
                                        const double* q, double eps) {
    double mx = kNegInf;
    for (int k = 0; k < n; ++k) mx = fmax(mx, v[k * stride] + negsq(p, q[k], eps));
    if (!isfinite(mx)) return kNegInf;
    double s = 0.0;
    for (int k = 0; k < n; ++k) {
        const double t = v[k * stride] + negsq(p, q[k], eps) - mx;
        if (t > -760.0) s += exp(t);
    }
    return log(s) + mx;
}

// One separable stage, in place of the reference's per-axis _lse
// (sinkhorn.py:57-67 / 159-175):
//   out[r][o] = log sum_k exp(in[r][k] - (p[o] - q[k])^2 / eps),  r < R, o < O, k < Kn,
// stored at out[o*R + r].  One warp per row: the warp takes the row max,
// writes its shifted weights, then contracts them against the kernel table
// Kt[o*so + k*sk] = exp(-(p[o]-q[k])^2/eps) with FMAs (a lane group per
// output).  An output whose shifted sum is below kTiny may have lost its
// dominant terms to underflow and is recomputed by the exact 1D
// log-sum-exp.  PREP(r, row) may fill row r of `in` first (warp-private).
// One block barrier at the end.
template <class Prep>
__device__ void lse_stage(double* in, int R, int Kn, const double* Kt, int so, int sk, int O,
                          const double* p, const double* q, double eps, double* wts, double* out,
                          Prep prep) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lanes per output: largest power of two with O * g <= 32 (at most 8)
    int g = 1;
    while (g < 8 && O * g * 2 <= 32) g *= 2;
    const int slots = 32 / g;
    const int sub = lane % g, slot = lane / g;
    for (int r = warp; r < R; r += DD_NW) {
        double* ir = in + (int64_t)r * Kn;
        prep(r, ir);
        __syncwarp();
        double m = kNegInf;
        for (int k = lane; k < Kn; k += 32) m = fmax(m, ir[k]);
        m = warp_max_all(m);
        double* wr = wts + (int64_t)r * Kn;
        const bool fin = isfinite(m);
        for (int k = lane; k < Kn; k += 32) wr[k] = fin ? exp(ir[k] - m) : 0.0;
        __syncwarp();
        for (int ob = 0; ob < O; ob += slots) {
            const int o = ob + slot;
            double s0 = 0.0, s1 = 0.0;
            if (o < O && fin) {
                const double* kr = Kt + (int64_t)o * so;
                int k = sub;
                for (; k + g < Kn; k += 2 * g) {
                    s0 = fma(wr[k], kr[(int64_t)k * sk], s0);
                    s1 = fma(wr[k + g], kr[(int64_t)(k + g) * sk], s1);
                }
                if (k < Kn) s0 = fma(wr[k], kr[(int64_t)k * sk], s0);
            }
            double sacc = s0 + s1;
            for (int d = g / 2; d > 0; d >>= 1) sacc += __shfl_down_sync(0xffffffffu, sacc, d, g);
            if (o < O && sub == 0) {
                double res;
                if (!fin) res = kNegInf;
                else if (sacc >= kTiny) res = log(sacc) + m;
                else res = lse1d(ir, 1, Kn, p[o], q, eps);
                out[(int64_t)o * R + r] = res;
            }
        }
        __syncwarp();
    }
    __syncthreads();
}

struct NoPrep {
    __device__ void operator()(int, double*) const {}
};

// L[x] = log sum_y exp(bv[y] - c(x,y)/eps), bv = beta/eps + lnu (built row by row
// into ty).  Stage 1 reduces y1 per row y0 -> T[x1][y0], stage 2 reduces y0 per
// x1 -> out[x0][x1].  K1 is [x1][y1], K0 is [x0][y0].
__device__ void cell_lse_x_staged(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                                  double* out) {
    const int ny0 = c.ye0, ny1 = c.ye1;
    double* T = w.mid;                  // [nw1][ny0]
    double* W = w.mid + w.ms;           // stage-2 weights
    const double* beta = w.beta;
    const double* lnu = w.lnu;
    auto prep = [=](int r, double* row) {
        const int lane = threadIdx.x & 31;
        for (int k = lane; k < ny1; k += 32) {
            const int64_t y = (int64_t)r * ny1 + k;
            row[k] = beta[y] / eps + lnu[y];
        }
    };
    lse_stage(w.ty, ny0, ny1, w.K1, ny1, 1, nw1, w.xc1, w.yc1, eps, w.wy, T, prep);
    lse_stage(T, nw1, ny0, w.K0, ny0, 1, nw0, w.xc0, w.yc0, eps, W, out, NoPrep());
}

// alpha = -ratio * L (row by row, fused), then
// z[y] = log sum_x exp(av[x] - c(x,y)/eps), av = alpha/eps + lmu (rows into tx).
__device__ void cell_lse_y_staged(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                                  double ratio, double* out) {
    const int ny0 = c.ye0, ny1 = c.ye1;
    double* T = w.mid;                  // [ny1][nw0]
    double* W = w.mid + w.ms;
    double* alpha = w.alpha;
    const double* L = w.L;
    const double* lmu = w.lmu;
    auto prep = [=](int r, double* row) {
        const int lane = threadIdx.x & 31;
        for (int k = lane; k < nw1; k += 32) {
            const int x = r * nw1 + k;
            if (ratio != 0.0) alpha[x] = -ratio * L[x];
            row[k] = alpha[x] / eps + lmu[x];
        }
    };
    lse_stage(w.tx, nw0, nw1, w.K1, 1, ny1, ny1, w.yc1, w.xc1, eps, w.wx, T, prep);
    lse_stage(T, ny1, nw0, w.K0, 1, ny0, ny0, w.yc0, w.xc0, eps, W, out, NoPrep());
}

// Fast path of both sweeps: one global max shift of the input vector and two
// FMA contractions through the factorised kernel, using the Y-normalised tables
// K_a^y = K_a exp(-c_a(y_a)) (the X sweep adds c0 + c1 to its Y input, the Y sweep
// adds them to its outputs) (the reference DenseKernel's
// "matrix" evaluation, sinkhorn.py:91-130, done axis by axis).  If any output's
// shifted sum is below kTiny it may have lost terms to underflow, and the
// whole sweep is redone by the stage-wise stabilised path above, so every
// output equals the log-domain value to rounding.
struct SweepScratch {
    double* redm;   // [2*DD_NW] block-max buffers
    int* flag;      // shared underflow flag
    int* par;       // block-max buffer parity
    double* f32s;   // fp32 mode: slopes the current tables use [X0, X1, Y0, Y1], valid [X, Y]
};

// gred != nullptr: the cell gap test's per-thread terms (cells.py:336-340) are summed in
// the output loop (thread t owns outputs t, t + DD_NT, ... in both loops, so the sums are
// the separate loop's bit for bit) and each warp's sum is published in gred[wid] before
// the sweep's final barrier.  Returns false when an output underflowed (the sweep was
// redone stage-wise and the fused terms are void).
__device__ bool cell_lse_x(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                           double* out, SweepScratch sc, double* gred = nullptr,
                           double lam = 1.0) {
    const int ny0 = c.ye0, ny1 = c.ye1, ny = c.ny, nx = nw0 * nw1;
    double lmax = kNegInf;
    int y = threadIdx.x;
    // four nodes per pass: all loads issue before the first store (the arrays are
    // distinct, which the compiler cannot prove through the workspace pointers)
    for (; y + 3 * DD_NT < ny; y += 4 * DD_NT) {
        double bt[4], ln[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) { bt[j] = w.beta[y + j * DD_NT]; ln[j] = w.lnu[y + j * DD_NT]; }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int yy = y + j * DD_NT, y0 = yy / ny1;
            const double bv = bt[j] / eps + ln[j] + (w.c0[y0] + w.c1[yy - y0 * ny1]);
            w.ty[yy] = bv;
            lmax = fmax(lmax, bv);
        }
    }
    for (; y < ny; y += DD_NT) {
        const int y0 = y / ny1;
        const double bv = w.beta[y] / eps + w.lnu[y] + (w.c0[y0] + w.c1[y - y0 * ny1]);
        w.ty[y] = bv;
        lmax = fmax(lmax, bv);
    }
    if (threadIdx.x == 0) *sc.flag = 0;
    double B = block_max1(lmax, sc.redm, *sc.par);
    if (!isfinite(B)) B = 0.0;
    y = threadIdx.x;
    for (; y + 3 * DD_NT < ny; y += 4 * DD_NT) {
        double tv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) tv[j] = w.ty[y + j * DD_NT];
#pragma unroll
        for (int j = 0; j < 4; ++j) w.wy[y + j * DD_NT] = exp(tv[j] - B);
    }
    for (; y < ny; y += DD_NT) w.wy[y] = exp(w.ty[y] - B);
    __syncthreads();
    *sc.par ^= 1;
    double* T = w.mid;   // [ny0][nw1]
    // A warp reads the same k of up to min(nw1, 16) K1 rows, ny1 doubles apart.  They
    // share banks when gcd(ny1, 16) * min(nw1, 16) > 16; then every row starts at its
    // own offset instead (below).
    const int low = ny1 & -ny1;
    const bool rotate = ny1 > 0 && (low < 16 ? low : 16) * (nw1 < 16 ? nw1 : 16) > 16;
    for (int o = threadIdx.x; o < ny0 * nw1; o += DD_NT) {
        const int y0 = o / nw1, x1 = o - y0 * nw1;
        const double* tr = w.wy + (int64_t)y0 * ny1;
        const double* kr = w.K1y + (int64_t)x1 * ny1;
        double s0 = 0.0, s1 = 0.0;
        if (!rotate) {
            // conflict-free row stride (e.g. ny1 odd)
            int k = 0;
            for (; k + 1 < ny1; k += 2) {
                s0 = fma(tr[k], kr[k], s0);
                s1 = fma(tr[k + 1], kr[k + 1], s1);
            }
            if (k < ny1) s0 = fma(tr[k], kr[k], s0);
        } else {
            // Each row starts at k = x1, which makes the effective stride ny1 + 1 (odd:
            // rotate implies ny1 even).  Only the summation order changes.
            int k = x1 % ny1;
            for (int j = 0; j < ny1; j += 2) {
                const int k1 = k + 1 == ny1 ? 0 : k + 1;
                s0 = fma(tr[k], kr[k], s0);
                s1 = fma(tr[k1], kr[k1], s1);
                k = k1 + 1 == ny1 ? 0 : k1 + 1;
            }
        }
        T[o] = s0 + s1;
    }
    __syncthreads();
    int bad = 0;
    double part = 0.0;
    for (int o = threadIdx.x; o < nx; o += DD_NT) {
        const int x0 = o / nw1, x1 = o - x0 * nw1;
        const double* kr = w.K0y + (int64_t)x0 * ny0;
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
        for (; k + 1 < ny0; k += 2) {
            s0 = fma(kr[k], T[(int64_t)k * nw1 + x1], s0);
            s1 = fma(kr[k + 1], T[(int64_t)(k + 1) * nw1 + x1], s1);
        }
        if (k < ny0) s0 = fma(kr[k], T[(int64_t)k * nw1 + x1], s0);
        const double sm = s0 + s1;
        if (sm >= kTiny) {
            const double Lv = log(sm) + B;
            out[o] = Lv;
            if (gred) {
                const double mu = w.mu[o];
                if (mu > 0) {
                    const double a = w.alpha[o];
                    const double lr = a / eps + Lv;
                    const double px = mu * exp(lr);
                    const double ref = mu * exp(-a / lam);
                    part += px * (lr + a / lam) - px + ref;
                }
            }
        } else {
            ++bad;
        }
    }
    if (gred) {
        part = warp_sum(part);
        if ((threadIdx.x & 31) == 0) gred[threadIdx.x >> 5] = part;
    }
    if (bad) *sc.flag = 1;
    __syncthreads();
    if (*sc.flag) {
        cell_lse_x_staged(w, c, nw0, nw1, eps, out);
        return false;
    }
    return true;
}


__device__ void cell_lse_y(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                           double ratio, double* out, SweepScratch sc) {
    const int ny0 = c.ye0, ny1 = c.ye1, ny = c.ny, nx = nw0 * nw1;
    double lmax = kNegInf;
    for (int x = threadIdx.x; x < nx; x += DD_NT) {
        if (ratio != 0.0) w.alpha[x] = -ratio * w.L[x];
        const double av = w.alpha[x] / eps + w.lmu[x];
        w.tx[x] = av;
        lmax = fmax(lmax, av);
    }
    if (threadIdx.x == 0) *sc.flag = 0;
    double A = block_max1(lmax, sc.redm, *sc.par);
    if (!isfinite(A)) A = 0.0;
    for (int x = threadIdx.x; x < nx; x += DD_NT) w.wx[x] = exp(w.tx[x] - A);
    __syncthreads();
    *sc.par ^= 1;
    double* T = w.mid;   // [nw0][ny1]
    for (int o = threadIdx.x; o < nw0 * ny1; o += DD_NT) {
        const int x0 = o / ny1, y1 = o - x0 * ny1;
        const double* tr = w.wx + (int64_t)x0 * nw1;
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
        for (; k + 1 < nw1; k += 2) {
            s0 = fma(tr[k], w.K1y[(int64_t)k * ny1 + y1], s0);
            s1 = fma(tr[k + 1], w.K1y[(int64_t)(k + 1) * ny1 + y1], s1);
        }
        if (k < nw1) s0 = fma(tr[k], w.K1y[(int64_t)k * ny1 + y1], s0);
        T[o] = s0 + s1;
    }
    __syncthreads();
    int bad = 0;
    // two outputs per pass: their FMA chains and logs are independent, so the
    // scheduler overlaps the two log latencies (same arithmetic per output)
    int o = threadIdx.x;
    for (; o + DD_NT < ny; o += 2 * DD_NT) {
        const int o2 = o + DD_NT;
        const int y0 = o / ny1, y1 = o - y0 * ny1;
        const int z0 = o2 / ny1, z1 = o2 - z0 * ny1;
        double s0 = 0.0, s1 = 0.0, u0 = 0.0, u1 = 0.0;
        int k = 0;
        for (; k + 1 < nw0; k += 2) {
            s0 = fma(w.K0y[(int64_t)k * ny0 + y0], T[(int64_t)k * ny1 + y1], s0);
            u0 = fma(w.K0y[(int64_t)k * ny0 + z0], T[(int64_t)k * ny1 + z1], u0);
            s1 = fma(w.K0y[(int64_t)(k + 1) * ny0 + y0], T[(int64_t)(k + 1) * ny1 + y1], s1);
            u1 = fma(w.K0y[(int64_t)(k + 1) * ny0 + z0], T[(int64_t)(k + 1) * ny1 + z1], u1);
        }
        if (k < nw0) {
            s0 = fma(w.K0y[(int64_t)k * ny0 + y0], T[(int64_t)k * ny1 + y1], s0);
            u0 = fma(w.K0y[(int64_t)k * ny0 + z0], T[(int64_t)k * ny1 + z1], u0);
        }
        const double sm = s0 + s1, um = u0 + u1;
        const double ls = log(sm), lu = log(um);
        if (sm >= kTiny) out[o] = ls + A + (w.c0[y0] + w.c1[y1]);
        else ++bad;
        if (um >= kTiny) out[o2] = lu + A + (w.c0[z0] + w.c1[z1]);
        else ++bad;
    }
    for (; o < ny; o += DD_NT) {
        const int y0 = o / ny1, y1 = o - y0 * ny1;
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
        for (; k + 1 < nw0; k += 2) {
            s0 = fma(w.K0y[(int64_t)k * ny0 + y0], T[(int64_t)k * ny1 + y1], s0);
            s1 = fma(w.K0y[(int64_t)(k + 1) * ny0 + y0], T[(int64_t)(k + 1) * ny1 + y1], s1);
        }
        if (k < nw0) s0 = fma(w.K0y[(int64_t)k * ny0 + y0], T[(int64_t)k * ny1 + y1], s0);
        const double sm = s0 + s1;
        if (sm >= kTiny) out[o] = log(sm) + A + (w.c0[y0] + w.c1[y1]);
        else ++bad;
    }
    if (bad) *sc.flag = 1;
    __syncthreads();
    // alpha is already updated; the staged redo must not apply the update twice
    if (*sc.flag) {
        cell_lse_y_staged(w, c, nw0, nw1, eps, 0.0, out);
    }
}

// ---- fp32 mode of the fast sweeps ----------------------------------------------
// The same two factorised contractions with the kernel tables, shifted weights and
// stage intermediates in fp32 (tables rounded from the fp64 values, weights by
// expf of the fp64-formed shifted argument, fmaf contractions, logf of the sum
// added to the fp64 shift).  Potentials, shifts, the Newton Y-step, the gap
// test and the epilogue stay fp64.  An output whose shifted fp32 sum is below
// kTinyF may have lost terms to fp32 underflow (< 1.2e-38, so dropped terms are
// < 1e-5 relative of such a sum for windows up to 1e4 nodes); the whole sweep is
// then redone by the fp64 stage-wise path.  north_star fp32 mode: 1e-4 relative.
constexpr float kTinyF = 1e-30f;

// sweeps of the fp32 fast path redone by the fp64 stage-wise path: [0] X, [1] Y
// (read and reset with dd_sweep_fallbacks)
__device__ unsigned long long g_sweep_fallbacks[4];

// Gradient-absorbed fp32 sweeps.  A cell's X-side potentials vary across the 2s x 2s
// window by (slope of alpha) x (window) / eps -- hundreds to thousands at fine eps --
// so one global shift leaves the dominant term of many outputs outside fp32's
// ~87-wide exponent range.  The linear part of that variation is moved into the
// per-axis tables, exactly (exp(v(x)) = exp(v(x) - s.x) exp(s.x) and exp(s.x) is
// separable):
//   X sweep  L[x] = log sum_y w[y] TX0[x0,y0] TX1[x1,y1] + B + th.x,
//            TXa = exp(-(xa-ya)^2/eps - th_a xa - cXa(ya)), w = exp(bv + cX0 + cX1 - B);
//   Y sweep  z[y] = log sum_x w[x] TY0[x0,y0] TY1[x1,y1] + A + cY0(y0) + cY1(y1),
//            TYa = exp(-(xa-ya)^2/eps + ps_a xa - cYa(ya)), w = exp(av - ps.x - A);
// with th = -slope(alpha)/ratio (the slope of L), ps = slope(alpha)/eps per node
// index, each column of a table normalised to max 1 (cXa, cYa in fp64).  The tables
// are rebuilt every sweep from the current alpha.
struct F32Tables {
    float* tx0; float* tx1;     // X-sweep tables [x0][y0], [x1][y1]
    float* ty0; float* ty1;     // Y-sweep tables
    double* cx0; double* cx1;   // X-sweep column shifts
    double* cy0; double* cy1;   // Y-sweep column shifts
};

__device__ __forceinline__ F32Tables f32_tables(const Ws& w, int nw0, int nw1, int ny0, int ny1) {
    F32Tables t;
    t.tx0 = reinterpret_cast<float*>(w.K0y);
    t.ty0 = t.tx0 + (int64_t)nw0 * ny0;
    t.tx1 = reinterpret_cast<float*>(w.K1y);
    t.ty1 = t.tx1 + (int64_t)nw1 * ny1;
    t.cx0 = w.c0;
    t.cx1 = w.c1;
    t.cy0 = w.mid + 2 * w.ms;
    t.cy1 = t.cy0 + ny0;
    return t;
}

// per-node-index slopes of alpha along each window axis (0 when not finite); one
// warp reduces, everyone reads sl[0..1] after the barrier
__device__ __forceinline__ void alpha_slopes(const double* alpha, int nw0, int nw1, double* sl) {
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        double d0 = 0.0, d1 = 0.0;
        if (nw0 > 1) for (int x1 = l; x1 < nw1; x1 += 32) d0 += alpha[(int64_t)(nw0 - 1) * nw1 + x1] - alpha[x1];
        if (nw1 > 1) for (int x0 = l; x0 < nw0; x0 += 32) d1 += alpha[(int64_t)x0 * nw1 + nw1 - 1] - alpha[(int64_t)x0 * nw1];
        d0 = warp_sum(d0);
        d1 = warp_sum(d1);
        if (l == 0) {
            const double s0 = nw0 > 1 ? d0 / ((double)nw1 * (nw0 - 1)) : 0.0;
            const double s1 = nw1 > 1 ? d1 / ((double)nw0 * (nw1 - 1)) : 0.0;
            sl[0] = isfinite(s0) ? s0 : 0.0;
            sl[1] = isfinite(s1) ? s1 : 0.0;
        }
    }
    __syncthreads();
}

// table T[xa][ya] = exp(-(xa-ya)^2/eps + s xa - c(ya)) with c(ya) the max over the
// window's xa (fp64).  f(x) = -(x0 + x h - y)^2/eps + s x is a concave parabola in the
// node index x, maximal at x* = (y - x0)/h + s eps/(2 h^2): the discrete max is at
// floor(x*) or floor(x*) + 1 clipped to the window, so c costs O(1) per ya.  The table
// entries need no fp64 division (fp32 accuracy suffices for them).
__device__ __forceinline__ void build_axis(const double* xc, const double* yc, int nw, int ny,
                                           double eps, double s, float* T, double* c) {
    const double inv_eps = 1.0 / eps;
    const double h = nw > 1 ? xc[1] - xc[0] : 1.0;
    for (int y = threadIdx.x; y < ny; y += DD_NT) {
        const double xs = (yc[y] - xc[0]) / h + s * eps / (2.0 * h * h);
        int k = (int)floor(fmin(fmax(xs, 0.0), (double)(nw - 1)));
        double m = kNegInf;
        for (int x = k; x <= k + 1 && x < nw; ++x) {
            const double d = xc[x] - yc[y];
            m = fmax(m, -(d * d) * inv_eps + s * (double)x);
        }
        c[y] = m;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < nw * ny; o += DD_NT) {
        const int x = o / ny, y = o - x * ny;
        const double d = xc[x] - yc[y];
        T[o] = expf((float)(-(d * d) * inv_eps + s * (double)x - c[y]));
    }
}

__device__ void cell_lse_x_f32(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                               double ratio, double* out, SweepScratch sc) {
    const int ny0 = c.ye0, ny1 = c.ye1, ny = c.ny, nx = nw0 * nw1;
    const F32Tables t = f32_tables(w, nw0, nw1, ny0, ny1);
    float* wyf = reinterpret_cast<float*>(w.wy);
    float* T = reinterpret_cast<float*>(w.mid);   // [ny0][nw1]
    __shared__ double sl[2];
    alpha_slopes(w.alpha, nw0, nw1, sl);
    // the tables are an exact rewrite for any slope; they are rebuilt only when the
    // slope of L has moved enough to widen the weights' range by more than ~8
    double th0 = -sl[0] / ratio, th1 = -sl[1] / ratio;   // slopes of L
    double* cur = sc.f32s;
    if (cur[4] == 0.0 || fabs(th0 - cur[0]) * (nw0 - 1) > 4.0 ||
        fabs(th1 - cur[1]) * (nw1 - 1) > 4.0) {
        build_axis(w.xc0, w.yc0, nw0, ny0, eps, -th0, t.tx0, t.cx0);
        build_axis(w.xc1, w.yc1, nw1, ny1, eps, -th1, t.tx1, t.cx1);
        __syncthreads();
        if (threadIdx.x == 0) { cur[0] = th0; cur[1] = th1; cur[4] = 1.0; }
    } else {
        th0 = cur[0];
        th1 = cur[1];
    }
    double lmax = kNegInf;
    __syncthreads();
    for (int y = threadIdx.x; y < ny; y += DD_NT) {
        const int y0 = y / ny1;
        const double bv = w.beta[y] / eps + w.lnu[y] + (t.cx0[y0] + t.cx1[y - y0 * ny1]);
        w.ty[y] = bv;
        lmax = fmax(lmax, bv);
    }
    if (threadIdx.x == 0) *sc.flag = 0;
    double B = block_max1(lmax, sc.redm, *sc.par);
    if (!isfinite(B)) B = 0.0;
    for (int y = threadIdx.x; y < ny; y += DD_NT) wyf[y] = expf((float)(w.ty[y] - B));
    __syncthreads();
    *sc.par ^= 1;
    // fp32: 32 words per bank cycle; rotate rows whose stride shares banks
    const int low = ny1 & -ny1;
    const bool rotate = ny1 > 0 && (low < 32 ? low : 32) * (nw1 < 32 ? nw1 : 32) > 32;
    for (int o = threadIdx.x; o < ny0 * nw1; o += DD_NT) {
        const int y0 = o / nw1, x1 = o - y0 * nw1;
        const float* tr = wyf + (int64_t)y0 * ny1;
        const float* kr = t.tx1 + (int64_t)x1 * ny1;
        float s0 = 0.f, s1 = 0.f;
        int k = rotate ? x1 % ny1 : 0;
        for (int j = 0; j + 1 < ny1; j += 2) {
            const int k1 = k + 1 == ny1 ? 0 : k + 1;
            s0 = fmaf(tr[k], kr[k], s0);
            s1 = fmaf(tr[k1], kr[k1], s1);
            k = k1 + 1 == ny1 ? 0 : k1 + 1;
        }
        if (ny1 & 1) s0 = fmaf(tr[k], kr[k], s0);
        T[o] = s0 + s1;
    }
    __syncthreads();
    int bad = 0;
    for (int o = threadIdx.x; o < nx; o += DD_NT) {
        const int x0 = o / nw1, x1 = o - x0 * nw1;
        const float* kr = t.tx0 + (int64_t)x0 * ny0;
        float s0 = 0.f, s1 = 0.f;
        int k = 0;
        for (; k + 1 < ny0; k += 2) {
            s0 = fmaf(kr[k], T[(int64_t)k * nw1 + x1], s0);
            s1 = fmaf(kr[k + 1], T[(int64_t)(k + 1) * nw1 + x1], s1);
        }
        if (k < ny0) s0 = fmaf(kr[k], T[(int64_t)k * nw1 + x1], s0);
        const float sm = s0 + s1;
        if (sm >= kTinyF) out[o] = (double)logf(sm) + B + (th0 * (double)x0 + th1 * (double)x1);
        else ++bad;
    }
    if (bad) *sc.flag = 1;
    __syncthreads();
    if (*sc.flag) {
        if (threadIdx.x == 0) atomicAdd(&g_sweep_fallbacks[0], 1ull);
        cell_lse_x_staged(w, c, nw0, nw1, eps, out);
    }
    if (threadIdx.x == 0) atomicAdd(&g_sweep_fallbacks[2], 1ull);
}

__device__ void cell_lse_y_f32(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                               double ratio, double* out, SweepScratch sc) {
    const int ny0 = c.ye0, ny1 = c.ye1, ny = c.ny, nx = nw0 * nw1;
    const F32Tables t = f32_tables(w, nw0, nw1, ny0, ny1);
    float* wxf = reinterpret_cast<float*>(w.wx);
    float* T = reinterpret_cast<float*>(w.mid);   // [nw0][ny1]
    for (int x = threadIdx.x; x < nx; x += DD_NT)
        if (ratio != 0.0) w.alpha[x] = -ratio * w.L[x];
    __syncthreads();
    __shared__ double sl[2];
    alpha_slopes(w.alpha, nw0, nw1, sl);
    double ps0 = sl[0] / eps, ps1 = sl[1] / eps;   // slopes of alpha/eps
    double* cur = sc.f32s;
    if (cur[5] == 0.0 || fabs(ps0 - cur[2]) * (nw0 - 1) > 4.0 ||
        fabs(ps1 - cur[3]) * (nw1 - 1) > 4.0) {
        build_axis(w.xc0, w.yc0, nw0, ny0, eps, ps0, t.ty0, t.cy0);
        build_axis(w.xc1, w.yc1, nw1, ny1, eps, ps1, t.ty1, t.cy1);
        __syncthreads();
        if (threadIdx.x == 0) { cur[2] = ps0; cur[3] = ps1; cur[5] = 1.0; }
    } else {
        ps0 = cur[2];
        ps1 = cur[3];
    }
    __syncthreads();
    double lmax = kNegInf;
    for (int x = threadIdx.x; x < nx; x += DD_NT) {
        const int x0 = x / nw1, x1 = x - x0 * nw1;
        const double av = w.alpha[x] / eps + w.lmu[x] - (ps0 * (double)x0 + ps1 * (double)x1);
        w.tx[x] = av;
        lmax = fmax(lmax, av);
    }
    if (threadIdx.x == 0) *sc.flag = 0;
    double A = block_max1(lmax, sc.redm, *sc.par);
    if (!isfinite(A)) A = 0.0;
    for (int x = threadIdx.x; x < nx; x += DD_NT) wxf[x] = expf((float)(w.tx[x] - A));
    __syncthreads();
    *sc.par ^= 1;
    for (int o = threadIdx.x; o < nw0 * ny1; o += DD_NT) {
        const int x0 = o / ny1, y1 = o - x0 * ny1;
        const float* tr = wxf + (int64_t)x0 * nw1;
        float s0 = 0.f, s1 = 0.f;
        int k = 0;
        for (; k + 1 < nw1; k += 2) {
            s0 = fmaf(tr[k], t.ty1[(int64_t)k * ny1 + y1], s0);
            s1 = fmaf(tr[k + 1], t.ty1[(int64_t)(k + 1) * ny1 + y1], s1);
        }
        if (k < nw1) s0 = fmaf(tr[k], t.ty1[(int64_t)k * ny1 + y1], s0);
        T[o] = s0 + s1;
    }
    __syncthreads();
    int bad = 0;
    for (int o = threadIdx.x; o < ny; o += DD_NT) {
        const int y0 = o / ny1, y1 = o - y0 * ny1;
        float s0 = 0.f, s1 = 0.f;
        int k = 0;
        for (; k + 1 < nw0; k += 2) {
            s0 = fmaf(t.ty0[(int64_t)k * ny0 + y0], T[(int64_t)k * ny1 + y1], s0);
            s1 = fmaf(t.ty0[(int64_t)(k + 1) * ny0 + y0], T[(int64_t)(k + 1) * ny1 + y1], s1);
        }
        if (k < nw0) s0 = fmaf(t.ty0[(int64_t)k * ny0 + y0], T[(int64_t)k * ny1 + y1], s0);
        const float sm = s0 + s1;
        if (sm >= kTinyF) out[o] = (double)logf(sm) + A + (t.cy0[y0] + t.cy1[y1]);
        else ++bad;
    }
    if (bad) *sc.flag = 1;
    __syncthreads();
    if (*sc.flag) {
        if (threadIdx.x == 0) atomicAdd(&g_sweep_fallbacks[1], 1ull);
        cell_lse_y_staged(w, c, nw0, nw1, eps, 0.0, out);
    }
    if (threadIdx.x == 0) atomicAdd(&g_sweep_fallbacks[3], 1ull);
}

template <bool F32>
__device__ __forceinline__ void sweep_x(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                                        double ratio, double* out, SweepScratch sc) {
    if constexpr (F32) cell_lse_x_f32(w, c, nw0, nw1, eps, ratio, out, sc);
    else cell_lse_x(w, c, nw0, nw1, eps, out, sc);
}

template <bool F32>
__device__ __forceinline__ void sweep_y(const Ws& w, const CellWin& c, int nw0, int nw1, double eps,
                                        double ratio, double* out, SweepScratch sc) {
    if constexpr (F32) cell_lse_y_f32(w, c, nw0, nw1, eps, ratio, out, sc);
    else cell_lse_y(w, c, nw0, nw1, eps, ratio, out, sc);
}

// Value of a boxed marginal at absolute node (r, q); zero outside.
__device__ __forceinline__ double boxed_at(const int32_t* box, const double* vals, int r, int q) {
    const int o0 = box[0], e0 = box[1], o1 = box[2], e1 = box[3];
    if (e0 <= 0 || e1 <= 0) return 0.0;
    const int a = r - o0, bq = q - o1;
    if (a < 0 || a >= e0 || bq < 0 || bq >= e1) return 0.0;
    return vals[(int64_t)a * e1 + bq];
}

// ---- the solve kernel -----------------------------------------------------

// ---- cluster variant of the Sinkhorn loop for large Y windows -----------------
//
// One thread-block cluster per composite cell (north_star: "one CTA, or a
// cluster for large composite cells").  The Y window's rows are split across
// the cluster's CTAs (each keeps its rows of beta / bv / weights in shared
// memory); the X-window state (alpha, L, mu) is replicated, and every CTA
// performs the identical X-side arithmetic so stopping decisions agree
// without communication.  Cross-CTA steps go through distributed shared
// memory in fixed rank order (deterministic): the global max of bv, the
// X-sweep's stage-2 partial sums over the row slices, and the gather of
// stage-1 rows for the exact fallback.  The loop's outputs (alpha, beta, L,
// stats) are written to the batch arenas; the single-CTA kernel then runs
// the epilogue for these cells in epilogue-only mode.

struct CluLayout {
    int64_t xc0, xc1, yc0, yc1, alpha, L, mu, lmu, tx, wx, beta, ty, wy, K0, K1, T1, P, T2, W, G,
        rmax, total;
};

__host__ __device__ inline CluLayout clu_layout(int nw0, int nw1, int ny0, int ny1, int rows) {
    CluLayout l;
    const int64_t nx = (int64_t)nw0 * nw1, nyl = (int64_t)rows * ny1;
    int64_t o = 0;
    l.xc0 = o; o += nw0;
    l.xc1 = o; o += nw1;
    l.yc0 = o; o += ny0;
    l.yc1 = o; o += ny1;
    l.alpha = o; o += nx;
    l.L = o; o += nx;
    l.mu = o; o += nx;
    l.lmu = o; o += nx;
    l.tx = o; o += nx;
    l.wx = o; o += nx;
    l.beta = o; o += nyl;
    l.ty = o; o += nyl;
    l.wy = o; o += nyl;
    l.K0 = o; o += (int64_t)nw0 * ny0;
    l.K1 = o; o += (int64_t)nw1 * ny1;
    l.T1 = o; o += (int64_t)rows * nw1;       // X sweep stage 1, local rows ([x1][row] when staged)
    l.P = o; o += 2 * nx;                     // double-buffered stage-2 partials
    l.T2 = o; o += (int64_t)nw0 * ny1;        // Y sweep stage 1 (replicated)
    int64_t wsz = (int64_t)nw1 * ny0;
    if ((int64_t)ny1 * nw0 > wsz) wsz = (int64_t)ny1 * nw0;
    if (nx > wsz) wsz = nx;
    if (nyl > wsz) wsz = nyl;
    l.W = o; o += wsz;                        // staged-stage weights
    l.G = o; o += (int64_t)nw1 * ny0;         // gathered stage-1 rows for the staged X fallback
    int64_t rm = ny0 > ny1 ? ny0 : ny1;
    if (nw0 > rm) rm = nw0;
    if (nw1 > rm) rm = nw1;
    l.rmax = o; o += rm;
    l.total = o;
    return l;
}

__device__ __forceinline__ int clu_row0(int ny0, int C, int rank) {
    return (int)(((int64_t)ny0 * rank) / C);
}

__global__ void __launch_bounds__(DD_NT, DD_CELL_MIN_BLOCKS) cell_loop_cluster_kernel(dd_geom g, dd_state s,
                                                                     dd_batch b,
                                                                     const int32_t* ids) {
    namespace cgx = cooperative_groups;
    cgx::cluster_group cluster = cgx::this_cluster();
    extern __shared__ double smem[];
    __shared__ double red[DD_NW + 1];
    __shared__ int redi[DD_NW + 1];
    __shared__ double xslot[4];          // scalar exchange slots (double-buffered pairs)
    __shared__ double xslot2[4];
    __shared__ int flag_sh;

    const int C = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int c = ids[blockIdx.x / C];
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t* off = b.offs + (int64_t)c * 4;
    const int nw0 = b.nxw0, nw1 = b.nxw1;
    const CellWin cw = load_win(d, nw0, nw1);
    const int j = d[0];
    const int nmem = d[9];
    const int32_t* mem = b.members + d[10];
    const int nx = cw.nx, ny0 = cw.ye0, ny1 = cw.ye1;
    const int r0 = clu_row0(ny0, C, rank), r1 = clu_row0(ny0, C, rank + 1);
    const int rows = r1 - r0;
    // layout sized for the largest row slice (identical in every CTA of the cluster)
    const CluLayout lay = clu_layout(nw0, nw1, ny0, ny1, (ny0 + C - 1) / C + 1);
    double* xc0 = smem + lay.xc0;
    double* xc1 = smem + lay.xc1;
    double* yc0 = smem + lay.yc0;
    double* yc1 = smem + lay.yc1;
    double* alpha = smem + lay.alpha;
    double* L = smem + lay.L;
    double* mu = smem + lay.mu;
    double* lmu = smem + lay.lmu;
    double* tx = smem + lay.tx;
    double* wx = smem + lay.wx;
    double* beta = smem + lay.beta;
    double* ty = smem + lay.ty;
    double* wy = smem + lay.wy;
    double* K0 = smem + lay.K0;
    double* K1 = smem + lay.K1;
    double* T1 = smem + lay.T1;
    double* P = smem + lay.P;
    double* T2 = smem + lay.T2;
    double* W = smem + lay.W;
    double* G = smem + lay.G;
    const double eps = g.eps, lam = g.lam;
    const double ratio = eps * lam / (eps + lam);
    const int tid = threadIdx.x;
    const int64_t yoff = off[0];
    const int64_t ybase = yoff + (int64_t)r0 * ny1;   // this CTA's first node in the y arenas
    const int nyl = rows * ny1;
    const double* lnu = b.lnuw + ybase;
    const double* mg = b.mdens + ybase;
    const double* lmg = b.lmw + ybase;

    // cluster helpers (fixed rank order => deterministic)
    int spar = 0;
    auto csum = [&](double v) -> double {
        v = block_sum(v, red);
        if (tid == 0) xslot[spar] = v;
        cluster.sync();
        double t = 0.0;
        for (int r = 0; r < C; ++r) t += *cluster.map_shared_rank(&xslot[spar], r);
        spar ^= 1;
        return t;
    };
    // two sums in one cluster exchange (own slot pair, same parity discipline)
    auto csum2 = [&](double v0, double v1, double& o1) -> double {
        v0 = block_sum(v0, red);
        v1 = block_sum(v1, red);
        if (tid == 0) { xslot2[2 * spar] = v0; xslot2[2 * spar + 1] = v1; }
        cluster.sync();
        double t0 = 0.0, t1 = 0.0;
        for (int r = 0; r < C; ++r) {
            t0 += *cluster.map_shared_rank(&xslot2[2 * spar], r);
            t1 += *cluster.map_shared_rank(&xslot2[2 * spar + 1], r);
        }
        spar ^= 1;
        o1 = t1;
        return t0;
    };
    auto cmax = [&](double v) -> double {
        v = block_max(v, red);
        if (tid == 0) xslot[2 + spar] = v;
        cluster.sync();
        double t = kNegInf;
        for (int r = 0; r < C; ++r) t = fmax(t, *cluster.map_shared_rank(&xslot[2 + spar], r));
        spar ^= 1;
        return t;
    };

    for (int i = tid; i < nw0; i += DD_NT) xc0[i] = g.x_org0 + g.x_dx * (double)(cw.xo0 + i);
    for (int i = tid; i < nw1; i += DD_NT) xc1[i] = g.x_org1 + g.x_dx * (double)(cw.xo1 + i);
    for (int i = tid; i < ny0; i += DD_NT) yc0[i] = g.y_org0 + g.y_dx * (double)(cw.yo0 + i);
    for (int i = tid; i < ny1; i += DD_NT) yc1[i] = g.y_org1 + g.y_dx * (double)(cw.yo1 + i);
    const bool has_dual = s.d_has[j] != 0;
    double musum_part = 0.0;
    for (int x = tid; x < nx; x += DD_NT) {
        const int x0 = x / nw1, x1 = x - x0 * nw1;
        const int r = cw.xo0 + x0, q = cw.xo1 + x1;
        double m = 0.0, lm = kNegInf;
        if (r >= 0 && r < g.nx0 && q >= 0 && q < g.nx1) {
            const int64_t id = (int64_t)r * g.nx1 + q;
            m = s.mu[id];
            lm = s.log_mu[id];
        }
        mu[x] = m;
        lmu[x] = lm;
        alpha[x] = has_dual ? s.d_alpha[(int64_t)j * nx + x] : 0.0;
        musum_part += m;
    }
    const double musum = block_sum(musum_part, red);   // replicated, identical in every CTA
    const double thr = b.delta * musum;
    const int32_t* dbox = s.d_box + (int64_t)j * 4;
    const double* dbeta = s.d_beta + (int64_t)j * s.d_cap;
    int nclamp = 0, anym = 0;
    for (int yl = tid; yl < nyl; yl += DD_NT) {
        const int y0 = r0 + yl / ny1, y1 = yl % ny1;
        const int rr = cw.yo0 + y0, q = cw.yo1 + y1;
        const int64_t id = (int64_t)rr * g.ny1 + q;
        const double nu = s.nu[id];
        b.lnuw[ybase + yl] = s.log_nu[id];
        double cs = 0.0;
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            cs += boxed_at(s.ybox + (int64_t)i * 4, s.yval + (int64_t)i * s.cap, rr, q);
        }
        const double pw = b.snapshot[id];
        const double diff = pw - cs;
        if (diff < -1e-12 * fmax(pw, cs)) ++nclamp;
        const double mm = fmax(diff, 0.0) / nu;
        b.mdens[ybase + yl] = mm;
        b.lmw[ybase + yl] = log(mm);
        if (mm != 0.0) anym = 1;
        beta[yl] = has_dual ? boxed_at(dbox, dbeta, rr, q) : 0.0;
    }
    const double n_clamped = csum((double)nclamp);
    const bool has_m = cmax((double)anym) > 0.0;
    for (int o = tid; o < nw0 * ny0; o += DD_NT) {
        const int x0 = o / ny0, y0 = o - x0 * ny0;
        K0[o] = exp(negsq(xc0[x0], yc0[y0], eps));
    }
    for (int o = tid; o < nw1 * ny1; o += DD_NT) {
        const int x1 = o / ny1, y1 = o - x1 * ny1;
        K1[o] = exp(negsq(xc1[x1], yc1[y1], eps));
    }
    __syncthreads();

    int ppar = 0;
    // X sweep: L[x] = log sum_y exp(bv - c/eps), bv = beta/eps + lnu; rows split.
    auto lse_x = [&]() {
        double lmax = kNegInf;
        for (int yl = tid; yl < nyl; yl += DD_NT) {
            const double bv = beta[yl] / eps + lnu[yl];
            ty[yl] = bv;
            lmax = fmax(lmax, bv);
        }
        double B = cmax(lmax);
        if (!isfinite(B)) B = 0.0;
        for (int yl = tid; yl < nyl; yl += DD_NT) wy[yl] = exp(ty[yl] - B);
        __syncthreads();
        for (int o = tid; o < rows * nw1; o += DD_NT) {
            const int rl = o / nw1, x1 = o - rl * nw1;
            const double* tr = wy + (int64_t)rl * ny1;
            const double* kr = K1 + (int64_t)x1 * ny1;
            double s0 = 0.0, s1 = 0.0;
            int k = 0;
            for (; k + 1 < ny1; k += 2) {
                s0 = fma(tr[k], kr[k], s0);
                s1 = fma(tr[k + 1], kr[k + 1], s1);
            }
            if (k < ny1) s0 = fma(tr[k], kr[k], s0);
            T1[o] = s0 + s1;
        }
        __syncthreads();
        double* Pp = P + ppar * nx;
        for (int x = tid; x < nx; x += DD_NT) {
            const int x0 = x / nw1, x1 = x - x0 * nw1;
            const double* kr = K0 + (int64_t)x0 * ny0 + r0;
            double s0 = 0.0, s1 = 0.0;
            int k = 0;
            for (; k + 1 < rows; k += 2) {
                s0 = fma(kr[k], T1[(int64_t)k * nw1 + x1], s0);
                s1 = fma(kr[k + 1], T1[(int64_t)(k + 1) * nw1 + x1], s1);
            }
            if (k < rows) s0 = fma(kr[k], T1[(int64_t)k * nw1 + x1], s0);
            Pp[x] = s0 + s1;
        }
        cluster.sync();
        int bad = 0;
        for (int x = tid; x < nx; x += DD_NT) {
            double sm = 0.0;
            for (int r = 0; r < C; ++r) sm += cluster.map_shared_rank(Pp, r)[x];
            if (sm >= kTiny) L[x] = log(sm) + B;
            else bad = 1;
        }
        ppar ^= 1;
        if (tid == 0) flag_sh = 0;
        __syncthreads();
        if (bad) flag_sh = 1;
        __syncthreads();
        if (flag_sh) {   // identical in every CTA (replicated arithmetic)
            // staged: stage 1 over own rows -> T1[x1][row], gather all rows -> G[x1][y0],
            // stage 2 per x1 row -> L
            lse_stage(ty, rows, ny1, K1, ny1, 1, nw1, xc1, yc1, eps, W, T1, NoPrep());
            cluster.sync();
            for (int t = tid; t < nw1 * ny0; t += DD_NT) {
                const int x1 = t / ny0, y0 = t - x1 * ny0;
                int r = 0;
                while (r + 1 < C && y0 >= clu_row0(ny0, C, r + 1)) ++r;
                const int rr0 = clu_row0(ny0, C, r), rrows = clu_row0(ny0, C, r + 1) - rr0;
                G[t] = cluster.map_shared_rank(T1, r)[(int64_t)x1 * rrows + (y0 - rr0)];
            }
            cluster.sync();
            lse_stage(G, nw1, ny0, K0, ny0, 1, nw0, xc0, yc0, eps, W, L, NoPrep());
        }
    };

    bool converged = false, have_first = false;
    double gap = __builtin_huge_val(), first_gap = 0.0;
    int iters = 0, newton_clamped = 0, stag_k = 0;
    long long newton_steps = 0;
    const long long t0c = clock64();
    for (int k = 1; k <= b.max_iters; ++k) {
        lse_x();
        if (k >= 2) {
            double part = 0.0;
            for (int x = tid; x < nx; x += DD_NT) {
                const double m = mu[x];
                if (m > 0) {
                    const double a = alpha[x];
                    const double lr = a / eps + L[x];
                    const double px = m * exp(lr);
                    const double ref = m * exp(-a / lam);
                    part += px * (lr + a / lam) - px + ref;
                }
            }
            gap = lam * block_sum(part, red);   // replicated
            if (!have_first) { first_gap = gap; have_first = true; }
            if (gap / lam <= thr) { converged = true; break; }
        }
        // Y sweep (replicated stage 1, own rows in stage 2), then Newton on own rows
        double lmax = kNegInf;
        for (int x = tid; x < nx; x += DD_NT) {
            alpha[x] = -ratio * L[x];
            const double av = alpha[x] / eps + lmu[x];
            tx[x] = av;
            lmax = fmax(lmax, av);
        }
        double A = block_max(lmax, red);
        if (!isfinite(A)) A = 0.0;
        for (int x = tid; x < nx; x += DD_NT) wx[x] = exp(tx[x] - A);
        __syncthreads();
        for (int o = tid; o < nw0 * ny1; o += DD_NT) {
            const int x0 = o / ny1, y1 = o - x0 * ny1;
            const double* tr = wx + (int64_t)x0 * nw1;
            double s0 = 0.0, s1 = 0.0;
            int kk = 0;
            for (; kk + 1 < nw1; kk += 2) {
                s0 = fma(tr[kk], K1[(int64_t)kk * ny1 + y1], s0);
                s1 = fma(tr[kk + 1], K1[(int64_t)(kk + 1) * ny1 + y1], s1);
            }
            if (kk < nw1) s0 = fma(tr[kk], K1[(int64_t)kk * ny1 + y1], s0);
            T2[o] = s0 + s1;
        }
        __syncthreads();
        int bad = 0;
        for (int yl = tid; yl < nyl; yl += DD_NT) {
            const int y0 = r0 + yl / ny1, y1 = yl % ny1;
            double s0 = 0.0, s1 = 0.0;
            int kk = 0;
            for (; kk + 1 < nw0; kk += 2) {
                s0 = fma(K0[(int64_t)kk * ny0 + y0], T2[(int64_t)kk * ny1 + y1], s0);
                s1 = fma(K0[(int64_t)(kk + 1) * ny0 + y0], T2[(int64_t)(kk + 1) * ny1 + y1], s1);
            }
            if (kk < nw0) s0 = fma(K0[(int64_t)kk * ny0 + y0], T2[(int64_t)kk * ny1 + y1], s0);
            const double sm = s0 + s1;
            if (sm >= kTiny) ty[yl] = log(sm) + A;
            else bad = 1;
        }
        if (tid == 0) flag_sh = 0;
        __syncthreads();
        if (bad) flag_sh = 1;
        __syncthreads();
        if (flag_sh) {   // local: this CTA's rows only
            lse_stage(tx, nw0, nw1, K1, 1, ny1, ny1, yc1, xc1, eps, W, T2, NoPrep());
            lse_stage(T2, ny1, nw0, K0 + r0, 1, ny0, rows, yc0 + r0, xc0, eps, W, ty, NoPrep());
        }
        int ndeg = 0;
        int moved = 0;
        for (int yl = tid; yl < nyl; yl += DD_NT) {
            int dg = 0;
            const double ob = beta[yl];
            const double nb = newton_node(ty[yl], mg[yl], has_m, ob, eps, lam, b.newton_tol,
                                          b.newton_max_iters, &dg, &newton_steps, nullptr,
                                          lmg[yl]);
            moved |= (nb != ob) ? 1 : 0;
            beta[yl] = nb;
            ndeg += dg;
        }
        // cluster-wide clamped-node count of this iteration (max over iterations, as
        // the single-CTA kernel and the reference) and whether any beta moved
        double n_moved = 0.0;
        const double nd = csum2((double)ndeg, (double)moved, n_moved);
        newton_clamped = max(newton_clamped, (int)nd);
        iters = k;
        if (b.skip_stagnant && k >= 2 && n_moved == 0.0) {
            stag_k = k;   // see the single-CTA kernel
            iters = b.max_iters;
            break;
        }
    }
    __syncthreads();
    if (!converged) {
        lse_x();
        double part = 0.0;
        for (int x = tid; x < nx; x += DD_NT) {
            const double m = mu[x];
            if (m > 0) {
                const double a = alpha[x];
                const double lr = a / eps + L[x];
                const double px = m * exp(lr);
                const double ref = m * exp(-a / lam);
                part += px * (lr + a / lam) - px + ref;
            }
        }
        gap = lam * block_sum(part, red);
        if (!have_first) { first_gap = gap; have_first = true; }
        converged = gap / lam <= thr;
        if (converged && stag_k) iters = stag_k;
    }
    const double cyc = (double)(clock64() - t0c);
    const double nst = csum((double)newton_steps);
    const double ncl = (double)newton_clamped;
    for (int yl = tid; yl < nyl; yl += DD_NT) b.beta[ybase + yl] = beta[yl];
    if (rank == 0) {
        for (int x = tid; x < nx; x += DD_NT) {
            b.alpha[(int64_t)c * nx + x] = alpha[x];
            b.lout[(int64_t)c * nx + x] = L[x];
        }
        if (tid == 0) {
            double* cs = b.cstat + (int64_t)c * 8;
            cs[0] = gap;
            cs[1] = first_gap;
            cs[2] = (double)iters;
            cs[3] = converged ? 1.0 : 0.0;
            cs[4] = n_clamped;
            cs[5] = ncl;
            double* c2 = b.cstat2 + (int64_t)c * 8;
            c2[2] = cyc;
            c2[3] = nst;
            c2[4] = (double)(stag_k ? stag_k : iters);
        }
    }
    cluster.sync();   // keep every CTA's shared memory alive until remote reads are done
}

// kPass 0: cells whose workspace fits the launch's shared memory (others exit);
// kPass 1: the remaining (large-window) cells, workspace in the global arena,
//          compiled as a separate function so it can run with a max-L1
//          carveout on a second stream, concurrently with pass 0.
// kLoop: the Sinkhorn loop only (window assembly, tables, loop, capped-cell final
// sweep), outputs as the cluster kernel leaves them (alpha, beta, lout, cstat); the
// epilogue then runs in the kPass 0 kernel for cells flagged 4.  Compiled for two
// CTAs per SM (<= 64 registers): the epilogue's register pressure is not in it.
template <int kPass, bool kF32, bool kLoop>
__global__ void __launch_bounds__(DD_NT, (kLoop ? 2 : (kPass == 0 ? DD_CELL_MIN_BLOCKS : 1)))
    cell_solve_kernel(dd_geom g, dd_state s, dd_batch b) {
    extern __shared__ double smem[];
    __shared__ double red[DD_NW + 1];
    __shared__ int redi[DD_NW + 1];
    __shared__ int sh_flag[4];

    // CTAs are dispatched in blockIdx order: the host orders cells by expected
    // cost (longest first) so the capped tail does not start last
    const int c = b.order ? b.order[blockIdx.x] : blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t* off = b.offs + (int64_t)c * 4;
    const int nw0 = b.nxw0, nw1 = b.nxw1;
    const CellWin cw = load_win(d, nw0, nw1);
    const int j = d[0];
    const int nmem = d[9];
    const int32_t* mem = b.members + d[10];
    const int nx = cw.nx, ny = cw.ny, ny0 = cw.ye0, ny1 = cw.ye1;
    const WsLayout lay = ws_layout(nw0, nw1, ny0, ny1);
    // per-cell placement: shared memory when this cell's workspace fits the
    // launch's dynamic allocation, else its slot of the global arena
    if (d[11] & 2) return;   // cell owned by another rank (sharded solve)
    // cells whose Sinkhorn loop ran on a cluster (flag bit 0) take their epilogue in the
    // global-workspace pass whatever their size (the host may cluster small cells)
    if constexpr (kLoop) {
        if (!(d[11] & 4)) return;          // not a split (loop kernel + epilogue) cell
    }
    const bool in_smem = kLoop || (!(d[11] & 1) && b.smem_mode &&
                                   lay.total * (int64_t)sizeof(double) <= (int64_t)b.smem_bytes);
    if (in_smem != (kPass == 0)) return;
    // cells whose Sinkhorn loop ran in the cluster kernel (bit 0) or the loop kernel
    // (bit 2): epilogue only
    const bool epi = !kLoop && (d[11] & 5) != 0;
    double* base = in_smem ? smem : (b.work + off[2]);
    Ws w = ws_bind(base, lay);
    w.lnu = b.lnuw + off[0];
    w.m = b.mdens + off[0];
    const double eps = g.eps, lam = g.lam;
    const double ratio = eps * lam / (eps + lam);
    const int tid = threadIdx.x;
    const int64_t yoff = off[0];
    double* marena = b.marena + off[1];

    // coordinates
    for (int i = tid; i < nw0; i += DD_NT) w.xc0[i] = g.x_org0 + g.x_dx * (double)(cw.xo0 + i);
    for (int i = tid; i < nw1; i += DD_NT) w.xc1[i] = g.x_org1 + g.x_dx * (double)(cw.xo1 + i);
    for (int i = tid; i < ny0; i += DD_NT) w.yc0[i] = g.y_org0 + g.y_dx * (double)(cw.yo0 + i);
    for (int i = tid; i < ny1; i += DD_NT) w.yc1[i] = g.y_org1 + g.y_dx * (double)(cw.yo1 + i);

    // X window: mu, log mu (zero / -inf off the grid), warm-start alpha
    const bool has_dual = s.d_has[j] != 0;
    double musum_part = 0.0;
    for (int x = tid; x < nx; x += DD_NT) {
        const int x0 = x / nw1, x1 = x - x0 * nw1;
        const int r = cw.xo0 + x0, q = cw.xo1 + x1;
        double mu = 0.0, lmu = kNegInf;
        if (r >= 0 && r < g.nx0 && q >= 0 && q < g.nx1) {
            const int64_t id = (int64_t)r * g.nx1 + q;
            mu = s.mu[id];
            lmu = s.log_mu[id];
        }
        w.mu[x] = mu;
        w.lmu[x] = lmu;
        w.alpha[x] = epi ? b.alpha[(int64_t)c * nx + x]
                         : (has_dual ? s.d_alpha[(int64_t)j * nx + x] : 0.0);
        if (epi) w.L[x] = b.lout[(int64_t)c * nx + x];
        musum_part += mu;
    }
    const double musum = block_sum(musum_part, red);
    const double thr = b.delta * musum;

    // Y window: log nu, background density m, warm-start beta
    const int32_t* dbox = s.d_box + (int64_t)j * 4;
    const double* dbeta = s.d_beta + (int64_t)j * s.d_cap;
    int nclamp = 0;
    int anym = 0;
    for (int y = tid; y < ny; y += DD_NT) {
        const int y0 = y / ny1, y1 = y - y0 * ny1;
        const int r = cw.yo0 + y0, q = cw.yo1 + y1;
        const int64_t id = (int64_t)r * g.ny1 + q;
        const double nu = s.nu[id];
        b.lnuw[yoff + y] = s.log_nu[id];
        double cs = 0.0;
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            cs += boxed_at(s.ybox + (int64_t)i * 4, s.yval + (int64_t)i * s.cap, r, q);
        }
        const double pw = b.snapshot[id];
        const double diff = pw - cs;
        if (diff < -1e-12 * fmax(pw, cs)) ++nclamp;
        const double mm = fmax(diff, 0.0) / nu;
        b.mdens[yoff + y] = mm;
        // log m, taken once per solve for the Newton Y-step of every iteration
        b.lmw[yoff + y] = log(mm);
        if (mm != 0.0) anym = 1;
        w.beta[y] = epi ? b.beta[yoff + y] : (has_dual ? boxed_at(dbox, dbeta, r, q) : 0.0);
    }
    int n_clamped = (int)block_sum((double)nclamp, red);
    const bool has_m = block_max_i(anym, redi) != 0;
    const double* lmw = b.lmw + yoff;

    // per-axis kernel tables K_a = exp(-(x_a - y_a)^2 / eps) (entries may underflow;
    // the sweeps recompute affected outputs exactly)
    for (int o = tid; o < nw0 * ny0; o += DD_NT) {
        const int x0 = o / ny0, y0 = o - x0 * ny0;
        w.K0[o] = exp(negsq(w.xc0[x0], w.yc0[y0], eps));
    }
    for (int o = tid; o < nw1 * ny1; o += DD_NT) {
        const int x1 = o / ny1, y1 = o - x1 * ny1;
        w.K1[o] = exp(negsq(w.xc1[x1], w.yc1[y1], eps));
    }
    // Y-sweep tables: each Y coordinate's column divided by its largest entry, so
    // far Y nodes do not underflow to zero geometrically (the factor returns in the
    // log domain: out = log(sum) + A + c0[y0] + c1[y1])
    for (int y0 = tid; y0 < ny0; y0 += DD_NT) {
        double cm = kNegInf;
        for (int x0 = 0; x0 < nw0; ++x0) cm = fmax(cm, negsq(w.xc0[x0], w.yc0[y0], eps));
        w.c0[y0] = cm;
    }
    for (int y1 = tid; y1 < ny1; y1 += DD_NT) {
        double cm = kNegInf;
        for (int x1 = 0; x1 < nw1; ++x1) cm = fmax(cm, negsq(w.xc1[x1], w.yc1[y1], eps));
        w.c1[y1] = cm;
    }
    __syncthreads();
    for (int o = tid; o < nw0 * ny0; o += DD_NT) {
        const int x0 = o / ny0, y0 = o - x0 * ny0;
        if constexpr (!kF32) w.K0y[o] = exp(negsq(w.xc0[x0], w.yc0[y0], eps) - w.c0[y0]);
    }
    for (int o = tid; o < nw1 * ny1; o += DD_NT) {
        const int x1 = o / ny1, y1 = o - x1 * ny1;
        if constexpr (!kF32) w.K1y[o] = exp(negsq(w.xc1[x1], w.yc1[y1], eps) - w.c1[y1]);
    }
    __syncthreads();
    // ---- Sinkhorn loop (sinkhorn.py:361-432 / cells.py:320-348) ----
    // ---- Sinkhorn loop (skipped for cells solved by the cluster kernel) ----
    bool converged = false;
    bool have_first = false;
    double gap = __builtin_huge_val(), first_gap = 0.0;
    int iters = 0, newton_clamped = 0, stag_k = 0, exec_iters = 0;
    double t_loop_d = 0.0, nsteps = 0.0;
    if (epi) {
        const double* cs = b.cstat + (int64_t)c * 8;
        gap = cs[0];
        first_gap = cs[1];
        iters = (int)cs[2];
        converged = cs[3] != 0.0;
        n_clamped = (int)cs[4];
        newton_clamped = (int)cs[5];
        t_loop_d = b.cstat2[(int64_t)c * 8 + 2];
        nsteps = b.cstat2[(int64_t)c * 8 + 3];
    } else {
        const long long t_loop0 = clock64();
        long long newton_steps = 0;
        __shared__ double red2[2 * DD_NW];
        __shared__ double redm[2 * DD_NW];
        __shared__ int sweep_flag;
        int mpar = 0;
        __shared__ double f32s[6];
        if (tid < 6) f32s[tid] = 0.0;   // no fp32 tables built yet for this cell
        const SweepScratch sc{redm, &sweep_flag, &mpar, f32s};
        __shared__ int ndeg_sh[2];
        __shared__ int moved_sh[2];
        if (tid < 2) { ndeg_sh[tid] = 0; moved_sh[tid] = 0; }
        int par = 0;
        stag_k = 0;
        auto gap_terms = [&]() {
            double part = 0.0;
            for (int x = tid; x < nx; x += DD_NT) {
                const double mu = w.mu[x];
                if (mu > 0) {
                    const double a = w.alpha[x];
                    const double lr = a / eps + w.L[x];
                    const double px = mu * exp(lr);
                    const double ref = mu * exp(-a / lam);
                    part += px * (lr + a / lam) - px + ref;
                }
            }
            return block_sum1(part, red2, par);
        };
        auto newton_loop = [&](int cur) {
            int ndeg = 0;
            bool moved = false;
            for (int y = tid; y < ny; y += DD_NT) {
                int dg = 0;
                const double ob = w.beta[y];
                const double nb = newton_node(w.ty[y], w.m[y], has_m, ob, eps, lam,
                                              b.newton_tol, b.newton_max_iters, &dg,
                                              &newton_steps, nullptr, lmw[y], kF32);
                moved |= (nb != ob);
                w.beta[y] = nb;
                ndeg += dg;
            }
            if (ndeg) atomicAdd(&ndeg_sh[cur], ndeg);
            if (moved) moved_sh[cur] = 1;
            __syncthreads();
        };
        for (int k = 1; k <= b.max_iters; ++k) {
            const int cur = k & 1;
            if constexpr (!kF32) {
                // fp64: the gap terms ride in the X sweep's output loop and its final
                // barrier (the same per-thread sums and warp order as gap_terms)
                const bool fused = cell_lse_x(w, cw, nw0, nw1, eps, w.L, sc,
                                              k >= 2 ? red2 + par * DD_NW : nullptr, lam);
                if (k >= 2) {
                    double t = 0.0;
                    if (fused) {
                        const double* r = red2 + par * DD_NW;
#pragma unroll
                        for (int q = 0; q < DD_NW; ++q) t += r[q];
                    } else {
                        t = gap_terms();
                    }
                    gap = lam * t;
                    par ^= 1;
                    if (!have_first) { first_gap = gap; have_first = true; }
                    if (gap / lam <= thr) { converged = true; break; }
                }
                // alpha = -ratio L is fused into the Y sweep's row preparation
                sweep_y<kF32>(w, cw, nw0, nw1, eps, ratio, w.ty, sc);
                newton_loop(cur);
            } else {
                sweep_x<kF32>(w, cw, nw0, nw1, eps, ratio, w.L, sc);
                if (k >= 2) {
                    gap = lam * gap_terms();
                    par ^= 1;
                    if (!have_first) { first_gap = gap; have_first = true; }
                    if (gap / lam <= thr) { converged = true; break; }
                }
                sweep_y<kF32>(w, cw, nw0, nw1, eps, ratio, w.ty, sc);
                newton_loop(cur);
            }
            // the previous iteration's count is final here (ordered by this barrier)
            newton_clamped = max(newton_clamped, ndeg_sh[cur]);
            const bool any_moved = moved_sh[cur] != 0;
            if (tid == 0) { ndeg_sh[cur ^ 1] = 0; moved_sh[cur ^ 1] = 0; }
            iters = k;
            if (!any_moved && k >= 2 && b.skip_stagnant) {
                // beta reproduced itself bitwise: iteration k+1 recomputes the same L
                // and tests it against the new alpha_k (the post-loop gap below); if
                // that fails, every later iteration repeats exactly the same state and
                // test, so the reference loop ends at the cap (cells.py:320-348)
                stag_k = k;
                iters = b.max_iters;
                break;
            }
        }
        __syncthreads();
        if (!converged) {
            // cap reached: final X sweep and gap for the last (post-Y-step) pair
            // (cells.py:341-348)
            sweep_x<kF32>(w, cw, nw0, nw1, eps, ratio, w.L, sc);
            double part = 0.0;
            for (int x = tid; x < nx; x += DD_NT) {
                const double mu = w.mu[x];
                if (mu > 0) {
                    const double a = w.alpha[x];
                    const double lr = a / eps + w.L[x];
                    const double px = mu * exp(lr);
                    const double ref = mu * exp(-a / lam);
                    part += px * (lr + a / lam) - px + ref;
                }
            }
            gap = lam * block_sum(part, red);
            if (!have_first) { first_gap = gap; have_first = true; }
            converged = gap / lam <= thr;
            // stagnant loop: the reference freezes the cell at iteration stag_k + 1
            if (converged && stag_k) iters = stag_k;
        }
        exec_iters = stag_k ? stag_k : iters;

        t_loop_d = (double)(clock64() - t_loop0);
        nsteps = block_sum((double)newton_steps, red);
    }
    if constexpr (kLoop) {
        for (int x = tid; x < nx; x += DD_NT) {
            b.alpha[(int64_t)c * nx + x] = w.alpha[x];
            b.lout[(int64_t)c * nx + x] = w.L[x];
        }
        for (int y = tid; y < ny; y += DD_NT) b.beta[yoff + y] = w.beta[y];
        if (tid == 0) {
            double* cs = b.cstat + (int64_t)c * 8;
            cs[0] = gap;
            cs[1] = first_gap;
            cs[2] = (double)iters;
            cs[3] = converged ? 1.0 : 0.0;
            cs[4] = (double)n_clamped;
            cs[5] = (double)newton_clamped;
            double* c2 = b.cstat2 + (int64_t)c * 8;
            c2[2] = t_loop_d;
            c2[3] = nsteps;
            c2[4] = (double)exec_iters;
        }
        return;
    }

    // outputs: duals
    for (int x = tid; x < nx; x += DD_NT) b.alpha[(int64_t)c * nx + x] = w.alpha[x];
    for (int y = tid; y < ny; y += DD_NT) b.beta[yoff + y] = w.beta[y];

    // balancing reference mu_bar = exp(-alpha_extra/lam) mu, alpha_extra = -ratio L
    for (int x = tid; x < nx; x += DD_NT) {
        const double ae = -ratio * w.L[x];
        w.L[x] = exp(-ae / lam) * w.mu[x];
        w.u[x] = w.alpha[x] / eps + w.lmu[x];
    }
    // v[y] = beta/eps + lnu (kept in ty for the epilogue)
    for (int y = tid; y < ny; y += DD_NT) w.ty[y] = w.beta[y] / eps + w.lnu[y];
    __syncthreads();

    // ---- per-member split of the plan's Y-marginal + fragment columns ----
    double* RAW = marena;
    double* TC = marena + (int64_t)nmem * ny;
    double* TL = marena + (int64_t)2 * nmem * ny;
    double* MC = marena + (int64_t)3 * nmem * ny;
    double* VALS = marena + (int64_t)4 * nmem * ny;
    double* NEWV = marena + (int64_t)5 * nmem * ny;
    double* M1 = w.mid;
    double* M2 = w.mid + w.ms;
    double* M3 = w.mid + 2 * w.ms;
    double* M4 = w.mid + 3 * w.ms;
    double* M5 = w.mid + 4 * w.ms;
    __shared__ double mbar[64], Ak[64], masses[64], targets[64], surplus[64], tol[64];
    for (int k = 0; k < nmem; ++k) {
        const int i = mem[k];
        const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
        const int r0 = bx[0] - cw.xo0, e0 = bx[1], c0 = bx[2] - cw.xo1, e1 = bx[3];
        double am = kNegInf, mb = 0.0;
        for (int t = tid; t < e0 * e1; t += DD_NT) {
            const int a0 = t / e1, a1 = t - a0 * e1;
            const int x = (r0 + a0) * nw1 + (c0 + a1);
            am = fmax(am, w.u[x]);
            mb += w.L[x];
        }
        const double A = block_max(am, red);
        const double mbk = block_sum(mb, red);
        if (tid == 0) { mbar[k] = mbk; Ak[k] = A; }
        double* raw = RAW + (int64_t)k * ny;
        double* tc = TC + (int64_t)k * ny;
        double* tl = TL + (int64_t)k * ny;
        double* mc = MC + (int64_t)k * ny;
        for (int t = tid; t < e0 * e1; t += DD_NT) {
            const int a0 = t / e1, a1 = t - a0 * e1;
            const int x = (r0 + a0) * nw1 + (c0 + a1);
            w.tx[x] = exp(w.u[x] - A);
        }
        __syncthreads();
        for (int o = tid; o < e0 * ny1; o += DD_NT) {
            const int a0 = o / ny1, y1 = o - a0 * ny1;
            const int x0 = r0 + a0;
            const double yc = w.yc1[y1];
            double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
            for (int a1 = 0; a1 < e1; ++a1) {
                const int x1 = c0 + a1;
                const int x = x0 * nw1 + x1;
                const double dd = w.xc1[x1] - yc;
                const double D1 = dd * dd;
                const double wk = w.tx[x] * w.K1[(int64_t)x1 * ny1 + y1];
                s1 += wk;
                s2 += wk * D1;
                s3 += wk * w.alpha[x];
                s4 += w.mu[x] * D1;
            }
            M1[o] = s1; M2[o] = s2; M3[o] = s3; M4[o] = s4;
        }
        for (int a0 = tid; a0 < e0; a0 += DD_NT) {
            double ssum = 0.0;
            for (int a1 = 0; a1 < e1; ++a1) ssum += w.mu[(r0 + a0) * nw1 + c0 + a1];
            M5[a0] = ssum;
        }
        __syncthreads();
        for (int y = tid; y < ny; y += DD_NT) {
            const int y0 = y / ny1, y1 = y - y0 * ny1;
            const double yc = w.yc0[y0];
            double P = 0.0, C = 0.0, Q = 0.0, MCv = 0.0;
            for (int a0 = 0; a0 < e0; ++a0) {
                const int x0 = r0 + a0;
                const double dd = w.xc0[x0] - yc;
                const double D0 = dd * dd;
                const double k0 = w.K0[(int64_t)x0 * ny0 + y0];
                const int64_t o = (int64_t)a0 * ny1 + y1;
                P += k0 * M1[o];
                C += k0 * (D0 * M1[o] + M2[o]);
                Q += k0 * M3[o];
                MCv += D0 * M5[a0] + M4[o];
            }
            // raw = e^{A + v} P in log form (no overflow of the scale alone);
            // tc, tl as raw times the plan-weighted means of c and sc
            if (P >= kTiny) {
                const double bv = w.beta[y] / eps;
                const double rv = exp(A + w.ty[y] + log(P));
                raw[y] = rv;
                tc[y] = rv * (C / P);
                tl[y] = rv * ((Q / P) / eps + bv - (C / P) / eps);
                mc[y] = MCv;
            } else {
                // exact per-entry evaluation (cells.py:357-374) where the
                // factorised sum may have lost terms to underflow
                double Pe = 0.0, Ce = 0.0, Te = 0.0, Me = 0.0;
                for (int a0 = 0; a0 < e0; ++a0) {
                    const int x0 = r0 + a0;
                    const double dd0 = w.xc0[x0] - w.yc0[y0];
                    for (int a1 = 0; a1 < e1; ++a1) {
                        const int x1 = c0 + a1;
                        const int x = x0 * nw1 + x1;
                        const double dd1 = w.xc1[x1] - w.yc1[y1];
                        const double cost = dd0 * dd0 + dd1 * dd1;
                        const double scv = w.alpha[x] / eps + w.beta[y] / eps + (-cost / eps);
                        const double pl = exp(scv + w.lmu[x] + w.lnu[y]);
                        Pe += pl;
                        Ce += pl * cost;
                        Te += pl * scv;
                        Me += cost * w.mu[x];
                    }
                }
                raw[y] = Pe;
                tc[y] = Ce;
                tl[y] = Te;
                mc[y] = Me;
            }
        }
        __syncthreads();
        for (int y = tid; y < ny; y += DD_NT) VALS[(int64_t)k * ny + y] = raw[y];
        __syncthreads();
    }

    // ---- balancing (cells.py:446-485) ----
    int fallbacks = 0, drift = 0;
    double target_miss = 0.0;
    {
        for (int k = 0; k < nmem; ++k) {
            double p = 0.0;
            for (int y = tid; y < ny; y += DD_NT) p += VALS[(int64_t)k * ny + y];
            const double mk = block_sum(p, red);
            if (tid == 0) masses[k] = mk;
        }
        __syncthreads();
        double total = 0.0, nu_j = 0.0;
        for (int k = 0; k < nmem; ++k) { total += mbar[k]; nu_j += masses[k]; }
        __syncthreads();
        if (tid == 0) {
            for (int k = 0; k < nmem; ++k) {
                targets[k] = mbar[k] * (nu_j / total);
                surplus[k] = masses[k] - targets[k];
                tol[k] = 1e-13 * fmax(targets[k], 1e-300);
            }
        }
        __syncthreads();
        int nd = 0, nr = 0;
        int donors[64], recips[64];
        for (int k = 0; k < nmem; ++k) {
            if (surplus[k] > tol[k]) donors[nd++] = k;
            if (surplus[k] < -tol[k]) recips[nr++] = k;
        }
        if (nd > 0 && nr > 0) {
            // column sums before (member order), kept in ty
            for (int y = tid; y < ny; y += DD_NT) {
                double cs = 0.0;
                for (int k = 0; k < nmem; ++k) cs += VALS[(int64_t)k * ny + y];
                w.ty[y] = cs;
            }
            __syncthreads();
            {
                // every thread follows the same control flow from the shared surplus
                // table; each _move_mass (cells.py:488-507) runs across the block
                __shared__ double stage_sh[256], pub_sh[4];
                int di = 0, ri = 0;
                while (di < nd && ri < nr) {
                    const int dk = donors[di], rk = recips[ri];
                    const double amount = fmin(surplus[dk], -surplus[rk]);
                    if (amount > 0)
                        fallbacks += move_mass_block<DD_NT, 256>(VALS + (int64_t)dk * ny,
                                                                 VALS + (int64_t)rk * ny, ny, amount,
                                                                 stage_sh, pub_sh);
                    const double sd = surplus[dk] - amount, sr = surplus[rk] + amount;
                    __syncthreads();
                    if (tid == 0) { surplus[dk] = sd; surplus[rk] = sr; }
                    __syncthreads();
                    if (sd <= tol[dk]) ++di;
                    if (sr >= -tol[rk]) ++ri;
                }
            }
            for (int k = 0; k < nmem; ++k)
                for (int y = tid; y < ny; y += DD_NT) {
                    double v = VALS[(int64_t)k * ny + y];
                    if (v < 0.0) VALS[(int64_t)k * ny + y] = 0.0;
                }
            __syncthreads();
            // restore column sums bitwise (cells.py:510-563)
            int bad = 0;
            for (int y = tid; y < ny; y += DD_NT) {
                const double target = w.ty[y];
                double cs = 0.0;
                for (int k = 0; k < nmem; ++k) cs += VALS[(int64_t)k * ny + y];
                if (cs == target) continue;
                // order by value descending
                int order[64];
                for (int k = 0; k < nmem; ++k) order[k] = k;
                for (int a = 1; a < nmem; ++a) {
                    int t = order[a];
                    int q = a - 1;
                    while (q >= 0 && VALS[(int64_t)order[q] * ny + y] < VALS[(int64_t)t * ny + y]) {
                        order[q + 1] = order[q];
                        --q;
                    }
                    order[q + 1] = t;
                }
                bool ok = false;
                for (int oi = 0; oi < nmem && !ok; ++oi) {
                    const int t = order[oi];
                    double* e = VALS + (int64_t)t * ny + y;
                    const double x0 = *e;
                    double x = x0;
                    for (int it = 0; it < 256; ++it) {
                        double sm = 0.0;
                        for (int k = 0; k < nmem; ++k) sm += VALS[(int64_t)k * ny + y];
                        if (sm == target) { ok = true; break; }
                        x = nextafter(x, sm < target ? __builtin_huge_val() : -__builtin_huge_val());
                        if (x < 0) break;
                        *e = x;
                    }
                    if (!ok) {
                        double sm = 0.0;
                        *e = x0;
                        for (int k = 0; k < nmem; ++k) sm += VALS[(int64_t)k * ny + y];
                        ok = sm == target;
                    }
                }
                if (!ok) ++bad;
            }
            drift = (int)block_sum((double)bad, red);
        }
        double miss = 0.0;
        for (int k = 0; k < nmem; ++k) {
            double p = 0.0;
            for (int y = tid; y < ny; y += DD_NT) p += VALS[(int64_t)k * ny + y];
            const double mk = block_sum(p, red);
            miss = fmax(miss, fabs(mk - targets[k]) / fmax(targets[k], 1e-300));
        }
        target_miss = miss;
    }

    // ---- truncation, fragments, x-marginals (cells.py:396-443) ----
    double trunc_total = 0.0;
    const int bs = s.block0 * s.block1;
    for (int k = 0; k < nmem; ++k) {
        const int i = mem[k];
        const double* vals = VALS + (int64_t)k * ny;
        const double* raw = RAW + (int64_t)k * ny;
        // bounding box of kept entries, removed mass
        int rmin = 0x7fffffff, rmax = -1, cmin = 0x7fffffff, cmax = -1;
        double rem = 0.0;
        for (int y = tid; y < ny; y += DD_NT) {
            const double v = vals[y];
            if (v >= b.trunc) {
                const int y0 = y / ny1, y1 = y - y0 * ny1;
                rmin = min(rmin, y0); rmax = max(rmax, y0);
                cmin = min(cmin, y1); cmax = max(cmax, y1);
            } else {
                rem += v;
            }
        }
        rmin = block_min_i(rmin, redi);
        rmax = block_max_i(rmax, redi);
        cmin = block_min_i(cmin, redi);
        cmax = block_max_i(cmax, redi);
        const double removed = block_sum(rem, red);
        trunc_total += removed;
        const int mslot = d[10] + k;
        int nb0 = 0, ne0 = 0, nb1 = 0, ne1 = 0;
        if (rmax >= 0) {
            nb0 = cw.yo0 + rmin; ne0 = rmax - rmin + 1;
            nb1 = cw.yo1 + cmin; ne1 = cmax - cmin + 1;
        }
        if (tid == 0) {
            b.mbox[(int64_t)mslot * 4 + 0] = nb0;
            b.mbox[(int64_t)mslot * 4 + 1] = ne0;
            b.mbox[(int64_t)mslot * 4 + 2] = nb1;
            b.mbox[(int64_t)mslot * 4 + 3] = ne1;
        }
        double* nv = NEWV + (int64_t)k * ny;
        for (int t = tid; t < ne0 * ne1; t += DD_NT) {
            const int a0 = t / ne1, a1 = t - a0 * ne1;
            const double v = vals[(int64_t)(rmin + a0) * ny1 + (cmin + a1)];
            nv[t] = v >= b.trunc ? v : 0.0;
        }
        const double mass = s.basic_mass[i];
        double S1 = 0, S2 = 0, S3 = 0, S4 = 0, S5 = 0, S6 = 0, SX = 0;
        const double* tc = TC + (int64_t)k * ny;
        const double* tl = TL + (int64_t)k * ny;
        const double* mc = MC + (int64_t)k * ny;
        for (int y = tid; y < ny; y += DD_NT) {
            const double v = vals[y];
            const double fin = v >= b.trunc ? v : 0.0;
            const double r = raw[y];
            const double fr = r > 0 ? fin / r : 0.0;
            const bool pos = r > 0 && isfinite(fr);
            const double f = pos ? fr : 0.0;
            const double extra = pos ? 0.0 : fin;
            S1 += f * tc[y];
            S2 += extra * mc[y];
            S3 += f * tl[y];
            S4 += xlogy(pos ? fin : 0.0, f);
            {
                const int y0 = y / ny1, y1 = y - y0 * ny1;
                const double nu = s.nu[(int64_t)(cw.yo0 + y0) * g.ny1 + (cw.yo1 + y1)];
                S5 += xlogy(extra, extra / (mass * nu));
            }
            S6 += fin;
            SX += extra;
            // stash f in the TL column (no longer needed after S3): use ty instead
        }
        S1 = block_sum(S1, red);
        S2 = block_sum(S2, red);
        S3 = block_sum(S3, red);
        S4 = block_sum(S4, red);
        S5 = block_sum(S5, red);
        S6 = block_sum(S6, red);
        SX = block_sum(SX, red);
        const double transport = S1 + S2 / mass;
        const double klv = S3 + S4 + S5 - S6 + mass * g.nu_total;
        if (tid == 0) {
            b.mstat[(int64_t)mslot * 4 + 0] = transport;
            b.mstat[(int64_t)mslot * 4 + 1] = klv;
            b.mstat[(int64_t)mslot * 4 + 2] = removed;
            b.mstat[(int64_t)mslot * 4 + 3] = SX;
        }
        // x-marginal: xm[x] = sum_y plan[x,y] f[y] (+ mu[x] SX/mass)
        const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
        const int r0 = bx[0] - cw.xo0, e0 = bx[1], c0 = bx[2] - cw.xo1, e1 = bx[3];
        double* xout = b.xarena + off[3] + (int64_t)k * bs;
        __syncthreads();
        const double A = Ak[k];
        // f into ty (ty currently holds v = beta/eps + lnu; rebuild after)
        __syncthreads();
        // gy[y] = exp(A + v[y] + log f[y] - G), G = max over y of the exponent
        double gmax = kNegInf;
        for (int y = tid; y < ny; y += DD_NT) {
            const double v = vals[y];
            const double fin = v >= b.trunc ? v : 0.0;
            const double r = raw[y];
            const double fr = r > 0 ? fin / r : 0.0;
            const double f = (r > 0 && isfinite(fr)) ? fr : 0.0;
            const double e = f > 0 ? A + w.beta[y] / eps + w.lnu[y] + log(f) : kNegInf;
            w.wy[y] = e;
            gmax = fmax(gmax, e);
        }
        const double G = block_max(gmax, red);
        for (int y = tid; y < ny; y += DD_NT) w.wy[y] = isfinite(G) ? exp(w.wy[y] - G) : 0.0;
        __syncthreads();
        for (int o = tid; o < ny0 * e1; o += DD_NT) {
            const int y0 = o / e1, a1 = o - y0 * e1;
            const int x1 = c0 + a1;
            double sacc = 0.0;
            for (int y1 = 0; y1 < ny1; ++y1)
                sacc = fma(w.wy[(int64_t)y0 * ny1 + y1], w.K1[(int64_t)x1 * ny1 + y1], sacc);
            M1[o] = sacc;
        }
        __syncthreads();
        for (int t = tid; t < e0 * e1; t += DD_NT) {
            const int a0 = t / e1, a1 = t - a0 * e1;
            const int x0 = r0 + a0;
            const int x = x0 * nw1 + (c0 + a1);
            double sacc = 0.0;
            for (int y0 = 0; y0 < ny0; ++y0)
                sacc = fma(w.K0[(int64_t)x0 * ny0 + y0], M1[(int64_t)y0 * e1 + a1], sacc);
            double xm = 0.0;
            if (w.mu[x] > 0) {
                if (sacc >= kTiny) {
                    xm = exp(w.u[x] - A + G + log(sacc));
                } else {
                    // exact: sum_y exp(sc + lmu + lnu) f[y]  (cells.py:436)
                    for (int y = 0; y < ny; ++y) {
                        const double v = vals[y];
                        const double fin = v >= b.trunc ? v : 0.0;
                        const double r = raw[y];
                        const double fr = r > 0 ? fin / r : 0.0;
                        const double f = (r > 0 && isfinite(fr)) ? fr : 0.0;
                        if (f == 0.0) continue;
                        const int y0 = y / ny1, y1 = y - y0 * ny1;
                        const double dd0 = w.xc0[x0] - w.yc0[y0];
                        const double dd1 = w.xc1[c0 + a1] - w.yc1[y1];
                        const double cost = dd0 * dd0 + dd1 * dd1;
                        const double scv = w.alpha[x] / eps + w.beta[y] / eps + (-cost / eps);
                        xm += exp(scv + w.lmu[x] + w.lnu[y]) * f;
                    }
                }
            }
            if (SX != 0.0) xm = xm + w.mu[x] * (SX / mass);
            xout[t] = w.mu[x] > 0 ? xm : 0.0;
        }
        __syncthreads();
    }

    if (tid == 0) {
        double* cs = b.cstat + (int64_t)c * 8;
        cs[0] = gap;
        cs[1] = first_gap;
        cs[2] = (double)iters;
        cs[3] = converged ? 1.0 : 0.0;
        cs[4] = (double)n_clamped;
        cs[5] = (double)newton_clamped;
        cs[6] = (double)fallbacks;
        cs[7] = target_miss;
        double* c2 = b.cstat2 + (int64_t)c * 8;
        c2[0] = (double)drift;    // (phase-timing builds keep the sweep-fallback stats here)
        c2[1] = trunc_total;
        c2[2] = t_loop_d;         // SM cycles spent in the Sinkhorn loop
        c2[3] = nsteps;           // Newton evaluations over all nodes and iterations
        if (!epi) c2[4] = (double)exec_iters;   // Sinkhorn iterations actually executed
    }
}

// ---- blend scoring -----------------------------------------------------------

// Old (current plan) and new (solution) window sums of one cell, and deltas.
__global__ void __launch_bounds__(DD_NT) cell_delta_kernel(dd_geom g, dd_state s, dd_batch b,
                                                           double* dy, double* cd) {
    __shared__ double red[DD_NW + 1];
    const int c = blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t* off = b.offs + (int64_t)c * 4;
    const CellWin cw = load_win(d, b.nxw0, b.nxw1);
    const int nmem = d[9];
    const int32_t* mem = b.members + d[10];
    const int ny = cw.ny, ny1 = cw.ye1;
    const int64_t yoff = off[0];
    if (d[11] & 2) {   // cell held by another rank (slab mode): no update from here
        for (int y = threadIdx.x; y < ny; y += DD_NT) dy[yoff + y] = 0.0;
        if (threadIdx.x < 4) cd[(int64_t)c * 4 + threadIdx.x] = 0.0;
        return;
    }
    const double* NEWV = b.marena + off[1] + (int64_t)5 * nmem * ny;
    for (int y = threadIdx.x; y < ny; y += DD_NT) {
        const int y0 = y / ny1, y1 = y - y0 * ny1;
        const int r = cw.yo0 + y0, q = cw.yo1 + y1;
        double yo = 0.0, yn = 0.0;
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            yo += boxed_at(s.ybox + (int64_t)i * 4, s.yval + (int64_t)i * s.cap, r, q);
            yn += boxed_at(b.mbox + (int64_t)(d[10] + k) * 4, NEWV + (int64_t)k * ny, r, q);
        }
        dy[yoff + y] = yn - yo;
    }
    // t_delta, k_delta, d1_old
    const int bs = s.block0 * s.block1;
    double d1o = 0.0;
    for (int k = 0; k < nmem; ++k) {
        const int i = mem[k];
        const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
        double p = 0.0;
        for (int t = threadIdx.x; t < bs; t += DD_NT) {
            const int a0 = t / bx[3], a1 = t - a0 * bx[3];
            const double mu = s.mu[(int64_t)(bx[0] + a0) * g.nx1 + (bx[2] + a1)];
            if (mu > 0) p += kl_term(s.x_marg[(int64_t)i * bs + t], mu);
        }
        d1o += block_sum(p, red);
    }
    if (threadIdx.x == 0) {
        double tn = 0.0, to = 0.0, kn = 0.0, ko = 0.0;
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            tn += b.mstat[(int64_t)(d[10] + k) * 4 + 0];
            kn += b.mstat[(int64_t)(d[10] + k) * 4 + 1];
            to += s.transport[i];
            ko += s.kl[i];
        }
        cd[(int64_t)c * 4 + 0] = tn - to;
        cd[(int64_t)c * 4 + 1] = kn - ko;
        cd[(int64_t)c * 4 + 2] = g.lam * d1o;
        cd[(int64_t)c * 4 + 3] = 0.0;
    }
}

// per-cell blend pieces: out[c*4] = theta*t_delta, theta*k_delta, d1_blend - d1_old
__global__ void __launch_bounds__(DD_NT) blend_cell_kernel(dd_geom g, dd_state s, dd_batch b,
                                                           const double* cd, const double* theta,
                                                           double* pc) {
    __shared__ double red[DD_NW + 1];
    const int c = blockIdx.x;
    const double th = theta[c];
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t* off = b.offs + (int64_t)c * 4;
    const int nmem = d[9];
    const int32_t* mem = b.members + d[10];
    const int bs = s.block0 * s.block1;
    double d1b = 0.0;
    if (th != 0.0) {
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
            const double* xn = b.xarena + off[3] + (int64_t)k * bs;
            double p = 0.0;
            for (int t = threadIdx.x; t < bs; t += DD_NT) {
                const int a0 = t / bx[3], a1 = t - a0 * bx[3];
                const double mu = s.mu[(int64_t)(bx[0] + a0) * g.nx1 + (bx[2] + a1)];
                if (mu > 0) {
                    const double xo = s.x_marg[(int64_t)i * bs + t];
                    p += kl_term((1.0 - th) * xo + th * xn[t], mu);
                }
            }
            d1b += block_sum(p, red);
        }
    }
    if (threadIdx.x == 0) {
        pc[(int64_t)c * 4 + 0] = th != 0.0 ? th * cd[(int64_t)c * 4 + 0] : 0.0;
        pc[(int64_t)c * 4 + 1] = th != 0.0 ? th * cd[(int64_t)c * 4 + 1] : 0.0;
        pc[(int64_t)c * 4 + 2] = th != 0.0 ? g.lam * d1b - cd[(int64_t)c * 4 + 2] : 0.0;
        pc[(int64_t)c * 4 + 3] = 0.0;
    }
}

// ---- commit ---------------------------------------------------------------------

__global__ void __launch_bounds__(DD_NT) cell_commit_kernel(dd_geom g, dd_state s, dd_batch b,
                                                            const double* theta,
                                                            double* alpha_grid, double* yrun,
                                                            double* errs) {
    __shared__ double red[DD_NW + 1];
    __shared__ int redi[DD_NW + 1];
    const int c = blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t* off = b.offs + (int64_t)c * 4;
    const int nw0 = b.nxw0, nw1 = b.nxw1;
    const CellWin cw = load_win(d, nw0, nw1);
    const int j = d[0];
    const int nmem = d[9];
    const int32_t* mem = b.members + d[10];
    const int ny = cw.ny, ny1 = cw.ye1, nx = cw.nx;
    const int64_t yoff = off[0];
    double* marena = b.marena + off[1];
    double* OLDW = marena;                        // raw region reused: old windows
    double* BW = marena + (int64_t)4 * nmem * ny;   // vals region reused: blended windows
    const double* NEWV = marena + (int64_t)5 * nmem * ny;
    const double th = theta[c];
    const int bs = s.block0 * s.block1;
    const int tid = threadIdx.x;
    if (d[11] & 2) {   // cell held by another rank (slab mode): its owner commits it
        if (tid < 4) errs[(int64_t)c * 4 + tid] = 0.0;
        return;
    }

    // old member windows on the cell's Y box
    for (int k = 0; k < nmem; ++k) {
        const int i = mem[k];
        for (int y = tid; y < ny; y += DD_NT) {
            const int y0 = y / ny1, y1 = y - y0 * ny1;
            OLDW[(int64_t)k * ny + y] =
                boxed_at(s.ybox + (int64_t)i * 4, s.yval + (int64_t)i * s.cap, cw.yo0 + y0, cw.yo1 + y1);
        }
    }
    __syncthreads();
    double added = 0.0;
    if (th >= 1.0) {
        added = b.cstat2[(int64_t)c * 8 + 1];
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            const int mslot = d[10] + k;
            const int32_t* nb = b.mbox + (int64_t)mslot * 4;
            const int n = (nb[1] > 0 && nb[3] > 0) ? nb[1] * nb[3] : 0;
            for (int t = tid; t < n; t += DD_NT) s.yval[(int64_t)i * s.cap + t] = NEWV[(int64_t)k * ny + t];
            if (tid < 4) s.ybox[(int64_t)i * 4 + tid] = n ? nb[tid] : 0;
            const double* xn = b.xarena + off[3] + (int64_t)k * bs;
            for (int t = tid; t < bs; t += DD_NT) s.x_marg[(int64_t)i * bs + t] = xn[t];
            if (tid == 0) {
                s.transport[i] = b.mstat[(int64_t)mslot * 4 + 0];
                s.kl[i] = b.mstat[(int64_t)mslot * 4 + 1];
            }
        }
    } else if (th > 0.0) {
        double removed_all = 0.0;
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            const int mslot = d[10] + k;
            const int32_t* nb = b.mbox + (int64_t)mslot * 4;
            double* bw = BW + (int64_t)k * ny;
            for (int y = tid; y < ny; y += DD_NT) {
                const int y0 = y / ny1, y1 = y - y0 * ny1;
                const double nv = boxed_at(nb, NEWV + (int64_t)k * ny, cw.yo0 + y0, cw.yo1 + y1);
                bw[y] = (1.0 - th) * OLDW[(int64_t)k * ny + y] + th * nv;
            }
            __syncthreads();
            int rmin = 0x7fffffff, rmax = -1, cmin = 0x7fffffff, cmax = -1;
            double rem = 0.0;
            for (int y = tid; y < ny; y += DD_NT) {
                const double v = bw[y];
                if (v >= b.trunc) {
                    const int y0 = y / ny1, y1 = y - y0 * ny1;
                    rmin = min(rmin, y0); rmax = max(rmax, y0);
                    cmin = min(cmin, y1); cmax = max(cmax, y1);
                } else {
                    rem += v;
                }
            }
            rmin = block_min_i(rmin, redi);
            rmax = block_max_i(rmax, redi);
            cmin = block_min_i(cmin, redi);
            cmax = block_max_i(cmax, redi);
            removed_all += block_sum(rem, red);
            int ne0 = 0, ne1 = 0;
            if (rmax >= 0) { ne0 = rmax - rmin + 1; ne1 = cmax - cmin + 1; }
            for (int t = tid; t < ne0 * ne1; t += DD_NT) {
                const int a0 = t / ne1, a1 = t - a0 * ne1;
                const double v = bw[(int64_t)(rmin + a0) * ny1 + (cmin + a1)];
                s.yval[(int64_t)i * s.cap + t] = v >= b.trunc ? v : 0.0;
            }
            if (tid == 0) {
                int* ob = s.ybox + (int64_t)i * 4;
                if (rmax >= 0) {
                    ob[0] = cw.yo0 + rmin; ob[1] = ne0; ob[2] = cw.yo1 + cmin; ob[3] = ne1;
                } else {
                    ob[0] = 0; ob[1] = 0; ob[2] = 0; ob[3] = 0;
                }
                s.transport[i] = (1.0 - th) * s.transport[i] + th * b.mstat[(int64_t)mslot * 4 + 0];
                s.kl[i] = (1.0 - th) * s.kl[i] + th * b.mstat[(int64_t)mslot * 4 + 1];
            }
            const double* xn = b.xarena + off[3] + (int64_t)k * bs;
            for (int t = tid; t < bs; t += DD_NT)
                s.x_marg[(int64_t)i * bs + t] = (1.0 - th) * s.x_marg[(int64_t)i * bs + t] + th * xn[t];
            __syncthreads();
        }
        added = th * b.cstat2[(int64_t)c * 8 + 1] + removed_all;
    }
    __syncthreads();
    // dual store
    double* da = s.d_alpha + (int64_t)j * nx;
    const double* al = b.alpha + (int64_t)c * nx;
    for (int x = tid; x < nx; x += DD_NT) da[x] = al[x];
    for (int y = tid; y < ny; y += DD_NT) s.d_beta[(int64_t)j * s.d_cap + y] = b.beta[yoff + y];
    if (tid == 0) {
        s.d_has[j] = 1;
        s.d_box[(int64_t)j * 4 + 0] = cw.yo0;
        s.d_box[(int64_t)j * 4 + 1] = cw.ye0;
        s.d_box[(int64_t)j * 4 + 2] = cw.yo1;
        s.d_box[(int64_t)j * 4 + 3] = cw.ye1;
    }
    __syncthreads();
    // residuals of the committed state against the solution duals
    double ye = 0.0;
    for (int y = tid; y < ny; y += DD_NT) {
        const int y0 = y / ny1, y1 = y - y0 * ny1;
        const int r = cw.yo0 + y0, q = cw.yo1 + y1;
        double yn = 0.0, yo = 0.0;
        for (int k = 0; k < nmem; ++k) {
            const int i = mem[k];
            yn += boxed_at(s.ybox + (int64_t)i * 4, s.yval + (int64_t)i * s.cap, r, q);
            yo += OLDW[(int64_t)k * ny + y];
        }
        if (th <= 0.0) yn = yo;
        const double nu = s.nu[(int64_t)r * g.ny1 + q];
        const double num = b.mdens[yoff + y] * nu;
        ye += fabs(yn + num - exp(-b.beta[yoff + y] / g.lam) * nu);
        if (yrun) {
            const int64_t id = (int64_t)r * g.ny1 + q;
            yrun[id] = fmax(yrun[id] + (yn - yo), 0.0);
        }
    }
    ye = block_sum(ye, red);
    double xe = 0.0;
    for (int k = 0; k < nmem; ++k) {
        const int i = mem[k];
        const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
        const int r0 = bx[0] - cw.xo0, c0 = bx[2] - cw.xo1, e1 = bx[3];
        double p = 0.0;
        for (int t = tid; t < bs; t += DD_NT) {
            const int a0 = t / e1, a1 = t - a0 * e1;
            const int gr = bx[0] + a0, gq = bx[2] + a1;
            const double mu = s.mu[(int64_t)gr * g.nx1 + gq];
            const double a = al[(r0 + a0) * nw1 + (c0 + a1)];
            if (alpha_grid) alpha_grid[(int64_t)gr * g.nx1 + gq] = a;
            if (mu > 0) p += fabs(s.x_marg[(int64_t)i * bs + t] - exp(-a / g.lam) * mu);
        }
        xe += block_sum(p, red);
    }
    if (tid == 0) {
        errs[(int64_t)c * 4 + 0] = xe;
        errs[(int64_t)c * 4 + 1] = ye;
        errs[(int64_t)c * 4 + 2] = added;
        errs[(int64_t)c * 4 + 3] = 0.0;
    }
}

// ---- opt strategy: derivative pieces of the 1D blend objective --------------------
// (engine.py:473-503 g_and_h).  out[0] = sum of member terms d*log(x/mn),
// out[1] = sum d^2/x, out[2] = sum dy*log(y/nu), out[3] = sum dy^2/y, all lam-free,
// with x = (1-th) xo + th xn and y = clip(clip(ycur - th_cur dy, 0) + th dy, 0).
__global__ void __launch_bounds__(DD_NT) opt_gh_kernel(dd_geom g, dd_state s, dd_batch b,
                                                       const double* dy, int c, double th,
                                                       double th_cur, const double* ycur,
                                                       double* out) {
    __shared__ double red[DD_NW + 1];
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t* off = b.offs + (int64_t)c * 4;
    const int nmem = d[9];
    const int32_t* mem = b.members + d[10];
    const int bs = s.block0 * s.block1;
    double gx = 0.0, hx = 0.0;
    for (int k = 0; k < nmem; ++k) {
        const int i = mem[k];
        const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
        const double* xn = b.xarena + off[3] + (int64_t)k * bs;
        for (int t = threadIdx.x; t < bs; t += DD_NT) {
            const int a0 = t / bx[3], a1 = t - a0 * bx[3];
            const double mu = s.mu[(int64_t)(bx[0] + a0) * g.nx1 + (bx[2] + a1)];
            if (!(mu > 0)) continue;
            const double xo = s.x_marg[(int64_t)i * bs + t];
            const double dd = xn[t] - xo;
            if (dd == 0.0) continue;
            const double x = (1.0 - th) * xo + th * xn[t];
            gx += dd * log(x / mu);
            hx += dd * dd / x;
        }
    }
    const int ye1 = d[8], ny = d[6] * d[8];
    const int64_t yoff = off[0];
    double gy = 0.0, hy = 0.0;
    for (int y = threadIdx.x; y < ny; y += DD_NT) {
        const double dv = dy[yoff + y];
        if (dv == 0.0) continue;
        const int y0 = y / ye1, y1 = y - y0 * ye1;
        const int64_t id = (int64_t)(d[5] + y0) * g.ny1 + (d[7] + y1);
        const double yb = fmax(ycur[id] - th_cur * dv, 0.0);
        const double yv = fmax(yb + th * dv, 0.0);
        gy += dv * log(yv / s.nu[id]);
        hy += dv * dv / yv;
    }
    gx = block_sum(gx, red);
    hx = block_sum(hx, red);
    gy = block_sum(gy, red);
    hy = block_sum(hy, red);
    if (threadIdx.x == 0) { out[0] = gx; out[1] = hx; out[2] = gy; out[3] = hy; }
}

// ycur[ids of cell c] = clip(ycur + dth * dy, 0)   (BlendScorer.set_theta)
__global__ void __launch_bounds__(DD_NT) opt_set_kernel(dd_batch b, const double* dy, int c,
                                                        double dth, double* ycur, int ny1g) {
    const int32_t* d = b.desc + (int64_t)c * 12;
    const int64_t yoff = b.offs[(int64_t)c * 4];
    const int ye1 = d[8], ny = d[6] * d[8];
    for (int y = threadIdx.x; y < ny; y += DD_NT) {
        const int y0 = y / ye1, y1 = y - y0 * ye1;
        const int64_t id = (int64_t)(d[5] + y0) * ny1g + (d[7] + y1);
        ycur[id] = fmax(ycur[id] + dth * dy[yoff + y], 0.0);
    }
}

}  // namespace dd

// ---- host wrappers ---------------------------------------------------------------

extern "C" int dd_set_error(cudaError_t e);

extern "C" int64_t dd_cell_ws_size(int nw0, int nw1, int ny0, int ny1) {
    return dd::ws_layout(nw0, nw1, ny0, ny1).total;
}

static int cluster_configure(int clu_smem) {
    static thread_local int clu_configured = -1;
    if (clu_smem <= clu_configured) return 0;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, dd::cell_loop_cluster_kernel);
    if (e != cudaSuccess) return dd_set_error(e);
    const int avail = optin - (int)fa.sharedSizeBytes;
    if (clu_smem > avail) return dd_set_error(cudaErrorInvalidValue);
    e = cudaFuncSetAttribute(dd::cell_loop_cluster_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, avail);
    if (e != cudaSuccess) return dd_set_error(e);
    e = cudaFuncSetAttribute(dd::cell_loop_cluster_kernel,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return dd_set_error(e);
    clu_configured = avail;
    return 0;
}

// groups: n_groups cluster launches; group k covers clu_ids[goff[k] .. goff[k+1])
// with cluster size gsize[k] and gsmem[k] bytes of shared memory per CTA.
static int cell_solve_launch(const dd_geom* g, const dd_state* s, const dd_batch* b,
                             cudaStream_t st, cudaStream_t st_big, int n_big,
                             const int32_t* clu_ids, int n_groups, const int32_t* goff,
                             const int32_t* gsize, const int32_t* gsmem) {
    const int smem = b->smem_mode ? b->smem_bytes : 0;
    static thread_local int configured = -1;
    static thread_local bool big_configured = false;
    if (smem > configured) {
        // opt in to the full per-block budget minus the kernel's static shared memory
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        // (each instantiation has its own static shared memory)
        cudaFuncAttributes fa, fb;
        cudaError_t e = cudaFuncGetAttributes(&fa, dd::cell_solve_kernel<0, false, false>);
        if (e != cudaSuccess) return dd_set_error(e);
        e = cudaFuncGetAttributes(&fb, dd::cell_solve_kernel<0, true, false>);
        if (e != cudaSuccess) return dd_set_error(e);
        const int avail_a = optin - (int)fa.sharedSizeBytes;
        const int avail_b = optin - (int)fb.sharedSizeBytes;
        const int avail = avail_a < avail_b ? avail_a : avail_b;
        if (smem > avail) return dd_set_error(cudaErrorInvalidValue);
        e = cudaFuncSetAttribute(dd::cell_solve_kernel<0, false, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, avail_a);
        if (e != cudaSuccess) return dd_set_error(e);
        e = cudaFuncSetAttribute(dd::cell_solve_kernel<0, true, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, avail_b);
        if (e != cudaSuccess) return dd_set_error(e);
        configured = avail;
    }
    if (!big_configured) {
        cudaError_t e = cudaFuncSetAttribute(dd::cell_solve_kernel<1, false, false>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout,
                                             (int)cudaSharedmemCarveoutMaxL1);
        if (e != cudaSuccess) return dd_set_error(e);
        e = cudaFuncSetAttribute(dd::cell_solve_kernel<1, true, false>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxL1);
        if (e != cudaSuccess) return dd_set_error(e);
        big_configured = true;
    }
    for (int k = 0; k < n_groups; ++k) {
        const int rc = cluster_configure(gsmem[k]);
        if (rc) return rc;
    }
    const bool f32 = b->precision == 1;
    auto launch_small = [&]() {
        if (b->split_smem_bytes > 0) {
            // split cells (flag 4): the Sinkhorn loop at two CTAs per SM first, then
            // their epilogue (with every other shared-memory cell) below
            static thread_local int split_configured = -1;
            if (b->split_smem_bytes > split_configured) {
                cudaFuncSetAttribute(dd::cell_solve_kernel<0, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     b->split_smem_bytes);
                cudaFuncSetAttribute(dd::cell_solve_kernel<0, true, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     b->split_smem_bytes);
                split_configured = b->split_smem_bytes;
            }
            const size_t ss = (size_t)b->split_smem_bytes;
            if (f32) dd::cell_solve_kernel<0, true, true><<<b->n_cells, DD_NT, ss, st>>>(*g, *s, *b);
            else dd::cell_solve_kernel<0, false, true><<<b->n_cells, DD_NT, ss, st>>>(*g, *s, *b);
        }
        if (f32) dd::cell_solve_kernel<0, true, false><<<b->n_cells, DD_NT, smem, st>>>(*g, *s, *b);
        else dd::cell_solve_kernel<0, false, false><<<b->n_cells, DD_NT, smem, st>>>(*g, *s, *b);
    };
    auto launch_big = [&](cudaStream_t sb) -> cudaError_t {
        for (int k = 0; k < n_groups; ++k) {
            const int ncl = goff[k + 1] - goff[k];
            if (ncl <= 0) continue;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(ncl * gsize[k]), 1, 1);
            cfg.blockDim = dim3(DD_NT, 1, 1);
            cfg.dynamicSmemBytes = (size_t)gsmem[k];
            cfg.stream = sb;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)gsize[k];
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, dd::cell_loop_cluster_kernel, *g, *s, *b,
                                               clu_ids + goff[k]);
            if (e != cudaSuccess) return e;
        }
        if (f32) dd::cell_solve_kernel<1, true, false><<<b->n_cells, DD_NT, 0, sb>>>(*g, *s, *b);
        else dd::cell_solve_kernel<1, false, false><<<b->n_cells, DD_NT, 0, sb>>>(*g, *s, *b);
        return cudaGetLastError();
    };
    if (n_big > 0 && st_big != nullptr && st_big != st) {
        // big cells on the side stream, ordered after everything already on st and
        // joined back before anything enqueued on st afterwards
        static thread_local cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
        if (!ev_fork) {
            cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
        }
        cudaEventRecord(ev_fork, st);
        cudaStreamWaitEvent(st_big, ev_fork, 0);
        cudaError_t e = launch_big(st_big);
        if (e != cudaSuccess) return dd_set_error(e);
        if (b->smem_mode) launch_small();
        e = cudaGetLastError();
        if (e != cudaSuccess) return dd_set_error(e);
        cudaEventRecord(ev_join, st_big);
        cudaStreamWaitEvent(st, ev_join, 0);
        return dd_set_error(cudaGetLastError());
    }
    if (b->smem_mode) launch_small();
    if (n_big > 0) {
        cudaError_t e = launch_big(st);
        if (e != cudaSuccess) return dd_set_error(e);
    }
    return dd_set_error(cudaGetLastError());
}

extern "C" int64_t dd_cell_cluster_ws(int nw0, int nw1, int ny0, int ny1, int clu_size) {
    return dd::clu_layout(nw0, nw1, ny0, ny1, (ny0 + clu_size - 1) / clu_size + 1).total;
}

extern "C" int dd_cell_solve(const dd_geom* g, const dd_state* s, const dd_batch* b, void* stream) {
    if (b->n_cells <= 0) return 0;
    return cell_solve_launch(g, s, b, (cudaStream_t)stream, nullptr, 1, nullptr, 0, nullptr,
                             nullptr, nullptr);
}

extern "C" int dd_cell_solve2(const dd_geom* g, const dd_state* s, const dd_batch* b, void* stream,
                              void* stream_big, int n_big, const int32_t* clu_ids, int n_groups,
                              const int32_t* goff, const int32_t* gsize, const int32_t* gsmem) {
    if (b->n_cells <= 0) return 0;
    return cell_solve_launch(g, s, b, (cudaStream_t)stream, (cudaStream_t)stream_big, n_big,
                             clu_ids, n_groups, goff, gsize, gsmem);
}

extern "C" int dd_cell_delta(const dd_geom* g, const dd_state* s, const dd_batch* b, double* dy,
                             double* cd, void* stream) {
    if (b->n_cells <= 0) return 0;
    dd::cell_delta_kernel<<<b->n_cells, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, dy, cd);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_reduce_rows(int64_t n_rows, int width, const double* in, double* out,
                              void* stream);

extern "C" int dd_grid_kl(int64_t n, const double* y, const double* nu, int clip, double* partial,
                          double* out, void* stream);

extern "C" int dd_blend_energy(const dd_geom* g, const dd_state* s, const dd_batch* b,
                               const double* dy, const double* cd, const double* theta,
                               double* ywork, double* partial, double* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)g->ny0 * g->ny1;
    cudaError_t e;
    // ywork = snapshot + sum_c theta_c dy_c over the cells' Y windows, in cell order
    int rc0 = dd_box_gather(b->n_cells, b->desc + 5, 12, dy, 0, b->offs, 4, theta, g->ny0, g->ny1,
                            b->snapshot, ywork, st);
    if (rc0) return rc0;
    int rc = dd_grid_kl(n, ywork, s->nu, 1, partial, out, stream);
    if (rc) return rc;
    if (b->n_cells > 0) {
        // per-cell pieces into partial + 2048.., then ordered row reduction
        double* pc = partial + 4096;
        dd::blend_cell_kernel<<<b->n_cells, DD_NT, 0, st>>>(*g, *s, *b, cd, theta, pc);
        e = cudaGetLastError();
        if (e != cudaSuccess) return dd_set_error(e);
        rc = dd_reduce_rows(b->n_cells, 4, pc, out + 1, stream);
        if (rc) return rc;
    } else {
        e = cudaMemsetAsync(out + 1, 0, 3 * sizeof(double), st);
        if (e != cudaSuccess) return dd_set_error(e);
    }
    return 0;
}

// Slab mode: the rank-local parts of dd_blend_energy.  dsum = sum_c theta_c dy_c over
// the cells with theta_c != 0 (no snapshot base; the caller masks theta to its own
// cells, sums dsum over the ranks and adds the snapshot), out[1..3] = the summed
// per-cell pieces of those cells, out[0] = 0.
extern "C" int dd_blend_parts(const dd_geom* g, const dd_state* s, const dd_batch* b,
                              const double* dy, const double* cd, const double* theta,
                              double* dsum, double* partial, double* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int rc = dd_box_gather(b->n_cells, b->desc + 5, 12, dy, 0, b->offs, 4, theta, g->ny0, g->ny1,
                           nullptr, dsum, st);
    if (rc) return rc;
    cudaError_t e = cudaMemsetAsync(out, 0, 4 * sizeof(double), st);
    if (e != cudaSuccess) return dd_set_error(e);
    if (b->n_cells > 0) {
        double* pc = partial + 4096;
        dd::blend_cell_kernel<<<b->n_cells, DD_NT, 0, st>>>(*g, *s, *b, cd, theta, pc);
        e = cudaGetLastError();
        if (e != cudaSuccess) return dd_set_error(e);
        rc = dd_reduce_rows(b->n_cells, 4, pc, out + 1, stream);
        if (rc) return rc;
    }
    return 0;
}

extern "C" int dd_cell_commit(const dd_geom* g, const dd_state* s, const dd_batch* b,
                              const double* theta, double* alpha_grid, double* yrun, double* errs,
                              void* stream) {
    if (b->n_cells <= 0) return 0;
    dd::cell_commit_kernel<<<b->n_cells, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, theta,
                                                                          alpha_grid, yrun, errs);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_opt_gh(const dd_geom* g, const dd_state* s, const dd_batch* b, const double* dy,
                         int c, double th, double th_cur, const double* ycur, double* out,
                         void* stream) {
    dd::opt_gh_kernel<<<1, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, dy, c, th, th_cur, ycur,
                                                             out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_opt_set(const dd_geom* g, const dd_batch* b, const double* dy, int c, double dth,
                          double* ycur, void* stream) {
    dd::opt_set_kernel<<<1, DD_NT, 0, (cudaStream_t)stream>>>(*b, dy, c, dth, ycur, g->ny1);
    return dd_set_error(cudaGetLastError());
}


extern "C" int dd_cell_min_blocks(void) { return DD_CELL_MIN_BLOCKS; }

// fp32-mode sweep statistics: out[0..3] = X fallbacks, Y fallbacks, X sweeps, Y sweeps
// since the last call (diagnostic; counters reset)
extern "C" int dd_sweep_fallbacks(unsigned long long* out) {
    cudaError_t e = cudaMemcpyFromSymbol(out, dd::g_sweep_fallbacks, 4 * sizeof(unsigned long long));
    if (e != cudaSuccess) return dd_set_error(e);
    unsigned long long z[4] = {0, 0, 0, 0};
    return dd_set_error(cudaMemcpyToSymbol(dd::g_sweep_fallbacks, z, sizeof(z)));
}
