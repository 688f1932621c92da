// Three-axis domain decomposition: grid LSE, cell solve, blend pieces, commit,
// assembly, starts.
//
// The same algorithm as cell.cu / grid.cu (the reference's cells.py, engine.py,
// sinkhorn.py), laid out for up to three grid axes: a 2D problem runs as
// (1, n0, n1), a 1D one as (1, 1, n), so the whole path can be checked against
// every 1D/2D reference fixture as well as against 3D fixtures.
//
// Cell kernel design (one 256-thread CTA per composite cell): 3D Y windows
// hold thousands to tens of thousands of nodes, so the per-cell workspace
// (potentials, background, log nu, per-axis kernel tables, stage scratch) lives
// in a global-memory arena that the SM's L1 and the 126 MB L2 keep hot.  Each
// Sinkhorn sweep is the factorised kernel K = K0 (x) K1 (x) K2 applied one axis
// at a time with FMA contractions against Y-normalised per-axis tables and one
// global max shift of the input (the reference DenseKernel's "matrix" form,
// sinkhorn.py:91-130); an output whose shifted sum falls below kTiny may have
// lost its dominant terms to underflow, and the whole sweep is then redone by
// the stage-wise log-domain path (each stage an exact two-pass log-sum-exp).

#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "common.cuh"
#include "domdec_b200.h"

extern "C" int dd_set_error(cudaError_t e);

namespace v3 {

constexpr int NT = 256;      // threads per CTA of the grid / blend / commit / start kernels
#ifndef DD3_CELL_NT
#define DD3_CELL_NT 512      // threads per CTA of the cell solve (the whole SM for one cell:
#endif                       // batches end on their longest cells, so latency rules)
constexpr int CELL_NT = DD3_CELL_NT;
constexpr int NW = NT / 32;
constexpr double kTiny = 1e-290;
constexpr double kNegInf = -__builtin_huge_val();
constexpr double kInf = __builtin_huge_val();

struct B3 {
    int o[3], e[3];
};

__device__ __forceinline__ B3 ldbox(const int32_t* p) {
    B3 b;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b.o[a] = p[2 * a];
        b.e[a] = p[2 * a + 1];
    }
    return b;
}
__device__ __forceinline__ bool bempty(const B3& b) {
    return b.e[0] <= 0 || b.e[1] <= 0 || b.e[2] <= 0;
}
__device__ __forceinline__ int64_t bsize(const B3& b) {
    return bempty(b) ? 0 : (int64_t)b.e[0] * b.e[1] * b.e[2];
}
// value of boxed compact row-major values at absolute node (r0, r1, r2); 0 outside
__device__ __forceinline__ double bat(const B3& b, const double* v, int r0, int r1, int r2) {
    const int a0 = r0 - b.o[0], a1 = r1 - b.o[1], a2 = r2 - b.o[2];
    if (a0 < 0 || a0 >= b.e[0] || a1 < 0 || a1 >= b.e[1] || a2 < 0 || a2 >= b.e[2]) return 0.0;
    return v[((int64_t)a0 * b.e[1] + a1) * b.e[2] + a2];
}
// (i0, i1, i2) of a flat row-major index (all window and grid indices are < 2^31)
__device__ __forceinline__ void unflat(int64_t t, int n1, int n2, int& i0, int& i1, int& i2) {
    const unsigned u = (unsigned)t;
    const unsigned q = u / (unsigned)n2;
    i2 = (int)(u - q * (unsigned)n2);
    i0 = (int)(q / (unsigned)n1);
    i1 = (int)(q - (unsigned)i0 * (unsigned)n1);
}

// block reductions for NT threads (all threads call; all receive the result;
// fixed order, so deterministic)
template <int T = NT>
__device__ __forceinline__ double bsum(double v, double* red) {
    v = dd::warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < (T / 32); ++k) t += red[k];
    return t;
}
template <int T = NT>
__device__ __forceinline__ double bmax(double v, double* red) {
    v = dd::warp_max(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = red[0];
#pragma unroll
    for (int k = 1; k < (T / 32); ++k) t = fmax(t, red[k]);
    return t;
}
template <int T = NT>
__device__ __forceinline__ int bmin_i(int v, int* red) {
    v = dd::warp_min_i(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = red[0];
#pragma unroll
    for (int k = 1; k < (T / 32); ++k) t = min(t, red[k]);
    return t;
}
template <int T = NT>
__device__ __forceinline__ int bmax_i(int v, int* red) {
    v = dd::warp_max_i(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = red[0];
#pragma unroll
    for (int k = 1; k < (T / 32); ++k) t = max(t, red[k]);
    return t;
}

// numpy's sum of a short strided double vector (pairwise_sum: sequential below 8
// terms, eight interleaved accumulators up to 128) -- used where the reference
// tests a recomputed sum for bitwise equality (cells.py:510-522).
__device__ double np_sum(const double* a, int64_t stride, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i * stride]);
        return r;
    }
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k * stride];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[(i + k) * stride]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
    return res;
}

// ---- full-grid three-axis LSE ------------------------------------------------------

struct GStage {
    const double* in;
    double* out;
    double* w;       // shifted weights, same shape as in
    double* rmax;    // row maxima [A*B]
    const double* tab;  // exp table [O*K]
    int A, K, B, O;
    double p_org, p_dx, q_org, q_dx, eps;
    const int* stop;    // nullable: device flag of the device-side Sinkhorn loop
};

// tab[k*O + o] = exp(-(d*d)/eps), d = p_o - q_k  (o fastest: coalesced across outputs)
__global__ void g_table_kernel(int O, int K, double po, double pd, double qo, double qd,
                               double eps, double* tab) {
    const int64_t n = (int64_t)O * K;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / O), o = (int)(t - (int64_t)k * O);
        const double d = (po + pd * (double)o) - (qo + qd * (double)k);
        tab[t] = exp(-(d * d) / eps);
    }
}

__global__ void g_rows_kernel(GStage s) {
    if (s.stop && *s.stop) return;
    const int64_t rows = (int64_t)s.A * s.B;
    if (s.B == 1) {
        // contiguous rows: one warp per row (coalesced)
        const int lane = threadIdx.x & 31;
        const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
        const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
        for (int64_t r = w0; r < rows; r += nw) {
            const double* src = s.in + r * s.K;
            double m = kNegInf;
            for (int k = lane; k < s.K; k += 32) m = fmax(m, src[k]);
            m = dd::warp_max_all(m);
            if (!isfinite(m)) m = 0.0;
            if (lane == 0) s.rmax[r] = m;
            double* dst = s.w + r * s.K;
            for (int k = lane; k < s.K; k += 32) dst[k] = exp(src[k] - m);
        }
        return;
    }
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t / s.B, b = t - a * s.B;
        const double* src = s.in + a * s.K * s.B + b;
        double m = kNegInf;
        for (int k = 0; k < s.K; ++k) m = fmax(m, src[(int64_t)k * s.B]);
        if (!isfinite(m)) m = 0.0;
        s.rmax[t] = m;
        double* dst = s.w + a * s.K * s.B + b;
        for (int k = 0; k < s.K; ++k) dst[(int64_t)k * s.B] = exp(src[(int64_t)k * s.B] - m);
    }
}

__global__ void g_contract_kernel(GStage s) {
    if (s.stop && *s.stop) return;
    const int64_t n = (int64_t)s.A * s.O * s.B;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ob = (int64_t)s.O * s.B;
        const int64_t a = t / ob;
        const int64_t r = t - a * ob;
        const int o = (int)(r / s.B);
        const int64_t b = r - (int64_t)o * s.B;
        const double* w = s.w + a * s.K * s.B + b;
        const double* tb = s.tab + o;
        double S = 0.0;
        for (int k = 0; k < s.K; ++k) S = fma(w[(int64_t)k * s.B], tb[(int64_t)k * s.O], S);
        double res;
        if (S >= kTiny) {
            res = log(S) + s.rmax[a * s.B + b];
        } else {
            // exact stage-wise value (sinkhorn.py:57-67 _lse over this axis)
            const double* src = s.in + a * s.K * s.B + b;
            const double p = s.p_org + s.p_dx * (double)o;
            double m = kNegInf;
            for (int k = 0; k < s.K; ++k) {
                const double d = p - (s.q_org + s.q_dx * (double)k);
                m = fmax(m, src[(int64_t)k * s.B] + (-(d * d) / s.eps));
            }
            if (!isfinite(m)) m = 0.0;
            double acc = 0.0;
            for (int k = 0; k < s.K; ++k) {
                const double d = p - (s.q_org + s.q_dx * (double)k);
                acc += exp(src[(int64_t)k * s.B] + (-(d * d) / s.eps) - m);
            }
            res = log(acc) + m;
        }
        s.out[t] = res;
    }
}

// ---- prolongation -----------------------------------------------------------------

__device__ __forceinline__ void lin_axis(int f, int nc, int& i0, int& i1, double& w) {
    i0 = 0; i1 = 0; w = 0.0;
    if (nc > 1) {
        const double p = 0.5 * (double)f - 0.25;
        const double pc = fmin(fmax(p, 0.0), (double)(nc - 1));
        i0 = min((int)floor(pc), nc - 2);
        i1 = i0 + 1;
        w = pc - (double)i0;
    }
}

__global__ void prolong3_kernel(int f0, int f1, int f2, int c0, int c1, int c2,
                                const double* c, double* f) {
    const int64_t n = (int64_t)f0 * f1 * f2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int r0, r1, r2;
        unflat(t, f1, f2, r0, r1, r2);
        int a0, a1, b0, b1, d0, d1;
        double wa, wb, wd;
        lin_axis(r0, c0, a0, a1, wa);
        lin_axis(r1, c1, b0, b1, wb);
        lin_axis(r2, c2, d0, d1, wd);
        auto C = [&](int i, int j, int k) { return c[((int64_t)i * c1 + j) * c2 + k]; };
        const double lo = (1.0 - wb) * ((1.0 - wd) * C(a0, b0, d0) + wd * C(a0, b0, d1)) +
                          wb * ((1.0 - wd) * C(a0, b1, d0) + wd * C(a0, b1, d1));
        const double hi = (1.0 - wb) * ((1.0 - wd) * C(a1, b0, d0) + wd * C(a1, b0, d1)) +
                          wb * ((1.0 - wd) * C(a1, b1, d0) + wd * C(a1, b1, d1));
        f[t] = (1.0 - wa) * lo + wa * hi;
    }
}

// ---- cell workspace ------------------------------------------------------------------

struct WsL {
    int64_t mu, lmu, alpha, L, av;          // X window (nx each)
    int64_t lnu, m, lm, beta, z;            // Y window (ny each)
    int64_t kn[3], c[3];                    // per-axis tables w_a x n_a, column shifts n_a
    int64_t s1, s2;                         // stage scratch
    int64_t total;
};

__host__ __device__ inline WsL ws_layout(const int* w, const int* n) {
    WsL l;
    const int64_t nx = (int64_t)w[0] * w[1] * w[2];
    const int64_t ny = (int64_t)n[0] * n[1] * n[2];
    int64_t p = 0;
    l.mu = p; p += nx;
    l.lmu = p; p += nx;
    l.alpha = p; p += nx;
    l.L = p; p += nx;
    l.av = p; p += nx;
    l.lnu = p; p += ny;
    l.m = p; p += ny;
    l.lm = p; p += ny;
    l.beta = p; p += ny;
    l.z = p; p += ny;
    for (int a = 0; a < 3; ++a) { l.kn[a] = p; p += (int64_t)w[a] * n[a]; }
    for (int a = 0; a < 3; ++a) { l.c[a] = p; p += n[a]; }
    const int64_t s1a = (int64_t)w[0] * w[1] * n[2], s1b = (int64_t)n[0] * n[1] * w[2];
    const int64_t s2a = (int64_t)w[0] * n[1] * n[2], s2b = (int64_t)n[0] * w[1] * w[2];
    l.s1 = p; p += s1a > s1b ? s1a : s1b;
    l.s2 = p; p += s2a > s2b ? s2a : s2b;
    l.total = p + 1;
    return l;
}

struct Cell {
    int w[3], n[3];
    int64_t nx, ny;
    B3 xb, yb;
    double *mu, *lmu, *alpha, *L, *av, *lnu, *m, *lm, *beta, *z, *kn[3], *c[3], *s1, *s2;
};

// Mixed-radix position (i0, i1, i2) over dims (., n1, n2) of the flat index
// t = (i0*n1 + i1)*n2 + i2, advanced by T per step without divisions (the block
// loops below visit t = threadIdx.x, threadIdx.x + T, ...).
template <int T>
struct Step3 {
    int i0, i1, i2, s0, s1, s2, n1, n2;
    __device__ __forceinline__ Step3(int t, int n1_, int n2_) : n1(n1_), n2(n2_) {
        const unsigned q = (unsigned)t / (unsigned)n2;
        i2 = t - (int)q * n2;
        i0 = (int)(q / (unsigned)n1);
        i1 = (int)q - i0 * n1;
        const unsigned qs = (unsigned)T / (unsigned)n2;
        s2 = T - (int)qs * n2;
        s0 = (int)(qs / (unsigned)n1);
        s1 = (int)qs - s0 * n1;
    }
    __device__ __forceinline__ void next() {
        i2 += s2;
        int c = i2 >= n2;
        if (c) i2 -= n2;
        i1 += s1 + c;
        c = i1 >= n1;
        if (c) i1 -= n1;
        i0 += s0 + c;
    }
};

// One in-CTA contraction stage: out[(a*O+o)*B+b] = sum_k in[(a*K+k)*B+b] * tab[k*tk + o*to]
template <int T>
__device__ __forceinline__ void cstage(const double* __restrict__ in, int A, int K, int B, int O,
                                       const double* __restrict__ tab, int tk, int to,
                                       double* __restrict__ out) {
    const int n = A * O * B;
    Step3<T> p(threadIdx.x, O, B);
    for (int t = threadIdx.x; t < n; t += T, p.next()) {
        const double* src = in + (p.i0 * K) * B + p.i2;
        const double* tp = tab + p.i1 * to;
        double S = 0.0;
        for (int k = 0; k < K; ++k) S = fma(src[k * B], tp[k * tk], S);
        out[t] = S;
    }
    __syncthreads();
}

// Exact stage: out[(a*O+o)*B+b] = log sum_k exp(in[(a*K+k)*B+b] - (p_o - q_k)^2 / eps)
template <int T>
__device__ __forceinline__ void xstage(const double* __restrict__ in, int A, int K, int B, int O,
                                       double po, double pdx, int poff, double qo, double qdx,
                                       int qoff, double eps, double* __restrict__ out) {
    const int n = A * O * B;
    Step3<T> q(threadIdx.x, O, B);
    for (int t = threadIdx.x; t < n; t += T, q.next()) {
        const double* src = in + (q.i0 * K) * B + q.i2;
        const double p = po + pdx * (double)(poff + q.i1);
        double m = kNegInf;
        for (int k = 0; k < K; ++k) {
            const double d = p - (qo + qdx * (double)(qoff + k));
            m = fmax(m, src[k * B] + (-(d * d) / eps));
        }
        if (!isfinite(m)) m = 0.0;
        double acc = 0.0;
        for (int k = 0; k < K; ++k) {
            const double d = p - (qo + qdx * (double)(qoff + k));
            acc += exp(src[k * B] + (-(d * d) / eps) - m);
        }
        out[t] = log(acc) + m;
    }
    __syncthreads();
}

struct Sh {
    double red[32];
    int redi[32];
    int flag;
    int ndeg;
    // fp32 mode: per-axis slopes the current tables absorb, rebuild request, force flag
    double slope[3];
    int rebuild;
    int force;
};

// X sweep: L[x] = log sum_y exp(b[y] - c(x,y)/eps), b = beta/eps + lnu.
// Fast path writes L; returns 1 if an output needed the exact path (then redone).
template <int T>
__device__ int sweep_x(const Cell& C, const dd3_geom& g, Sh& sh) {
    const double eps = g.eps;
    const int ny = (int)C.ny, nx = (int)C.nx;
    // b' = b + sum_a c_a(y_a) into z (scratch), and its max
    double mx = kNegInf;
    {
        Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
        for (int y = threadIdx.x; y < ny; y += T, p.next()) {
            const double b = C.beta[y] / eps + C.lnu[y];
            const double bp = b + (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]);
            C.z[y] = bp;
            mx = fmax(mx, bp);
        }
    }
    double M = bmax<T>(mx, sh.red);
    if (!isfinite(M)) M = 0.0;
    for (int y = threadIdx.x; y < ny; y += T) C.z[y] = exp(C.z[y] - M);
    if (threadIdx.x == 0) sh.flag = 0;
    __syncthreads();
    // U1[y0,y1,x2] = sum_y2 w * Kn2[x2][y2]; U2[y0,x1,x2]; S[x0,x1,x2]
    cstage<T>(C.z, C.n[0] * C.n[1], C.n[2], 1, C.w[2], C.kn[2], 1, C.n[2], C.s1);
    cstage<T>(C.s1, C.n[0], C.n[1], C.w[2], C.w[1], C.kn[1], 1, C.n[1], C.s2);
    int bad = 0;
    {
        const int ob = C.w[1] * C.w[2];
        const int n0 = C.n[0];
        Step3<T> p(threadIdx.x, 1, ob);
        for (int t = threadIdx.x; t < nx; t += T, p.next()) {
            const double* s2 = C.s2 + p.i2;
            const double* kt = C.kn[0] + p.i0 * n0;
            double S = 0.0;
            for (int k = 0; k < n0; ++k) S = fma(s2[k * ob], kt[k], S);
            if (!(S >= kTiny)) bad = 1;
            C.L[t] = log(S) + M;
        }
    }
    if (bad) sh.flag = 1;
    __syncthreads();
    if (!sh.flag) return 0;
    // exact stage-wise path on b = beta/eps + lnu
    for (int y = threadIdx.x; y < ny; y += T) C.z[y] = C.beta[y] / eps + C.lnu[y];
    __syncthreads();
    const int* xo = C.xb.o;
    const int* yo = C.yb.o;
    xstage<T>(C.z, C.n[0] * C.n[1], C.n[2], 1, C.w[2], g.x_org[2], g.x_dx, xo[2], g.y_org[2],
           g.y_dx, yo[2], eps, C.s1);
    xstage<T>(C.s1, C.n[0], C.n[1], C.w[2], C.w[1], g.x_org[1], g.x_dx, xo[1], g.y_org[1], g.y_dx,
           yo[1], eps, C.s2);
    xstage<T>(C.s2, 1, C.n[0], C.w[1] * C.w[2], C.w[0], g.x_org[0], g.x_dx, xo[0], g.y_org[0],
           g.y_dx, yo[0], eps, C.L);
    return 1;
}

// Y sweep: z[y] = log sum_x exp(a[x] - c(x,y)/eps), a = alpha/eps + lmu (built into av).
template <int T>
__device__ int sweep_y(const Cell& C, const dd3_geom& g, Sh& sh) {
    const double eps = g.eps;
    const int ny = (int)C.ny, nx = (int)C.nx;
    double mx = kNegInf;
    for (int x = threadIdx.x; x < nx; x += T) {
        const double a = C.alpha[x] / eps + C.lmu[x];
        C.av[x] = a;
        mx = fmax(mx, a);
    }
    double M = bmax<T>(mx, sh.red);
    if (!isfinite(M)) M = 0.0;
    // shifted weights into L (rebuilt by the next X sweep)
    for (int x = threadIdx.x; x < nx; x += T) C.L[x] = exp(C.av[x] - M);
    if (threadIdx.x == 0) sh.flag = 0;
    __syncthreads();
    // T1[x0,x1,y2] = sum_x2 w * Kn2[x2][y2]; T2[x0,y1,y2]; S[y0,y1,y2]
    cstage<T>(C.L, C.w[0] * C.w[1], C.w[2], 1, C.n[2], C.kn[2], C.n[2], 1, C.s1);
    cstage<T>(C.s1, C.w[0], C.w[1], C.n[2], C.n[1], C.kn[1], C.n[1], 1, C.s2);
    int bad = 0;
    {
        const int ob = C.n[1] * C.n[2];
        const int n0 = C.n[0], w0 = C.w[0];
        Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
        for (int t = threadIdx.x; t < ny; t += T, p.next()) {
            const double* s2 = C.s2 + (p.i1 * C.n[2] + p.i2);
            const double* kt = C.kn[0] + p.i0;
            double S = 0.0;
            for (int k = 0; k < w0; ++k) S = fma(s2[k * ob], kt[k * n0], S);
            if (!(S >= kTiny)) bad = 1;
            C.z[t] = log(S) + M + (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]);
        }
    }
    if (bad) sh.flag = 1;
    __syncthreads();
    if (!sh.flag) return 0;
    const int* xo = C.xb.o;
    const int* yo = C.yb.o;
    xstage<T>(C.av, C.w[0] * C.w[1], C.w[2], 1, C.n[2], g.y_org[2], g.y_dx, yo[2], g.x_org[2],
           g.x_dx, xo[2], eps, C.s1);
    xstage<T>(C.s1, C.w[0], C.w[1], C.n[2], C.n[1], g.y_org[1], g.y_dx, yo[1], g.x_org[1], g.x_dx,
           xo[1], eps, C.s2);
    xstage<T>(C.s2, 1, C.w[0], C.n[1] * C.n[2], C.n[0], g.y_org[0], g.y_dx, yo[0], g.x_org[0],
           g.x_dx, xo[0], eps, C.z);
    return 1;
}

// lam-free gap sum (sinkhorn.py:336-351) over the X window
template <int T>
__device__ double gap_sum(const Cell& C, const dd3_geom& g, Sh& sh) {
    double s = 0.0;
    for (int64_t x = threadIdx.x; x < C.nx; x += T) {
        const double mu = C.mu[x];
        if (mu > 0) {
            const double a = C.alpha[x];
            const double lr = a / g.eps + C.L[x];
            const double px = mu * exp(lr);
            const double ref = mu * exp(-a / g.lam);
            s += px * (lr + a / g.lam) - px + ref;
        }
    }
    return bsum<T>(s, sh.red);
}

__device__ __forceinline__ double coord(const double* org, double dx, int a, int idx) {
    return org[a] + dx * (double)idx;
}

// ---- fp32 mode of the fast sweeps (north_star fp32 mode: 1e-4 relative) ---------------
// The six contractions, their tables, weights and stage intermediates run in fp32; the
// state (alpha, beta, L, z), the Newton Y-step, the gap test and the epilogue stay fp64.
// A cell's X-side potential a = alpha/eps + log mu varies by (displacement / h) per node,
// hundreds across the 2s-node window: more than fp32's exponent range, so one global
// shift would underflow the dominant terms of most outputs.  Its linear part is
// absorbed into the per-axis tables instead (still separable):
//   a[x] - c(x,y)/eps = (a[x] - s.x) + sum_a (-(x_a - y_a)^2/eps + s_a x_a)
//   L[x] + s.x        = log sum_y exp(b[y]) prod_a exp(-(x_a - y_a)^2/eps + s_a x_a)
// with s_a the per-node slope of alpha/eps along axis a (x_a = window index), so the
// shifted weights of both sweeps stay O(curvature).  Tables are Y-normalised as in the
// fp64 path (column shifts c_a in fp64) and rebuilt when a slope moves by more than
// kSlopeTol over the window.  An output whose shifted fp32 sum is below kTinyF may have
// lost terms to underflow: that sweep is redone by the exact fp64 stage-wise path and
// the slopes are refreshed.
constexpr float kTinyF = 1e-30f;
constexpr double kSlopeTol = 4.0;

__device__ __forceinline__ float* f32p(double* p) { return reinterpret_cast<float*>(p); }

// slopes of alpha/eps along the window's centre lines (one thread)
__device__ __forceinline__ void slopes_now(const Cell& C, double eps, double* s) {
    const int m0 = C.w[0] / 2, m1 = C.w[1] / 2, m2 = C.w[2] / 2;
    const int w1 = C.w[1], w2 = C.w[2];
    s[0] = C.w[0] > 1 ? (C.alpha[((C.w[0] - 1) * w1 + m1) * w2 + m2] - C.alpha[m1 * w2 + m2]) /
                            ((C.w[0] - 1) * eps) : 0.0;
    s[1] = w1 > 1 ? (C.alpha[(m0 * w1 + w1 - 1) * w2 + m2] - C.alpha[(m0 * w1) * w2 + m2]) /
                        ((w1 - 1) * eps) : 0.0;
    s[2] = w2 > 1 ? (C.alpha[(m0 * w1 + m1) * w2 + w2 - 1] - C.alpha[(m0 * w1 + m1) * w2]) /
                        ((w2 - 1) * eps) : 0.0;
    for (int a = 0; a < 3; ++a) if (!isfinite(s[a])) s[a] = 0.0;
}

// Tf_a[x_a][y_a] = exp(-(d^2)/eps + s_a x_a - c_a(y_a)), c_a(y_a) = max over x_a (fp64)
template <int T>
__device__ void build_tables_f32(const Cell& C, const dd3_geom& g, const Sh& sh) {
    const double eps = g.eps;
    for (int a = 0; a < 3; ++a) {
        const double sa = sh.slope[a];
        float* tf = f32p(C.kn[a]);
        for (int ya = threadIdx.x; ya < C.n[a]; ya += T) {
            const double yc = coord(g.y_org, g.y_dx, a, C.yb.o[a] + ya);
            double cm = kNegInf;
            for (int xa = 0; xa < C.w[a]; ++xa) {
                const double dd_ = coord(g.x_org, g.x_dx, a, C.xb.o[a] + xa) - yc;
                cm = fmax(cm, -(dd_ * dd_) / eps + sa * (double)xa);
            }
            C.c[a][ya] = cm;
            for (int xa = 0; xa < C.w[a]; ++xa) {
                const double dd_ = coord(g.x_org, g.x_dx, a, C.xb.o[a] + xa) - yc;
                tf[(int64_t)xa * C.n[a] + ya] = expf((float)(-(dd_ * dd_) / eps + sa * (double)xa - cm));
            }
        }
    }
    __syncthreads();
}

// Thread 0 compares the slopes of the current alpha with the ones the tables absorb;
// the tables are rebuilt when one moved by more than kSlopeTol over the window (or after
// a fallback).  Called by every thread after a barrier that published alpha.
template <int T>
__device__ void refresh_tables_f32(const Cell& C, const dd3_geom& g, Sh& sh) {
    if (threadIdx.x == 0) {
        double s[3];
        slopes_now(C, g.eps, s);
        int mv = sh.force;
        for (int a = 0; a < 3; ++a)
            if (fabs(s[a] - sh.slope[a]) * (double)(C.w[a] - 1) > kSlopeTol) mv = 1;
        if (mv) for (int a = 0; a < 3; ++a) sh.slope[a] = s[a];
        sh.rebuild = mv;
        sh.force = 0;
    }
    __syncthreads();
    if (sh.rebuild) build_tables_f32<T>(C, g, sh);
}

// fp32 contraction stage (cstage's indexing)
template <int T>
__device__ __forceinline__ void cstage32(const float* __restrict__ in, int A, int K, int B, int O,
                                         const float* __restrict__ tab, int tk, int to,
                                         float* __restrict__ out) {
    const int n = A * O * B;
    Step3<T> p(threadIdx.x, O, B);
    for (int t = threadIdx.x; t < n; t += T, p.next()) {
        const float* src = in + (p.i0 * K) * B + p.i2;
        const float* tp = tab + p.i1 * to;
        float S0 = 0.f, S1 = 0.f;
        int k = 0;
        for (; k + 1 < K; k += 2) {
            S0 = fmaf(src[k * B], tp[k * tk], S0);
            S1 = fmaf(src[(k + 1) * B], tp[(k + 1) * tk], S1);
        }
        if (k < K) S0 = fmaf(src[k * B], tp[k * tk], S0);
        out[t] = S0 + S1;
    }
    __syncthreads();
}

template <int T>
__device__ int sweep_x32(const Cell& C, const dd3_geom& g, Sh& sh) {
    const double eps = g.eps, inv_eps = 1.0 / g.eps;
    const int ny = (int)C.ny, nx = (int)C.nx;
    const double sl0 = sh.slope[0], sl1 = sh.slope[1], sl2 = sh.slope[2];
    double mx = kNegInf;
    {
        Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
        for (int y = threadIdx.x; y < ny; y += T, p.next()) {
            const double bp = C.beta[y] * inv_eps + C.lnu[y] +
                              (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]);
            mx = fmax(mx, bp);
        }
    }
    double M = bmax<T>(mx, sh.red);
    if (!isfinite(M)) M = 0.0;
    float* zf = f32p(C.z);
    float* s1f = f32p(C.s1);
    float* s2f = f32p(C.s2);
    {
        Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
        for (int y = threadIdx.x; y < ny; y += T, p.next()) {
            const double bp = C.beta[y] * inv_eps + C.lnu[y] +
                              (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]);
            zf[y] = expf((float)(bp - M));
        }
    }
    if (threadIdx.x == 0) sh.flag = 0;
    __syncthreads();
    cstage32<T>(zf, C.n[0] * C.n[1], C.n[2], 1, C.w[2], f32p(C.kn[2]), 1, C.n[2], s1f);
    cstage32<T>(s1f, C.n[0], C.n[1], C.w[2], C.w[1], f32p(C.kn[1]), 1, C.n[1], s2f);
    int bad = 0;
    {
        const int ob = C.w[1] * C.w[2];
        const int n0 = C.n[0];
        const float* k0 = f32p(C.kn[0]);
        for (int t = threadIdx.x; t < nx; t += T) {
            int x0, x1, x2;
            unflat(t, C.w[1], C.w[2], x0, x1, x2);
            const float* s2 = s2f + (x1 * C.w[2] + x2);
            const float* kt = k0 + x0 * n0;
            float S0 = 0.f, S1 = 0.f;
            int k = 0;
            for (; k + 1 < n0; k += 2) {
                S0 = fmaf(s2[k * ob], kt[k], S0);
                S1 = fmaf(s2[(k + 1) * ob], kt[k + 1], S1);
            }
            if (k < n0) S0 = fmaf(s2[k * ob], kt[k], S0);
            const float S = S0 + S1;
            if (!(S >= kTinyF)) bad = 1;
            C.L[t] = (double)logf(S) + M - (sl0 * (double)x0 + sl1 * (double)x1 + sl2 * (double)x2);
        }
    }
    if (bad) sh.flag = 1;
    __syncthreads();
    if (!sh.flag) return 0;
    // exact stage-wise path on b = beta/eps + lnu (fp64); slopes refreshed afterwards
    for (int y = threadIdx.x; y < ny; y += T) C.z[y] = C.beta[y] / eps + C.lnu[y];
    if (threadIdx.x == 0) sh.force = 1;
    __syncthreads();
    const int* xo = C.xb.o;
    const int* yo = C.yb.o;
    xstage<T>(C.z, C.n[0] * C.n[1], C.n[2], 1, C.w[2], g.x_org[2], g.x_dx, xo[2], g.y_org[2],
           g.y_dx, yo[2], eps, C.s1);
    xstage<T>(C.s1, C.n[0], C.n[1], C.w[2], C.w[1], g.x_org[1], g.x_dx, xo[1], g.y_org[1], g.y_dx,
           yo[1], eps, C.s2);
    xstage<T>(C.s2, 1, C.n[0], C.w[1] * C.w[2], C.w[0], g.x_org[0], g.x_dx, xo[0], g.y_org[0],
           g.y_dx, yo[0], eps, C.L);
    return 1;
}

template <int T>
__device__ int sweep_y32(const Cell& C, const dd3_geom& g, Sh& sh) {
    const double eps = g.eps, inv_eps = 1.0 / g.eps;
    const int ny = (int)C.ny, nx = (int)C.nx;
    const double sl0 = sh.slope[0], sl1 = sh.slope[1], sl2 = sh.slope[2];
    double mx = kNegInf;
    for (int x = threadIdx.x; x < nx; x += T) {
        int x0, x1, x2;
        unflat(x, C.w[1], C.w[2], x0, x1, x2);
        const double a = C.alpha[x] * inv_eps + C.lmu[x];
        C.av[x] = a;
        mx = fmax(mx, a - (sl0 * (double)x0 + sl1 * (double)x1 + sl2 * (double)x2));
    }
    double M = bmax<T>(mx, sh.red);
    if (!isfinite(M)) M = 0.0;
    float* lf = f32p(C.L);
    float* s1f = f32p(C.s1);
    float* s2f = f32p(C.s2);
    for (int x = threadIdx.x; x < nx; x += T) {
        int x0, x1, x2;
        unflat(x, C.w[1], C.w[2], x0, x1, x2);
        lf[x] = expf((float)(C.av[x] - (sl0 * (double)x0 + sl1 * (double)x1 + sl2 * (double)x2) - M));
    }
    if (threadIdx.x == 0) sh.flag = 0;
    __syncthreads();
    cstage32<T>(lf, C.w[0] * C.w[1], C.w[2], 1, C.n[2], f32p(C.kn[2]), C.n[2], 1, s1f);
    cstage32<T>(s1f, C.w[0], C.w[1], C.n[2], C.n[1], f32p(C.kn[1]), C.n[1], 1, s2f);
    int bad = 0;
    {
        const int ob = C.n[1] * C.n[2];
        const int n0 = C.n[0], w0 = C.w[0];
        const float* k0 = f32p(C.kn[0]);
        Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
        for (int t = threadIdx.x; t < ny; t += T, p.next()) {
            const float* s2 = s2f + (p.i1 * C.n[2] + p.i2);
            const float* kt = k0 + p.i0;
            float S0 = 0.f, S1 = 0.f;
            int k = 0;
            for (; k + 1 < w0; k += 2) {
                S0 = fmaf(s2[k * ob], kt[k * n0], S0);
                S1 = fmaf(s2[(k + 1) * ob], kt[(k + 1) * n0], S1);
            }
            if (k < w0) S0 = fmaf(s2[k * ob], kt[k * n0], S0);
            const float S = S0 + S1;
            if (!(S >= kTinyF)) bad = 1;
            C.z[t] = (double)logf(S) + M + (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]);
        }
    }
    if (bad) sh.flag = 1;
    __syncthreads();
    if (!sh.flag) return 0;
    if (threadIdx.x == 0) sh.force = 1;
    const int* xo = C.xb.o;
    const int* yo = C.yb.o;
    xstage<T>(C.av, C.w[0] * C.w[1], C.w[2], 1, C.n[2], g.y_org[2], g.y_dx, yo[2], g.x_org[2],
           g.x_dx, xo[2], eps, C.s1);
    xstage<T>(C.s1, C.w[0], C.w[1], C.n[2], C.n[1], g.y_org[1], g.y_dx, yo[1], g.x_org[1], g.x_dx,
           xo[1], eps, C.s2);
    xstage<T>(C.s2, 1, C.w[0], C.n[1] * C.n[2], C.n[0], g.y_org[0], g.y_dx, yo[0], g.x_org[0],
           g.x_dx, xo[0], eps, C.z);
    return 1;
}

// cost and -cost/eps of window nodes x (X window index) and y (Y window index)
__device__ __forceinline__ double cell_cost(const Cell& C, const dd3_geom& g, int x0, int x1,
                                            int x2, int y0, int y1, int y2) {
    const double d0 = coord(g.x_org, g.x_dx, 0, C.xb.o[0] + x0) - coord(g.y_org, g.y_dx, 0, C.yb.o[0] + y0);
    const double d1 = coord(g.x_org, g.x_dx, 1, C.xb.o[1] + x1) - coord(g.y_org, g.y_dx, 1, C.yb.o[1] + y1);
    const double d2 = coord(g.x_org, g.x_dx, 2, C.xb.o[2] + x2) - coord(g.y_org, g.y_dx, 2, C.yb.o[2] + y2);
    return d0 * d0 + d1 * d1 + d2 * d2;
}

// Y-normalised fp64 tables Kn_a[x_a][y_a] = exp(-(d^2)/eps - c_a(y_a)), c_a = max over x_a
template <int T>
__device__ void build_tables_f64(const Cell& C, const dd3_geom& g) {
    const double eps = g.eps;
    for (int a = 0; a < 3; ++a) {
        for (int ya = threadIdx.x; ya < C.n[a]; ya += T) {
            const double yc = coord(g.y_org, g.y_dx, a, C.yb.o[a] + ya);
            double cm = kNegInf;
            for (int xa = 0; xa < C.w[a]; ++xa) {
                const double dd_ = coord(g.x_org, g.x_dx, a, C.xb.o[a] + xa) - yc;
                cm = fmax(cm, -(dd_ * dd_) / eps);
            }
            C.c[a][ya] = cm;
            for (int xa = 0; xa < C.w[a]; ++xa) {
                const double dd_ = coord(g.x_org, g.x_dx, a, C.xb.o[a] + xa) - yc;
                C.kn[a][(int64_t)xa * C.n[a] + ya] = exp(-(dd_ * dd_) / eps - cm);
            }
        }
    }
}

// cstage with the squared axis distance folded in (x -> y direction, tab[k*tk + o]):
//   out[(a*O+o)*B+b] (+)= sum_k in[(a*K+k)*B+b] * d(k,o)^2 * tab[k*tk + o],
// d(k,o) = x coordinate of window node xi0 + k minus y coordinate of window node o.
template <int T>
__device__ __forceinline__ void cstage_sq(const double* __restrict__ in, int A, int K, int B, int O,
                                          const double* __restrict__ tab, int tk, const Cell& C,
                                          const dd3_geom& g, int axis, int xi0, bool accumulate,
                                          double* __restrict__ out) {
    const int n = A * O * B;
    Step3<T> p(threadIdx.x, O, B);
    for (int t = threadIdx.x; t < n; t += T, p.next()) {
        const double* src = in + (p.i0 * K) * B + p.i2;
        const double* tp = tab + p.i1;
        const double yc = coord(g.y_org, g.y_dx, axis, C.yb.o[axis] + p.i1);
        double S = 0.0;
        for (int k = 0; k < K; ++k) {
            const double d = coord(g.x_org, g.x_dx, axis, C.xb.o[axis] + xi0 + k) - yc;
            S = fma(src[k * B] * (d * d), tp[k * tk], S);
        }
        out[t] = accumulate ? out[t] + S : S;
    }
    __syncthreads();
}

// ---- the cell solve kernel -----------------------------------------------------------

__device__ __forceinline__ void member_block(const dd3_state& s, const Cell& C, int i, int* lo,
                                             int* be) {
    const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = bx.o[a] - C.xb.o[a];
        be[a] = bx.e[a];
    }
}

#ifndef DD3_MIN_BLOCKS
#define DD3_MIN_BLOCKS 2   // resident cell CTAs per SM (2: <= 128 registers, no spills)
#endif
template <int T, int F32>
__global__ void __launch_bounds__(T, T >= 512 ? 1 : DD3_MIN_BLOCKS)
    cell_solve3_kernel(dd3_geom g, dd3_state s, dd3_batch b) {
    __shared__ Sh sh;
    __shared__ double smem_d[64 * 6];
    const int c = blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 16;
    const int j = d[0];
    Cell C;
    C.xb = ldbox(d + 1);
    C.yb = ldbox(d + 7);
    const int n_mem = d[13], mb = d[14];
    for (int a = 0; a < 3; ++a) { C.w[a] = b.nxw[a]; C.n[a] = C.yb.e[a]; }
    C.nx = (int64_t)C.w[0] * C.w[1] * C.w[2];
    C.ny = (int64_t)C.n[0] * C.n[1] * C.n[2];
    const int64_t yoff = b.offs[(int64_t)c * 4 + 0], moff = b.offs[(int64_t)c * 4 + 1];
    const int64_t woff = b.offs[(int64_t)c * 4 + 2], xoff = b.offs[(int64_t)c * 4 + 3];
    const WsL l = ws_layout(C.w, C.n);
    double* W = b.work + woff;
    C.mu = W + l.mu; C.lmu = W + l.lmu; C.alpha = W + l.alpha; C.L = W + l.L; C.av = W + l.av;
    C.lnu = W + l.lnu; C.m = W + l.m; C.lm = W + l.lm; C.beta = W + l.beta; C.z = W + l.z;
    for (int a = 0; a < 3; ++a) { C.kn[a] = W + l.kn[a]; C.c[a] = W + l.c[a]; }
    C.s1 = W + l.s1; C.s2 = W + l.s2;
    {
        // the arrays every Sinkhorn iteration re-reads (z, beta, the stage scratch, the axis
        // tables) in shared memory when they fit this CTA's dynamic allocation
        extern __shared__ double dyn[];
        const int64_t s1n = l.s2 - l.s1, s2n = l.total - 1 - l.s2;
        const int64_t tabn = l.s1 - l.kn[0];
        const int64_t need = 2 * C.ny + s1n + s2n + tabn;
        if (need <= b.smem_doubles) {
            double* p = dyn;
            C.z = p; p += C.ny;
            C.beta = p; p += C.ny;
            C.s1 = p; p += s1n;
            C.s2 = p; p += s2n;
            for (int a = 0; a < 3; ++a) { C.kn[a] = p + (l.kn[a] - l.kn[0]); C.c[a] = p + (l.c[a] - l.kn[0]); }
        }
    }
    const double eps = g.eps, lam = g.lam;
    const double ratio = eps * lam / (eps + lam);
    const int bs = s.block[0] * s.block[1] * s.block[2];
    const int has = s.d_has[j];
    // X window (cells.py:188 extract_window, fill 0 off the grid)
    double ms = 0.0;
    for (int64_t x = threadIdx.x; x < C.nx; x += T) {
        int x0, x1, x2;
        unflat(x, C.w[1], C.w[2], x0, x1, x2);
        const int r0 = C.xb.o[0] + x0, r1 = C.xb.o[1] + x1, r2 = C.xb.o[2] + x2;
        double mu = 0.0, lmu = kNegInf;
        if (r0 >= 0 && r0 < g.nx[0] && r1 >= 0 && r1 < g.nx[1] && r2 >= 0 && r2 < g.nx[2]) {
            const int64_t id = ((int64_t)r0 * g.nx[1] + r1) * g.nx[2] + r2;
            mu = s.mu[id];
            lmu = mu > 0 ? s.log_mu[id] : kNegInf;
        }
        C.mu[x] = mu;
        C.lmu[x] = lmu;
        C.alpha[x] = has ? s.d_alpha[(int64_t)j * C.nx + x] : 0.0;
        ms += mu;
    }
    const double mass = bsum<T>(ms, sh.red);
    // member blocks and the old member boxes
    int* mlo = (int*)smem_d;                     // [64*3]
    int* mbe = mlo + 64 * 3;                     // [64*3]
    __shared__ int32_t sobox[64 * 6];
    for (int k = threadIdx.x; k < n_mem; k += T) {
        const int i = b.members[mb + k];
        member_block(s, C, i, mlo + 3 * k, mbe + 3 * k);
        for (int q = 0; q < 6; ++q) sobox[k * 6 + q] = s.ybox[(int64_t)i * 6 + q];
    }
    __syncthreads();
    double* R = b.marena + moff;                 // raw split, later f
    double* V = R + (int64_t)n_mem * C.ny;       // member values
    double* TC = V + (int64_t)n_mem * C.ny;
    double* TL = TC + (int64_t)n_mem * C.ny;
    double* MC = TL + (int64_t)n_mem * C.ny;
    double* cst = b.cstat + (int64_t)c * 8;
    double* cst2 = b.cstat2 + (int64_t)c * 8;
    // Y window: log nu, background m = clip(snapshot - own, 0) / nu (cells.py:141-160),
    // warm beta reboxed from the dual store (cells.py:207-212)
    B3 db;
    if (has) db = ldbox(s.d_box + (int64_t)j * 6);
    const double* dbeta = s.d_beta + (int64_t)j * s.d_cap;
    int nclamp = 0;
    for (int64_t y = threadIdx.x; y < C.ny; y += T) {
        int y0, y1, y2;
        unflat(y, C.n[1], C.n[2], y0, y1, y2);
        const int r0 = C.yb.o[0] + y0, r1 = C.yb.o[1] + y1, r2 = C.yb.o[2] + y2;
        const int64_t id = ((int64_t)r0 * g.ny[1] + r1) * g.ny[2] + r2;
        const double nu = s.nu[id];
        double own = 0.0;
        for (int k = 0; k < n_mem; ++k) {
            const int i = b.members[mb + k];
            B3 ob;
            for (int a = 0; a < 3; ++a) { ob.o[a] = sobox[k * 6 + 2 * a]; ob.e[a] = sobox[k * 6 + 2 * a + 1]; }
            own += bempty(ob) ? 0.0 : bat(ob, s.yval + (int64_t)i * s.cap, r0, r1, r2);
        }
        const double pw = b.snapshot[id];
        const double diff = pw - own;
        if (diff < -1e-12 * fmax(pw, own)) ++nclamp;
        const double m = fmax(diff, 0.0) / nu;
        C.lnu[y] = s.log_nu[id];
        C.m[y] = m;
        C.lm[y] = m > 0 ? log(m) : kNegInf;
        C.beta[y] = has ? bat(db, dbeta, r0, r1, r2) : 0.0;
        b.mdens[yoff + y] = m;
    }
    // per-axis Y-normalised tables Kn_a[x_a][y_a] = exp(-(d^2)/eps - c_a(y_a)),
    // c_a(y_a) = max over x_a of -(d^2)/eps
    if (!F32) build_tables_f64<T>(C, g);
    const int nclamped = (int)bsum<T>((double)nclamp, sh.red);   // (barrier)
    if (!(mass > 0)) {
        // zero-mass cell: untouched, converged (cells.py:245-264)
        for (int64_t x = threadIdx.x; x < C.nx; x += T) b.alpha[(int64_t)c * C.nx + x] = C.alpha[x];
        for (int64_t y = threadIdx.x; y < C.ny; y += T) b.beta[yoff + y] = C.beta[y];
        for (int64_t t = threadIdx.x; t < 2 * (int64_t)n_mem * C.ny; t += T) R[t] = 0.0;
        for (int64_t t = threadIdx.x; t < (int64_t)n_mem * bs; t += T) b.xarena[xoff + t] = 0.0;
        for (int k = threadIdx.x; k < n_mem; k += T) {
            for (int q = 0; q < 6; ++q) b.mbox[(int64_t)(mb + k) * 6 + q] = 0;
            for (int q = 0; q < 4; ++q) b.mstat[(int64_t)(mb + k) * 4 + q] = 0.0;
        }
        if (threadIdx.x == 0) {
            cst[0] = 0; cst[1] = 0; cst[2] = 0; cst[3] = 1; cst[4] = nclamped; cst[5] = 0;
            cst[6] = 0; cst[7] = 0;
            for (int q = 0; q < 8; ++q) cst2[q] = 0.0;
        }
        return;
    }
    // ---- Sinkhorn loop (cells.py:320-348)
    const double thr = b.delta * mass;
    double gap = kInf, first_g = __builtin_nan("");
    bool conv = false, have_first = false;
    int iters = 0, ndeg_max = 0, nfb = 0;
    long long nsteps = 0;        // Newton evaluations of this thread (diagnostic)
    const long long t_loop0 = clock64();
    if (F32) {
        // fp32 mode: tables absorb the slopes of the warm alpha (barrier above published it)
        if (threadIdx.x == 0) sh.force = 1;
        refresh_tables_f32<T>(C, g, sh);
    }
    for (int k = 1; k <= b.max_iters; ++k) {
        nfb += F32 ? sweep_x32<T>(C, g, sh) : sweep_x<T>(C, g, sh);
        if (k >= 2) {
            const double gg = lam * gap_sum<T>(C, g, sh);
            if (!have_first) { first_g = gg; have_first = true; }
            if (gg / lam <= thr) { gap = gg; conv = true; break; }
        }
        for (int64_t x = threadIdx.x; x < C.nx; x += T) C.alpha[x] = -ratio * C.L[x];
        __syncthreads();
        if (F32) refresh_tables_f32<T>(C, g, sh);
        nfb += F32 ? sweep_y32<T>(C, g, sh) : sweep_y<T>(C, g, sh);
        if (threadIdx.x == 0) sh.ndeg = 0;
        __syncthreads();
        int nd = 0;
        for (int64_t y = threadIdx.x; y < C.ny; y += T) {
            int deg = 0;
            C.beta[y] = dd::newton_node(C.z[y], C.m[y], true, C.beta[y], eps, lam, b.newton_tol,
                                        b.newton_max_iters, &deg, &nsteps, nullptr, C.lm[y],
                                        F32 != 0);
            nd += deg;
        }
        if (nd) atomicAdd(&sh.ndeg, nd);
        __syncthreads();
        ndeg_max = max(ndeg_max, sh.ndeg);
        iters = k;
    }
    if (!conv) {
        nfb += F32 ? sweep_x32<T>(C, g, sh) : sweep_x<T>(C, g, sh);
        const double gg = lam * gap_sum<T>(C, g, sh);
        gap = gg;
        if (!have_first) first_g = gg;
        conv = gg / lam <= thr;
    }
    const long long t_loop = clock64() - t_loop0;
    const double nsteps_all = bsum<T>((double)nsteps, sh.red);
    // ---- epilogue: split by members (cells.py:350-393)
    // mu_bar = exp(-alpha'/lam) mu, alpha' = -ratio L (the extra X half-step)
    for (int64_t x = threadIdx.x; x < C.nx; x += T)
        C.av[x] = exp(-(-ratio * C.L[x]) / lam) * C.mu[x];
    __syncthreads();
    // Exact per-term split of member k at Y node y (the reference's dense evaluation)
    auto split_exact = [&](int k, int64_t y) {
        int y0, y1, y2;
        unflat(y, C.n[1], C.n[2], y0, y1, y2);
        const double bt = C.beta[y] / eps;
        const double ln = C.lnu[y];
        const int* lo = mlo + 3 * k;
        const int* be = mbe + 3 * k;
        double sp = 0.0, stc = 0.0, stl = 0.0, smc = 0.0;
        for (int t0 = 0; t0 < be[0]; ++t0)
            for (int t1 = 0; t1 < be[1]; ++t1)
                for (int t2 = 0; t2 < be[2]; ++t2) {
                    const int x0 = lo[0] + t0, x1 = lo[1] + t1, x2 = lo[2] + t2;
                    const int64_t x = ((int64_t)x0 * C.w[1] + x1) * C.w[2] + x2;
                    const double cost = cell_cost(C, g, x0, x1, x2, y0, y1, y2);
                    const double sc = C.alpha[x] / eps + bt + (-cost / eps);
                    const double p = exp(sc + C.lmu[x] + ln);
                    sp += p;
                    stc += p * cost;
                    stl += p * sc;
                    smc += cost * C.mu[x];
                }
        const int64_t q = (int64_t)k * C.ny + y;
        R[q] = sp;
        V[q] = sp;
        TC[q] = stc;
        TL[q] = stl;
        MC[q] = smc;
    };
    // Separable split: per member k the sums over its block x of p = exp(a[x] + b[y] -
    // c(x,y)/eps) (a = alpha/eps + log mu, b = beta/eps + log nu), of p cost and of
    // p alpha/eps are three-stage contractions of the block weights u = exp(a - max a)
    // against the Y-normalised tables (one table carrying d_a^2 for the cost sums);
    // sum p sc follows from sc = alpha/eps + beta/eps - cost/eps.  A node whose shifted
    // sum is below kTiny may have lost terms to underflow and is redone per term.
    // Scratch: block weights and stage-1 outputs in s1, stage-2 outputs in s2.
    bool sep = true;
    {
        const int64_t s1cap = l.s2 - l.s1, s2cap = l.total - 1 - l.s2;
        for (int k = 0; k < n_mem; ++k) {
            const int* be = mbe + 3 * k;
            const int nbk = be[0] * be[1] * be[2];
            if (2 * (int64_t)nbk + 3 * (int64_t)be[0] * be[1] * C.n[2] > s1cap) sep = false;
            if ((int64_t)be[0] * C.n[1] * C.n[2] > s2cap) sep = false;
            if (be[0] > 16 || be[1] > 16 || be[2] > 16) sep = false;
        }
    }
    if (!sep) {
        for (int64_t y = threadIdx.x; y < C.ny; y += T)
            for (int k = 0; k < n_mem; ++k) split_exact(k, y);
        __syncthreads();
    } else {
        if (F32) { build_tables_f64<T>(C, g); __syncthreads(); }
        __shared__ double s_ma[3][16];
        for (int k = 0; k < n_mem; ++k) {
            const int* lo = mlo + 3 * k;
            const int* be = mbe + 3 * k;
            const int nbk = be[0] * be[1] * be[2];
            double* U = C.s1;
            double* UA = U + nbk;
            double* T1 = UA + nbk;
            double* T1a = T1 + be[0] * be[1] * C.n[2];
            double* T1c = T1a + be[0] * be[1] * C.n[2];
            double* T2 = C.s2;
            // block weights, shifted by the block's own maximum; mu marginals per axis
            double amx = kNegInf;
            for (int t = threadIdx.x; t < nbk; t += T) {
                int t0, t1, t2;
                unflat(t, be[1], be[2], t0, t1, t2);
                const int64_t x = ((int64_t)(lo[0] + t0) * C.w[1] + lo[1] + t1) * C.w[2] + lo[2] + t2;
                amx = fmax(amx, C.alpha[x] / eps + C.lmu[x]);
            }
            double Ak = bmax<T>(amx, sh.red);
            if (!isfinite(Ak)) Ak = 0.0;
            if (threadIdx.x < 48) s_ma[threadIdx.x / 16][threadIdx.x % 16] = 0.0;
            __syncthreads();
            for (int t = threadIdx.x; t < nbk; t += T) {
                int t0, t1, t2;
                unflat(t, be[1], be[2], t0, t1, t2);
                const int64_t x = ((int64_t)(lo[0] + t0) * C.w[1] + lo[1] + t1) * C.w[2] + lo[2] + t2;
                const double ae = C.alpha[x] / eps;
                const double u = exp(ae + C.lmu[x] - Ak);
                U[t] = u;
                UA[t] = u * ae;
            }
            if (threadIdx.x < be[0] + be[1] + be[2]) {
                // marginals of mu over the other two block axes (sequential, fixed order)
                const int a = threadIdx.x < be[0] ? 0 : (threadIdx.x < be[0] + be[1] ? 1 : 2);
                const int i = threadIdx.x - (a == 0 ? 0 : (a == 1 ? be[0] : be[0] + be[1]));
                double m = 0.0;
                for (int t0 = 0; t0 < be[0]; ++t0)
                    for (int t1 = 0; t1 < be[1]; ++t1)
                        for (int t2 = 0; t2 < be[2]; ++t2) {
                            if ((a == 0 ? t0 : (a == 1 ? t1 : t2)) != i) continue;
                            m += C.mu[((int64_t)(lo[0] + t0) * C.w[1] + lo[1] + t1) * C.w[2] + lo[2] + t2];
                        }
                s_ma[a][i] = m;
            }
            __syncthreads();
            // stage 1 (x2 -> y2): plain weights, alpha-weighted, d2^2-weighted
            const double* k2 = C.kn[2] + (int64_t)lo[2] * C.n[2];
            const double* k1 = C.kn[1] + (int64_t)lo[1] * C.n[1];
            const double* k0 = C.kn[0] + (int64_t)lo[0] * C.n[0];
            cstage<T>(U, be[0] * be[1], be[2], 1, C.n[2], k2, C.n[2], 1, T1);
            cstage<T>(UA, be[0] * be[1], be[2], 1, C.n[2], k2, C.n[2], 1, T1a);
            cstage_sq<T>(U, be[0] * be[1], be[2], 1, C.n[2], k2, C.n[2], C, g, 2, lo[2], false, T1c);
            const int ob = C.n[1] * C.n[2];
            const int n0 = C.n[0];
            // pass A: S = sum p-weights, cost part along axis 0
            cstage<T>(T1, be[0], be[1], C.n[2], C.n[1], k1, C.n[1], 1, T2);
            {
                Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
                for (int t = threadIdx.x; t < (int)C.ny; t += T, p.next()) {
                    const double* s2 = T2 + (p.i1 * C.n[2] + p.i2);
                    const double yc = coord(g.y_org, g.y_dx, 0, C.yb.o[0] + p.i0);
                    double S = 0.0, Cc = 0.0;
                    for (int q = 0; q < be[0]; ++q) {
                        const double kv = k0[(int64_t)q * n0 + p.i0];
                        const double d = coord(g.x_org, g.x_dx, 0, C.xb.o[0] + lo[0] + q) - yc;
                        S = fma(s2[q * ob], kv, S);
                        Cc = fma(s2[q * ob] * (d * d), kv, Cc);
                    }
                    R[(int64_t)k * C.ny + t] = S;
                    TC[(int64_t)k * C.ny + t] = Cc;
                }
            }
            __syncthreads();
            // pass B: alpha-weighted sum
            cstage<T>(T1a, be[0], be[1], C.n[2], C.n[1], k1, C.n[1], 1, T2);
            {
                Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
                for (int t = threadIdx.x; t < (int)C.ny; t += T, p.next()) {
                    const double* s2 = T2 + (p.i1 * C.n[2] + p.i2);
                    double Sa = 0.0;
                    for (int q = 0; q < be[0]; ++q) Sa = fma(s2[q * ob], k0[(int64_t)q * n0 + p.i0], Sa);
                    TL[(int64_t)k * C.ny + t] = Sa;
                }
            }
            __syncthreads();
            // pass C: cost parts along axes 2 and 1, then the per-node results
            cstage<T>(T1c, be[0], be[1], C.n[2], C.n[1], k1, C.n[1], 1, T2);
            cstage_sq<T>(T1, be[0], be[1], C.n[2], C.n[1], k1, C.n[1], C, g, 1, lo[1], true, T2);
            {
                Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
                for (int t = threadIdx.x; t < (int)C.ny; t += T, p.next()) {
                    const double* s2 = T2 + (p.i1 * C.n[2] + p.i2);
                    double Cc = 0.0;
                    for (int q = 0; q < be[0]; ++q) Cc = fma(s2[q * ob], k0[(int64_t)q * n0 + p.i0], Cc);
                    const int64_t q = (int64_t)k * C.ny + t;
                    const double S = R[q];
                    if (!(S >= kTiny)) {
                        split_exact(k, t);
                        continue;
                    }
                    const double bt = C.beta[t] / eps;
                    const double lsp = bt + C.lnu[t] + (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]) +
                                       Ak + log(S);
                    const double sp = exp(lsp);
                    const double mc = (TC[q] + Cc) / S;     // plan-weighted mean cost
                    const double ma = TL[q] / S;            // plan-weighted mean alpha/eps
                    R[q] = sp;
                    V[q] = sp;
                    TC[q] = sp * mc;
                    TL[q] = sp * (ma + bt - mc / eps);
                    // sum_x cost mu[x] = sum_a sum_i marg_a[i] d_a(i, y_a)^2
                    double smc = 0.0;
                    for (int a = 0; a < 3; ++a) {
                        const int ya = a == 0 ? p.i0 : (a == 1 ? p.i1 : p.i2);
                        const double yc = coord(g.y_org, g.y_dx, a, C.yb.o[a] + ya);
                        for (int i = 0; i < be[a]; ++i) {
                            const double d = coord(g.x_org, g.x_dx, a, C.xb.o[a] + lo[a] + i) - yc;
                            smc = fma(s_ma[a][i], d * d, smc);
                        }
                    }
                    MC[q] = smc;
                }
            }
            __syncthreads();
        }
    }
    // ---- balancing (cells.py:446-480): member reference masses and targets
    __shared__ double s_mbar[64], s_mass[64], s_tgt[64], s_sur[64];
    __shared__ int s_fb, s_moved;
    __shared__ double stage_sh[T], pub_sh[4];
    for (int k = 0; k < n_mem; ++k) {
        const int* lo = mlo + 3 * k;
        const int* be = mbe + 3 * k;
        const int nb = be[0] * be[1] * be[2];
        double p = 0.0;
        for (int t = threadIdx.x; t < nb; t += T) {
            int t0, t1, t2;
            unflat(t, be[1], be[2], t0, t1, t2);
            p += C.av[((int64_t)(lo[0] + t0) * C.w[1] + lo[1] + t1) * C.w[2] + lo[2] + t2];
        }
        const double mbar = bsum<T>(p, sh.red);
        double q = 0.0;
        for (int64_t y = threadIdx.x; y < C.ny; y += T) q += V[(int64_t)k * C.ny + y];
        const double mk = bsum<T>(q, sh.red);
        if (threadIdx.x == 0) { s_mbar[k] = mbar; s_mass[k] = mk; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0, nu_j = 0.0;
        for (int k = 0; k < n_mem; ++k) { total += s_mbar[k]; nu_j += s_mass[k]; }
        int nd = 0, nr = 0;
        for (int k = 0; k < n_mem; ++k) {
            s_tgt[k] = s_mbar[k] * (nu_j / total);
            s_sur[k] = s_mass[k] - s_tgt[k];
            const double tol = 1e-13 * fmax(s_tgt[k], 1e-300);
            if (s_sur[k] > tol) ++nd;
            if (s_sur[k] < -tol) ++nr;
        }
        s_moved = (nd > 0 && nr > 0) ? 1 : 0;
        s_fb = 0;
    }
    __syncthreads();
    const bool moved = s_moved != 0;
    if (moved) {
        // column sums before (sequential over members) into z
        for (int64_t y = threadIdx.x; y < C.ny; y += T) {
            double cs = V[y];
            for (int k = 1; k < n_mem; ++k) cs = __dadd_rn(cs, V[(int64_t)k * C.ny + y]);
            C.z[y] = cs;
        }
        __syncthreads();
        {
            // donor / recipient walk (cells.py:446-480): every thread follows the same
            // control flow from the shared surplus table; each move runs across the block
            int donors[64], recips[64];
            int nd = 0, nr = 0;
            for (int k = 0; k < n_mem; ++k) {
                const double tol = 1e-13 * fmax(s_tgt[k], 1e-300);
                if (s_sur[k] > tol) donors[nd++] = k;
                if (s_sur[k] < -tol) recips[nr++] = k;
            }
            int di = 0, ri = 0, fb = 0;
            while (di < nd && ri < nr) {
                const int dk = donors[di], rk = recips[ri];
                const double amount = fmin(s_sur[dk], -s_sur[rk]);
                if (amount > 0)
                    fb += dd::move_mass_block<T>(V + (int64_t)dk * C.ny, V + (int64_t)rk * C.ny,
                                                 C.ny, amount, stage_sh, pub_sh);
                const double sd = s_sur[dk] - amount, sr = s_sur[rk] + amount;
                __syncthreads();
                if (threadIdx.x == 0) { s_sur[dk] = sd; s_sur[rk] = sr; }
                __syncthreads();
                if (sd <= 1e-13 * fmax(s_tgt[dk], 1e-300)) ++di;
                if (sr >= -1e-13 * fmax(s_tgt[rk], 1e-300)) ++ri;
            }
            if (threadIdx.x == 0) s_fb = fb;
        }
        __syncthreads();
        // clip, then restore every column's sum bitwise (cells.py:505-545)
        for (int64_t t = threadIdx.x; t < (int64_t)n_mem * C.ny; t += T) V[t] = fmax(V[t], 0.0);
        __syncthreads();
    }
    int drift = 0;
    if (moved) {
        for (int64_t y = threadIdx.x; y < C.ny; y += T) {
            const double target = C.z[y];
            double* col = V + y;
            const int64_t st = C.ny;
            double seq = col[0];
            for (int k = 1; k < n_mem; ++k) seq = __dadd_rn(seq, col[k * st]);
            if (seq == target) continue;   // vals.sum(axis=0) is sequential over members
            // entries in descending order (stable sort reversed)
            int order[64];
            for (int k = 0; k < n_mem; ++k) order[k] = k;
            for (int a = 1; a < n_mem; ++a) {
                const int v = order[a];
                int q = a - 1;
                while (q >= 0 && col[order[q] * st] > col[v * st]) { order[q + 1] = order[q]; --q; }
                order[q + 1] = v;
            }
            bool ok = false;
            for (int oi = n_mem - 1; oi >= 0 && !ok; --oi) {
                const int t = order[oi];
                const double x0 = col[t * st];
                double x = x0;
                for (int it = 0; it < 256; ++it) {
                    const double sm = np_sum(col, st, n_mem);
                    if (sm == target) { ok = true; break; }
                    x = nextafter(x, sm < target ? kInf : kNegInf);
                    if (x < 0) break;
                    col[t * st] = x;
                }
                if (!ok) {
                    col[t * st] = x0;
                    ok = np_sum(col, st, n_mem) == target;
                }
            }
            if (!ok) ++drift;
        }
    }
    const int drift_nodes = (int)bsum<T>((double)drift, sh.red);
    // balance_target_miss
    double miss = 0.0;
    for (int k = 0; k < n_mem; ++k) {
        double q = 0.0;
        for (int64_t y = threadIdx.x; y < C.ny; y += T) q += V[(int64_t)k * C.ny + y];
        const double mk = bsum<T>(q, sh.red);
        miss = fmax(miss, fabs(mk - s_tgt[k]) / fmax(s_tgt[k], 1e-300));
    }
    // ---- finalize (cells.py:396-443): truncate, fragments, x-marginals
    double trunc_total = 0.0;
    for (int k = 0; k < n_mem; ++k) {
        const int i = b.members[mb + k];
        const double mass_i = s.basic_mass[i];
        double* Rk = R + (int64_t)k * C.ny;
        double* Vk = V + (int64_t)k * C.ny;
        double rem = 0.0, s_ftc = 0.0, s_emc = 0.0, s_ftl = 0.0, s_xl = 0.0, s_fin = 0.0,
               s_ext = 0.0;
        int lo0 = INT_MAX, lo1 = INT_MAX, lo2 = INT_MAX, hi0 = -1, hi1 = -1, hi2 = -1;
        for (int64_t y = threadIdx.x; y < C.ny; y += T) {
            int y0, y1, y2;
            unflat(y, C.n[1], C.n[2], y0, y1, y2);
            const double v = Vk[y];
            const bool keep = v >= b.trunc;
            double fin = 0.0;
            if (keep) {
                fin = v;
                lo0 = min(lo0, y0); hi0 = max(hi0, y0);
                lo1 = min(lo1, y1); hi1 = max(hi1, y1);
                lo2 = min(lo2, y2); hi2 = max(hi2, y2);
            } else {
                rem += v;
            }
            const double r = Rk[y];
            const bool pos = r > 0;
            const double f = pos ? fin / r : 0.0;
            const double extra = pos ? 0.0 : fin;
            s_ftc += f * TC[(int64_t)k * C.ny + y];
            s_emc += extra * MC[(int64_t)k * C.ny + y];
            s_ftl += f * TL[(int64_t)k * C.ny + y];
            if (pos) s_xl += dd::xlogy(fin, f);
            if (extra != 0.0) {
                int r0 = C.yb.o[0] + y0, r1 = C.yb.o[1] + y1, r2 = C.yb.o[2] + y2;
                const double nu = s.nu[((int64_t)r0 * g.ny[1] + r1) * g.ny[2] + r2];
                s_xl += dd::xlogy(extra, extra / (mass_i * nu));
            }
            s_fin += fin;
            s_ext += extra;
            Vk[y] = fin;
            Rk[y] = f;
        }
        rem = bsum<T>(rem, sh.red);
        s_ftc = bsum<T>(s_ftc, sh.red);
        s_emc = bsum<T>(s_emc, sh.red);
        s_ftl = bsum<T>(s_ftl, sh.red);
        s_xl = bsum<T>(s_xl, sh.red);
        s_fin = bsum<T>(s_fin, sh.red);
        s_ext = bsum<T>(s_ext, sh.red);
        lo0 = bmin_i<T>(lo0, sh.redi); lo1 = bmin_i<T>(lo1, sh.redi); lo2 = bmin_i<T>(lo2, sh.redi);
        hi0 = bmax_i<T>(hi0, sh.redi); hi1 = bmax_i<T>(hi1, sh.redi); hi2 = bmax_i<T>(hi2, sh.redi);
        trunc_total += rem;
        if (threadIdx.x == 0) {
            int32_t* nb = b.mbox + (int64_t)(mb + k) * 6;
            if (hi0 >= 0) {
                nb[0] = C.yb.o[0] + lo0; nb[1] = hi0 - lo0 + 1;
                nb[2] = C.yb.o[1] + lo1; nb[3] = hi1 - lo1 + 1;
                nb[4] = C.yb.o[2] + lo2; nb[5] = hi2 - lo2 + 1;
            } else {
                for (int q = 0; q < 6; ++q) nb[q] = 0;
            }
            double* ms4 = b.mstat + (int64_t)(mb + k) * 4;
            ms4[0] = s_ftc + s_emc / mass_i;
            ms4[1] = s_ftl + s_xl - s_fin + mass_i * g.nu_total;
            ms4[2] = rem;
            ms4[3] = 0.0;
        }
        // x-marginal: xm[x] = sum_y plan[x,y] f[y] (+ mu[x] extra_sum / mass_i)
        const int* lo = mlo + 3 * k;
        const int* be = mbe + 3 * k;
        const int nbk = be[0] * be[1] * be[2];
        __shared__ double part_sum[T];
        bool xdone = false;
        if (sep && nbk <= T) {
            // separable form: weights v[y] = f[y] exp(b[y] + sum_a c_a(y_a) - B) (B their
            // maximum shift) contracted along axis 2, 1, 0 against the Y-normalised tables
            // restricted to the member's block; xm[x] = exp(a[x] + B + log S[x]).  A block
            // node whose sum is below kTiny (or overflowed) sends the member to the
            // per-term path below.
            double bmx = kNegInf;
            {
                Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
                for (int y = threadIdx.x; y < (int)C.ny; y += T, p.next()) {
                    if (Rk[y] > 0)
                        bmx = fmax(bmx, C.beta[y] / eps + C.lnu[y] +
                                            (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]));
                }
            }
            double Bk = bmax<T>(bmx, sh.red);
            const bool anyf = isfinite(Bk);   // false: every f is 0, the member keeps nothing
            if (!anyf) Bk = 0.0;
            {
                Step3<T> p(threadIdx.x, C.n[1], C.n[2]);
                for (int y = threadIdx.x; y < (int)C.ny; y += T, p.next()) {
                    const double f = Rk[y];
                    C.z[y] = f > 0 ? f * exp(C.beta[y] / eps + C.lnu[y] +
                                             (C.c[0][p.i0] + C.c[1][p.i1] + C.c[2][p.i2]) - Bk)
                                   : 0.0;
                }
            }
            if (threadIdx.x == 0) sh.flag = 0;
            __syncthreads();
            cstage<T>(C.z, C.n[0] * C.n[1], C.n[2], 1, be[2], C.kn[2] + (int64_t)lo[2] * C.n[2], 1,
                      C.n[2], C.s1);
            cstage<T>(C.s1, C.n[0], C.n[1], be[2], be[1], C.kn[1] + (int64_t)lo[1] * C.n[1], 1,
                      C.n[1], C.s2);
            {
                const int obx = be[1] * be[2];
                const int n0 = C.n[0];
                int bad = 0;
                for (int t = threadIdx.x; t < nbk; t += T) {
                    int t0, t1, t2;
                    unflat(t, be[1], be[2], t0, t1, t2);
                    const int64_t xx = ((int64_t)(lo[0] + t0) * C.w[1] + lo[1] + t1) * C.w[2] + lo[2] + t2;
                    const double* s2 = C.s2 + (t1 * be[2] + t2);
                    const double* kt = C.kn[0] + (int64_t)(lo[0] + t0) * n0;
                    double S = 0.0;
                    for (int q = 0; q < n0; ++q) S = fma(s2[q * obx], kt[q], S);
                    double xm = 0.0;
                    if (C.mu[xx] > 0) {
                        if (!anyf) xm = 0.0;
                        else if (!(S >= kTiny) || !(S < kInf)) bad = 1;
                        else xm = exp(C.alpha[xx] / eps + C.lmu[xx] + Bk + log(S));
                    }
                    part_sum[t] = xm;
                }
                if (bad) sh.flag = 1;
            }
            __syncthreads();
            if (!sh.flag) {
                for (int t = threadIdx.x; t < nbk; t += T) {
                    int t0, t1, t2;
                    unflat(t, be[1], be[2], t0, t1, t2);
                    const int64_t xx = ((int64_t)(lo[0] + t0) * C.w[1] + lo[1] + t1) * C.w[2] + lo[2] + t2;
                    double xm = part_sum[t];
                    if (s_ext != 0.0) xm = xm + C.mu[xx] * (s_ext / mass_i);
                    b.xarena[xoff + (int64_t)k * bs + t] = C.mu[xx] > 0 ? xm : 0.0;
                }
                xdone = true;
            }
            __syncthreads();
        }
        if (!xdone) {
            const int P = max(1, T / max(nbk, 1));
            const int rowi = threadIdx.x / P, part = threadIdx.x - rowi * P;
            double acc = 0.0;
            int64_t xw = -1;
            if (rowi < nbk) {
                int t0, t1, t2;
                unflat(rowi, be[1], be[2], t0, t1, t2);
                const int x0 = lo[0] + t0, x1 = lo[1] + t1, x2 = lo[2] + t2;
                xw = ((int64_t)x0 * C.w[1] + x1) * C.w[2] + x2;
                if (C.mu[xw] > 0) {
                    const double av = C.alpha[xw] / eps;
                    for (int64_t y = part; y < C.ny; y += P) {
                        const double f = Rk[y];
                        if (f == 0.0) continue;
                        int y0, y1, y2;
                        unflat(y, C.n[1], C.n[2], y0, y1, y2);
                        const double cost = cell_cost(C, g, x0, x1, x2, y0, y1, y2);
                        const double sc = av + C.beta[y] / eps + (-cost / eps);
                        acc += exp(sc + C.lmu[xw] + C.lnu[y]) * f;
                    }
                }
            }
            // rows beyond T are handled below, one thread per row
            __syncthreads();
            part_sum[threadIdx.x] = acc;
            __syncthreads();
            if (part == 0 && rowi < nbk) {
                double xm = 0.0;
                for (int q = 0; q < P; ++q) xm += part_sum[threadIdx.x + q];
                if (s_ext != 0.0) xm = xm + C.mu[xw] * (s_ext / mass_i);
                b.xarena[xoff + (int64_t)k * bs + rowi] = C.mu[xw] > 0 ? xm : 0.0;
            }
            for (int rr = T; rr < nbk; rr += T) {   // blocks above T nodes: one thread per row
                const int row = rr + threadIdx.x;
                if (row < nbk) {
                    int t0, t1, t2;
                    unflat(row, be[1], be[2], t0, t1, t2);
                    const int x0 = lo[0] + t0, x1 = lo[1] + t1, x2 = lo[2] + t2;
                    const int64_t xx = ((int64_t)x0 * C.w[1] + x1) * C.w[2] + x2;
                    double xm = 0.0;
                    if (C.mu[xx] > 0) {
                        for (int64_t y = 0; y < C.ny; ++y) {
                            const double f = Rk[y];
                            if (f == 0.0) continue;
                            int y0, y1, y2;
                            unflat(y, C.n[1], C.n[2], y0, y1, y2);
                            const double cost = cell_cost(C, g, x0, x1, x2, y0, y1, y2);
                            const double sc = C.alpha[xx] / eps + C.beta[y] / eps + (-cost / eps);
                            xm += exp(sc + C.lmu[xx] + C.lnu[y]) * f;
                        }
                        if (s_ext != 0.0) xm = xm + C.mu[xx] * (s_ext / mass_i);
                    }
                    b.xarena[xoff + (int64_t)k * bs + row] = xm;
                }
            }
        }
        __syncthreads();
    }
    // outputs: duals, per-cell statistics
    for (int64_t x = threadIdx.x; x < C.nx; x += T) b.alpha[(int64_t)c * C.nx + x] = C.alpha[x];
    for (int64_t y = threadIdx.x; y < C.ny; y += T) b.beta[yoff + y] = C.beta[y];
    if (threadIdx.x == 0) {
        cst[0] = gap; cst[1] = first_g; cst[2] = iters; cst[3] = conv ? 1.0 : 0.0;
        cst[4] = nclamped; cst[5] = ndeg_max; cst[6] = s_fb; cst[7] = miss;
        cst2[0] = drift_nodes; cst2[1] = trunc_total; cst2[2] = iters; cst2[3] = nfb;
        cst2[4] = nsteps_all; cst2[5] = (double)t_loop; cst2[6] = 0; cst2[7] = 0;
    }
}

// ---- blend pieces (engine.py:388-433) ------------------------------------------------

__device__ __forceinline__ double block_kl(const dd3_geom& g, const dd3_state& s, int i,
                                           const double* x, double th, const double* xo,
                                           int mode) {
    // sum over the basic block of kl_term(value, mu); mode 0: value = x; mode 1:
    // (1 - th) xo + th x
    const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
    const int nb = bx.e[0] * bx.e[1] * bx.e[2];
    double p = 0.0;
    for (int t = threadIdx.x; t < nb; t += NT) {
        int t0, t1, t2;
        unflat(t, bx.e[1], bx.e[2], t0, t1, t2);
        const double mu = s.mu[((int64_t)(bx.o[0] + t0) * g.nx[1] + bx.o[1] + t1) * g.nx[2] +
                               bx.o[2] + t2];
        if (!(mu > 0)) continue;
        const double v = mode == 0 ? x[t] : (1.0 - th) * xo[t] + th * x[t];
        p += dd::kl_term(v, mu);
    }
    return p;
}

__global__ void __launch_bounds__(NT) cell_delta3_kernel(dd3_geom g, dd3_state s, dd3_batch b,
                                                         double th_safe, double* dy, double* cd) {
    __shared__ double red[NW];
    __shared__ int32_t sobox[64 * 6];
    const int c = blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 16;
    const B3 yb = ldbox(d + 7);
    const int n_mem = d[13], mb = d[14];
    const int64_t ny = bsize(yb);
    const int64_t yoff = b.offs[(int64_t)c * 4 + 0], moff = b.offs[(int64_t)c * 4 + 1];
    const int64_t xoff = b.offs[(int64_t)c * 4 + 3];
    const double* V = b.marena + moff + (int64_t)n_mem * ny;
    const int bs = s.block[0] * s.block[1] * s.block[2];
    for (int k = threadIdx.x; k < n_mem; k += NT) {
        const int i = b.members[mb + k];
        for (int q = 0; q < 6; ++q) sobox[k * 6 + q] = s.ybox[(int64_t)i * 6 + q];
    }
    __syncthreads();
    for (int64_t y = threadIdx.x; y < ny; y += NT) {
        int y0, y1, y2;
        unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
        const int r0 = yb.o[0] + y0, r1 = yb.o[1] + y1, r2 = yb.o[2] + y2;
        double yo = 0.0, yn = 0.0;
        for (int k = 0; k < n_mem; ++k) {
            const int i = b.members[mb + k];
            B3 ob;
            for (int a = 0; a < 3; ++a) { ob.o[a] = sobox[k * 6 + 2 * a]; ob.e[a] = sobox[k * 6 + 2 * a + 1]; }
            yo += bempty(ob) ? 0.0 : bat(ob, s.yval + (int64_t)i * s.cap, r0, r1, r2);
            yn += V[(int64_t)k * ny + y];
        }
        dy[yoff + y] = yn - yo;
    }
    double t_old = 0.0, k_old = 0.0, t_new = 0.0, k_new = 0.0, d1o = 0.0, d1a = 0.0, d1s = 0.0;
    for (int k = 0; k < n_mem; ++k) {
        const int i = b.members[mb + k];
        const double* xo = s.x_marg + (int64_t)i * bs;
        const double* xn = b.xarena + xoff + (int64_t)k * bs;
        const double po = bsum(block_kl(g, s, i, xo, 0.0, xo, 0), red);
        const double pa = bsum(block_kl(g, s, i, xn, 0.0, xn, 0), red);
        const double ps = bsum(block_kl(g, s, i, xn, th_safe, xo, 1), red);
        d1o += po; d1a += pa; d1s += ps;
        t_old += s.transport[i];
        k_old += s.kl[i];
        t_new += b.mstat[(int64_t)(mb + k) * 4 + 0];
        k_new += b.mstat[(int64_t)(mb + k) * 4 + 1];
    }
    if (threadIdx.x == 0) {
        double* o = cd + (int64_t)c * 8;
        o[0] = t_new - t_old;
        o[1] = k_new - k_old;
        o[2] = g.lam * d1o;
        o[3] = g.lam * d1a;
        o[4] = g.lam * d1s;
        o[5] = 0.0; o[6] = 0.0; o[7] = 0.0;
    }
}

// ---- opt strategy pieces (engine.py:378-470, 473-527) ---------------------------------

// out[c] = lam * sum over cell c's members of KL((1 - theta_c) xo + theta_c xn | mu)
// (BlendScorer._d1_blend at a per-cell weight; energy_at of a general theta vector)
__global__ void __launch_bounds__(NT) blend_d1_3_kernel(dd3_geom g, dd3_state s, dd3_batch b,
                                                        const double* theta, double* out) {
    __shared__ double red[NW];
    const int c = blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 16;
    const int n_mem = d[13], mb = d[14];
    const int64_t xoff = b.offs[(int64_t)c * 4 + 3];
    const int bs = s.block[0] * s.block[1] * s.block[2];
    const double th = theta[c];
    double tot = 0.0;
    for (int k = 0; k < n_mem; ++k) {
        const int i = b.members[mb + k];
        const double* xo = s.x_marg + (int64_t)i * bs;
        const double* xn = b.xarena + xoff + (int64_t)k * bs;
        tot += bsum(block_kl(g, s, i, xn, th, xo, 1), red);
    }
    if (threadIdx.x == 0) out[c] = g.lam * tot;
}

// Derivative pieces of the blend objective in cell c's weight (coordinate descent):
// out[0] = sum d log(x/mu), out[1] = sum d^2/x over the members' X blocks, d = xn - xo,
// x = (1-th) xo + th xn; out[2] = sum dy log(y/nu), out[3] = sum dy^2/y over the cell's
// Y window, y = clip(clip(ycur - th_cur dy, 0) + th dy, 0).  Entries with a zero update
// direction are skipped (the reference's np.where(d == 0, 0, ...)).  All lam-free.
__global__ void __launch_bounds__(NT) opt_gh3_kernel(dd3_geom g, dd3_state s, dd3_batch b,
                                                     const double* dy, int c, double th,
                                                     double th_cur, const double* ycur,
                                                     double* out) {
    __shared__ double red[NW];
    const int32_t* d = b.desc + (int64_t)c * 16;
    const B3 yb = ldbox(d + 7);
    const int n_mem = d[13], mb = d[14];
    const int64_t ny = bsize(yb);
    const int64_t yoff = b.offs[(int64_t)c * 4 + 0], xoff = b.offs[(int64_t)c * 4 + 3];
    const int bs = s.block[0] * s.block[1] * s.block[2];
    double gx = 0.0, hx = 0.0;
    for (int k = 0; k < n_mem; ++k) {
        const int i = b.members[mb + k];
        const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
        const int nb = bx.e[0] * bx.e[1] * bx.e[2];
        const double* xo = s.x_marg + (int64_t)i * bs;
        const double* xn = b.xarena + xoff + (int64_t)k * bs;
        for (int t = threadIdx.x; t < nb; t += NT) {
            int t0, t1, t2;
            unflat(t, bx.e[1], bx.e[2], t0, t1, t2);
            const double mu = s.mu[((int64_t)(bx.o[0] + t0) * g.nx[1] + bx.o[1] + t1) * g.nx[2] +
                                   bx.o[2] + t2];
            if (!(mu > 0)) continue;
            const double dd = xn[t] - xo[t];
            if (dd == 0.0) continue;
            const double x = (1.0 - th) * xo[t] + th * xn[t];
            gx += dd * log(x / mu);
            hx += dd * dd / x;
        }
    }
    double gy = 0.0, hy = 0.0;
    for (int64_t y = threadIdx.x; y < ny; y += NT) {
        const double dv = dy[yoff + y];
        if (dv == 0.0) continue;
        int y0, y1, y2;
        unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
        const int64_t id = ((int64_t)(yb.o[0] + y0) * g.ny[1] + yb.o[1] + y1) * g.ny[2] +
                           yb.o[2] + y2;
        const double ybv = fmax(ycur[id] - th_cur * dv, 0.0);
        const double yv = fmax(ybv + th * dv, 0.0);
        gy += dv * log(yv / s.nu[id]);
        hy += dv * dv / yv;
    }
    gx = bsum(gx, red);
    hx = bsum(hx, red);
    gy = bsum(gy, red);
    hy = bsum(hy, red);
    if (threadIdx.x == 0) { out[0] = gx; out[1] = hx; out[2] = gy; out[3] = hy; }
}

// ycur[window of cell c] = clip(ycur + dth * dy, 0)   (BlendScorer.set_theta)
__global__ void __launch_bounds__(NT) opt_set3_kernel(dd3_geom g, dd3_batch b, const double* dy,
                                                      int c, double dth, double* ycur) {
    const int32_t* d = b.desc + (int64_t)c * 16;
    const B3 yb = ldbox(d + 7);
    const int64_t ny = bsize(yb);
    const int64_t yoff = b.offs[(int64_t)c * 4 + 0];
    for (int64_t y = threadIdx.x; y < ny; y += NT) {
        int y0, y1, y2;
        unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
        const int64_t id = ((int64_t)(yb.o[0] + y0) * g.ny[1] + yb.o[1] + y1) * g.ny[2] +
                           yb.o[2] + y2;
        ycur[id] = fmax(ycur[id] + dth * dy[yoff + y], 0.0);
    }
}

// ---- commit (engine.py:726-785) ------------------------------------------------------

__global__ void __launch_bounds__(NT) cell_commit3_kernel(dd3_geom g, dd3_state s, dd3_batch b,
                                                          const double* theta, double* alpha_grid,
                                                          double* yrun, double* errs) {
    __shared__ double red[NW];
    __shared__ int redi[NW];
    __shared__ int32_t sobox[64 * 6];
    const int c = blockIdx.x;
    const int32_t* d = b.desc + (int64_t)c * 16;
    const int j = d[0];
    const B3 xb = ldbox(d + 1);
    const B3 yb = ldbox(d + 7);
    const int n_mem = d[13], mb = d[14];
    const int w1 = b.nxw[1], w2 = b.nxw[2];
    const int64_t nx = (int64_t)b.nxw[0] * w1 * w2;
    const int64_t ny = bsize(yb);
    const int64_t yoff = b.offs[(int64_t)c * 4 + 0], moff = b.offs[(int64_t)c * 4 + 1];
    const int64_t xoff = b.offs[(int64_t)c * 4 + 3];
    double* V = b.marena + moff + (int64_t)n_mem * ny;      // new (truncated) member values
    double* OLD = V + 3 * (int64_t)n_mem * ny;              // mc slot: old window values
    const int bs = s.block[0] * s.block[1] * s.block[2];
    const double th = theta[c];
    const double* alpha = b.alpha + (int64_t)c * nx;
    const double* beta = b.beta + yoff;
    for (int k = threadIdx.x; k < n_mem; k += NT) {
        const int i = b.members[mb + k];
        for (int q = 0; q < 6; ++q) sobox[k * 6 + q] = s.ybox[(int64_t)i * 6 + q];
    }
    __syncthreads();
    // old member windows (before any slot is rewritten)
    for (int64_t y = threadIdx.x; y < ny; y += NT) {
        int y0, y1, y2;
        unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
        const int r0 = yb.o[0] + y0, r1 = yb.o[1] + y1, r2 = yb.o[2] + y2;
        for (int k = 0; k < n_mem; ++k) {
            const int i = b.members[mb + k];
            B3 ob;
            for (int a = 0; a < 3; ++a) { ob.o[a] = sobox[k * 6 + 2 * a]; ob.e[a] = sobox[k * 6 + 2 * a + 1]; }
            OLD[(int64_t)k * ny + y] = bempty(ob) ? 0.0 : bat(ob, s.yval + (int64_t)i * s.cap, r0, r1, r2);
        }
    }
    __syncthreads();
    double added = 0.0;
    if (th > 0.0) {
        double sol_trunc = 0.0;
        for (int k = 0; k < n_mem; ++k) sol_trunc += b.mstat[(int64_t)(mb + k) * 4 + 2];
        added = th >= 1.0 ? sol_trunc : th * sol_trunc;
        for (int k = 0; k < n_mem; ++k) {
            const int i = b.members[mb + k];
            double* Vk = V + (int64_t)k * ny;
            const double* Ok = OLD + (int64_t)k * ny;
            B3 nb;
            if (th >= 1.0) {
                nb = ldbox(b.mbox + (int64_t)(mb + k) * 6);
            } else {
                // blend on the cell window, re-truncate (engine.py:752-758)
                int lo0 = INT_MAX, lo1 = INT_MAX, lo2 = INT_MAX, hi0 = -1, hi1 = -1, hi2 = -1;
                double rem = 0.0;
                for (int64_t y = threadIdx.x; y < ny; y += NT) {
                    int y0, y1, y2;
                    unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
                    const double bw = (1.0 - th) * Ok[y] + th * Vk[y];
                    if (bw >= b.trunc) {
                        lo0 = min(lo0, y0); hi0 = max(hi0, y0);
                        lo1 = min(lo1, y1); hi1 = max(hi1, y1);
                        lo2 = min(lo2, y2); hi2 = max(hi2, y2);
                        Vk[y] = bw;
                    } else {
                        rem += bw;
                        Vk[y] = 0.0;
                    }
                }
                const double removed = bsum(rem, red);
                lo0 = bmin_i(lo0, redi); lo1 = bmin_i(lo1, redi); lo2 = bmin_i(lo2, redi);
                hi0 = bmax_i(hi0, redi); hi1 = bmax_i(hi1, redi); hi2 = bmax_i(hi2, redi);
                if (hi0 >= 0) {
                    nb.o[0] = yb.o[0] + lo0; nb.e[0] = hi0 - lo0 + 1;
                    nb.o[1] = yb.o[1] + lo1; nb.e[1] = hi1 - lo1 + 1;
                    nb.o[2] = yb.o[2] + lo2; nb.e[2] = hi2 - lo2 + 1;
                } else {
                    for (int a = 0; a < 3; ++a) { nb.o[a] = 0; nb.e[a] = 0; }
                }
                added += removed;
            }
            // write the slot: compact values of the new box (all inside the window)
            const int64_t nn = bsize(nb);
            double* slot = s.yval + (int64_t)i * s.cap;
            for (int64_t t = threadIdx.x; t < nn; t += NT) {
                int a0, a1, a2;
                unflat(t, nb.e[1], nb.e[2], a0, a1, a2);
                const int64_t y = ((int64_t)(nb.o[0] + a0 - yb.o[0]) * yb.e[1] +
                                   (nb.o[1] + a1 - yb.o[1])) * yb.e[2] + (nb.o[2] + a2 - yb.o[2]);
                slot[t] = Vk[y];
            }
            const double* xn = b.xarena + xoff + (int64_t)k * bs;
            double* xs = s.x_marg + (int64_t)i * bs;
            for (int t = threadIdx.x; t < bs; t += NT)
                xs[t] = th >= 1.0 ? xn[t] : (1.0 - th) * xs[t] + th * xn[t];
            if (threadIdx.x == 0) {
                for (int a = 0; a < 3; ++a) {
                    s.ybox[(int64_t)i * 6 + 2 * a] = bempty(nb) ? 0 : nb.o[a];
                    s.ybox[(int64_t)i * 6 + 2 * a + 1] = bempty(nb) ? 0 : nb.e[a];
                }
                const double* ms4 = b.mstat + (int64_t)(mb + k) * 4;
                if (th >= 1.0) {
                    s.transport[i] = ms4[0];
                    s.kl[i] = ms4[1];
                } else {
                    s.transport[i] = (1.0 - th) * s.transport[i] + th * ms4[0];
                    s.kl[i] = (1.0 - th) * s.kl[i] + th * ms4[1];
                }
            }
            __syncthreads();
        }
    }
    // residuals against the solution's duals
    double yerr = 0.0;
    for (int64_t y = threadIdx.x; y < ny; y += NT) {
        int y0, y1, y2;
        unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
        const int64_t id = ((int64_t)(yb.o[0] + y0) * g.ny[1] + yb.o[1] + y1) * g.ny[2] + yb.o[2] + y2;
        const double nu = s.nu[id];
        double yn = 0.0, yo = 0.0;
        for (int k = 0; k < n_mem; ++k) {
            yn += th > 0.0 ? V[(int64_t)k * ny + y] : OLD[(int64_t)k * ny + y];
            yo += OLD[(int64_t)k * ny + y];
        }
        const double num = b.mdens[yoff + y] * nu;
        yerr += fabs(yn + num - exp(-beta[y] / g.lam) * nu);
        // sequential mode: running Y-marginal += new window - old window, clipped at 0
        // (engine.py:829-830)
        if (yrun) yrun[id] = fmax(yrun[id] + (yn - yo), 0.0);
    }
    double xerr = 0.0;
    for (int k = 0; k < n_mem; ++k) {
        const int i = b.members[mb + k];
        const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
        const double* xs = s.x_marg + (int64_t)i * bs;
        for (int t = threadIdx.x; t < bs; t += NT) {
            int t0, t1, t2;
            unflat(t, bx.e[1], bx.e[2], t0, t1, t2);
            const int r0 = bx.o[0] + t0, r1 = bx.o[1] + t1, r2 = bx.o[2] + t2;
            const int64_t gid = ((int64_t)r0 * g.nx[1] + r1) * g.nx[2] + r2;
            const int64_t xw = ((int64_t)(r0 - xb.o[0]) * w1 + (r1 - xb.o[1])) * w2 + (r2 - xb.o[2]);
            const double mu = s.mu[gid];
            if (mu > 0) xerr += fabs(xs[t] - exp(-alpha[xw] / g.lam) * mu);
            if (alpha_grid) alpha_grid[gid] = alpha[xw];
        }
    }
    // dual store
    for (int64_t x = threadIdx.x; x < nx; x += NT) s.d_alpha[(int64_t)j * nx + x] = alpha[x];
    for (int64_t y = threadIdx.x; y < ny; y += NT) s.d_beta[(int64_t)j * s.d_cap + y] = beta[y];
    if (threadIdx.x < 6) s.d_box[(int64_t)j * 6 + threadIdx.x] = d[7 + threadIdx.x];
    if (threadIdx.x == 0) s.d_has[j] = 1;
    yerr = bsum(yerr, red);
    xerr = bsum(xerr, red);
    if (threadIdx.x == 0) {
        errs[(int64_t)c * 4 + 0] = xerr;
        errs[(int64_t)c * 4 + 1] = yerr;
        errs[(int64_t)c * 4 + 2] = added;
        errs[(int64_t)c * 4 + 3] = 0.0;
    }
}

// ---- fixed-order boxed gather (measures.py:410-425) ------------------------------

struct GItems {
    int n;
    const int32_t* box;
    int bstride;
    const double* vals;
    int64_t vstride;
    const int64_t* voff;
    const double* scale;
};

// one CTA per tile (T0 x T1 x T2 nodes, one per thread); the items whose boxes meet
// the tile are compacted in index order, chunk by chunk, and every node accumulates
// them in that order (no atomics: bitwise reproducible)
__global__ void __launch_bounds__(NT) gather3_kernel(dd3_geom g, GItems it, int T0, int T1,
                                                     int T2, const double* base, double* out,
                                                     int kl_mode, const double* nu,
                                                     double* partial) {
    __shared__ int sid[NT];
    __shared__ int wcnt[NW + 1];
    __shared__ double red[NW];
    const int n0 = g.ny[0], n1 = g.ny[1], n2 = g.ny[2];
    const int tiles2 = (n2 + T2 - 1) / T2, tiles1 = (n1 + T1 - 1) / T1;
    const int tb = blockIdx.x;
    const int tz = tb / (tiles1 * tiles2), rem = tb - tz * tiles1 * tiles2;
    const int ty = rem / tiles2, tx = rem - ty * tiles2;
    const int b0 = tz * T0, b1 = ty * T1, b2 = tx * T2;
    const int e0 = min(T0, n0 - b0), e1 = min(T1, n1 - b1), e2 = min(T2, n2 - b2);
    const int l0 = threadIdx.x / (T1 * T2), lr = threadIdx.x - l0 * T1 * T2;
    const int l1 = lr / T2, l2 = lr - l1 * T2;
    const bool valid = threadIdx.x < T0 * T1 * T2 && l0 < e0 && l1 < e1 && l2 < e2;
    const int r0 = b0 + l0, r1 = b1 + l1, r2 = b2 + l2;
    const int64_t id = valid ? ((int64_t)r0 * n1 + r1) * n2 + r2 : 0;
    double acc = (valid && base) ? base[id] : 0.0;
    for (int c0 = 0; c0 < it.n; c0 += NT) {
        const int i = c0 + threadIdx.x;
        bool hit = false;
        if (i < it.n) {
            const int32_t* p = it.box + (int64_t)i * it.bstride;
            const bool live = p[1] > 0 && p[3] > 0 && p[5] > 0 && !(it.scale && it.scale[i] == 0.0);
            hit = live && p[0] < b0 + e0 && p[0] + p[1] > b0 && p[2] < b1 + e1 &&
                  p[2] + p[3] > b1 && p[4] < b2 + e2 && p[4] + p[5] > b2;
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
        if (ln == 0) wcnt[w] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            int sacc = 0;
            for (int k = 0; k < NW; ++k) { const int v = wcnt[k]; wcnt[k] = sacc; sacc += v; }
            wcnt[NW] = sacc;
        }
        __syncthreads();
        if (hit) sid[wcnt[w] + __popc(m & ((1u << ln) - 1u))] = i;
        __syncthreads();
        const int cnt = wcnt[NW];
        if (valid) {
            for (int q = 0; q < cnt; ++q) {
                const int k = sid[q];
                const int32_t* p = it.box + (int64_t)k * it.bstride;
                const int a0 = r0 - p[0], a1 = r1 - p[2], a2 = r2 - p[4];
                if (a0 < 0 || a0 >= p[1] || a1 < 0 || a1 >= p[3] || a2 < 0 || a2 >= p[5]) continue;
                const double* v = it.vals + (it.voff ? it.voff[k] : (int64_t)k * it.vstride);
                const double x = v[((int64_t)a0 * p[3] + a1) * p[5] + a2];
                acc = __dadd_rn(acc, it.scale ? __dmul_rn(it.scale[k], x) : x);
            }
        }
        __syncthreads();
    }
    if (valid && out) out[id] = acc;
    if (kl_mode) {
        double t = 0.0;
        if (valid) {
            const double y = kl_mode == 2 ? fmax(acc, 0.0) : acc;
            t = dd::kl_term(y, nu[id]);
        }
        t = bsum(t, red);
        if (threadIdx.x == 0) partial[blockIdx.x] = t;
    }
}

// ---- per basic cell energy pieces (engine.py:185-196) ------------------------------------

__global__ void __launch_bounds__(NT) cell_terms3_kernel(dd3_geom g, dd3_state s, double* out) {
    __shared__ double red[NW];
    const int i = blockIdx.x;
    const int bs = s.block[0] * s.block[1] * s.block[2];
    const double p = bsum(block_kl(g, s, i, s.x_marg + (int64_t)i * bs, 0.0, nullptr, 0), red);
    if (threadIdx.x == 0) {
        out[(int64_t)i * 4 + 0] = s.transport[i];
        out[(int64_t)i * 4 + 1] = s.kl[i];
        out[(int64_t)i * 4 + 2] = p;
        out[(int64_t)i * 4 + 3] = 0.0;
    }
}

// ---- product start (engine.py:234-257, cells.py:566-606) ------------------------------

__global__ void __launch_bounds__(NT) product_init3_kernel(dd3_geom g, dd3_state s,
                                                           double mu_total) {
    __shared__ double red[NW];
    const int i = blockIdx.x;
    const int64_t ny = (int64_t)g.ny[0] * g.ny[1] * g.ny[2];
    const double scale = s.basic_mass[i] / mu_total;
    const double ratio = g.nu_total / mu_total;
    double* v = s.yval + (int64_t)i * s.cap;
    double mnu = 0.0, ent = 0.0, sy1[3] = {0, 0, 0}, sy2[3] = {0, 0, 0};
    for (int64_t t = threadIdx.x; t < ny; t += NT) {
        int yi[3];
        unflat(t, g.ny[1], g.ny[2], yi[0], yi[1], yi[2]);
        const double nu = s.nu[t];
        const double val = nu * scale;
        v[t] = val;
        mnu += val;
        for (int a = 0; a < 3; ++a) {
            const double yc = coord(g.y_org, g.y_dx, a, yi[a]);
            sy1[a] += val * yc;
            sy2[a] += val * (yc * yc);
        }
        ent += dd::xlogy(val, val / nu);
    }
    mnu = bsum(mnu, red);
    ent = bsum(ent, red);
    for (int a = 0; a < 3; ++a) { sy1[a] = bsum(sy1[a], red); sy2[a] = bsum(sy2[a], red); }
    const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
    const int bs = s.block[0] * s.block[1] * s.block[2];
    double mmu = 0.0, sx1[3] = {0, 0, 0}, sx2[3] = {0, 0, 0};
    for (int t = threadIdx.x; t < bs; t += NT) {
        int t0, t1, t2;
        unflat(t, bx.e[1], bx.e[2], t0, t1, t2);
        const int xi[3] = {bx.o[0] + t0, bx.o[1] + t1, bx.o[2] + t2};
        const double mu = s.mu[((int64_t)xi[0] * g.nx[1] + xi[1]) * g.nx[2] + xi[2]];
        s.x_marg[(int64_t)i * bs + t] = mu > 0 ? mu * ratio : 0.0;
        if (mu > 0) {
            mmu += mu;
            for (int a = 0; a < 3; ++a) {
                const double xc = coord(g.x_org, g.x_dx, a, xi[a]);
                sx1[a] += mu * xc;
                sx2[a] += mu * (xc * xc);
            }
        }
    }
    mmu = bsum(mmu, red);
    for (int a = 0; a < 3; ++a) { sx1[a] = bsum(sx1[a], red); sx2[a] = bsum(sx2[a], red); }
    if (threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a) {
            s.ybox[(int64_t)i * 6 + 2 * a] = 0;
            s.ybox[(int64_t)i * 6 + 2 * a + 1] = g.ny[a];
        }
        if (mnu == 0.0) {
            s.transport[i] = 0.0;
            s.kl[i] = mmu * g.nu_total;
        } else {
            double tr = 0.0;
            for (int a = g.first_axis; a < 3; ++a)
                tr += sx2[a] * mnu - 2.0 * sx1[a] * sy1[a] + mmu * sy2[a];
            tr /= mmu;
            s.transport[i] = tr;
            s.kl[i] = ent - mnu * log(mmu) - mnu + mmu * g.nu_total;
        }
    }
}

// ---- plan cut (engine.py:294-322) ----------------------------------------------------

constexpr int kCutTile = 4;

// per Y tile (kCutTile^3 nodes): max of beta/eps + log nu
__global__ void cut_tiles_kernel(dd3_geom g, const double* beta, const double* log_nu,
                                 double* tmax) {
    const int t0n = (g.ny[0] + kCutTile - 1) / kCutTile, t1n = (g.ny[1] + kCutTile - 1) / kCutTile,
              t2n = (g.ny[2] + kCutTile - 1) / kCutTile;
    const int64_t nt = (int64_t)t0n * t1n * t2n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int a, bq, cq;
        unflat(t, t1n, t2n, a, bq, cq);
        double m = kNegInf;
        for (int i0 = a * kCutTile; i0 < min(g.ny[0], (a + 1) * kCutTile); ++i0)
            for (int i1 = bq * kCutTile; i1 < min(g.ny[1], (bq + 1) * kCutTile); ++i1)
                for (int i2 = cq * kCutTile; i2 < min(g.ny[2], (cq + 1) * kCutTile); ++i2) {
                    const int64_t id = ((int64_t)i0 * g.ny[1] + i1) * g.ny[2] + i2;
                    m = fmax(m, beta[id] / g.eps + log_nu[id]);
                }
        tmax[t] = m;
    }
}

__device__ __forceinline__ double gap1(double lo, double hi, double ylo, double yhi) {
    return fmax(0.0, fmax(ylo - hi, lo - yhi));   // distance between [lo,hi] and [ylo,yhi]
}

__device__ __forceinline__ double cut_col(const dd3_geom& g, const double* xs_c0,
                                          const double* xs_c1, const double* xs_c2,
                                          const double* xs_a, const double* xs_lm,
                                          const double* xs_mu, int nxn, double yc0, double yc1,
                                          double yc2, double nu, double lnu, double bt,
                                          double cut_log, double* tr, double* klp, double* xacc) {
    double col = 0.0;
    for (int k = 0; k < nxn; ++k) {
        const double d0 = xs_c0[k] - yc0, d1 = xs_c1[k] - yc1, d2 = xs_c2[k] - yc2;
        const double cost = d0 * d0 + d1 * d1 + d2 * d2;
        const double lr = (xs_a[k] + bt - cost) / g.eps;
        if (lr + xs_lm[k] + lnu < cut_log) continue;
        const double blk = exp(lr) * xs_mu[k] * nu;
        col += blk;
        if (tr) {
            *tr += cost * blk;
            *klp += blk * lr;
            xacc[k] += blk;
        }
    }
    return col;
}

__global__ void __launch_bounds__(NT) cut_plan3_kernel(dd3_geom g, dd3_state s,
                                                       const double* alpha, const double* beta,
                                                       double trunc, double cut_log,
                                                       const double* tmax, double* trunc_out,
                                                       int32_t* boxes_out) {
    __shared__ double red[NW];
    __shared__ int redi[NW];
    __shared__ double xs_a[64], xs_lm[64], xs_mu[64], xs_c0[64], xs_c1[64], xs_c2[64];
    __shared__ int xs_t[64];
    __shared__ int n_sh;
    __shared__ double s_amax;
    const int i = blockIdx.x;
    const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
    const int bs = s.block[0] * s.block[1] * s.block[2];
    const double eps = g.eps;
    if (threadIdx.x == 0) {
        int n = 0;
        double am = kNegInf;
        for (int t = 0; t < bs && n < 64; ++t) {
            int t0, t1, t2;
            unflat(t, bx.e[1], bx.e[2], t0, t1, t2);
            const int xi0 = bx.o[0] + t0, xi1 = bx.o[1] + t1, xi2 = bx.o[2] + t2;
            const int64_t id = ((int64_t)xi0 * g.nx[1] + xi1) * g.nx[2] + xi2;
            const double mu = s.mu[id];
            if (mu > 0) {
                xs_a[n] = alpha[id];
                xs_lm[n] = log(mu);
                xs_mu[n] = mu;
                xs_c0[n] = coord(g.x_org, g.x_dx, 0, xi0);
                xs_c1[n] = coord(g.x_org, g.x_dx, 1, xi1);
                xs_c2[n] = coord(g.x_org, g.x_dx, 2, xi2);
                xs_t[n] = t;
                am = fmax(am, alpha[id] / eps + log(mu));
                ++n;
            }
        }
        n_sh = n;
        s_amax = am;
    }
    __syncthreads();
    const int nxn = n_sh;
    const double amax = s_amax;
    double xlo[3], xhi[3];
    for (int a = 0; a < 3; ++a) {
        xlo[a] = coord(g.x_org, g.x_dx, a, bx.o[a]);
        xhi[a] = coord(g.x_org, g.x_dx, a, bx.o[a] + bx.e[a] - 1);
    }
    const int tn0 = (g.ny[0] + kCutTile - 1) / kCutTile, tn1 = (g.ny[1] + kCutTile - 1) / kCutTile,
              tn2 = (g.ny[2] + kCutTile - 1) / kCutTile;
    const int64_t ntile = (int64_t)tn0 * tn1 * tn2;
    double xacc[64];
    for (int k = 0; k < 64; ++k) xacc[k] = 0.0;
    double mass = 0.0, tr = 0.0, klp = 0.0, rem = 0.0;
    int lo0 = INT_MAX, lo1 = INT_MAX, lo2 = INT_MAX, hi0 = -1, hi1 = -1, hi2 = -1;
    for (int64_t t = threadIdx.x; t < ntile; t += NT) {
        int ta0, ta1, ta2;
        unflat(t, tn1, tn2, ta0, ta1, ta2);
        const int yl0 = ta0 * kCutTile, yl1 = ta1 * kCutTile, yl2 = ta2 * kCutTile;
        const int yh0 = min(g.ny[0], yl0 + kCutTile) - 1, yh1 = min(g.ny[1], yl1 + kCutTile) - 1,
                  yh2 = min(g.ny[2], yl2 + kCutTile) - 1;
        const double g0 = gap1(xlo[0], xhi[0], coord(g.y_org, g.y_dx, 0, yl0), coord(g.y_org, g.y_dx, 0, yh0));
        const double g1 = gap1(xlo[1], xhi[1], coord(g.y_org, g.y_dx, 1, yl1), coord(g.y_org, g.y_dx, 1, yh1));
        const double g2 = gap1(xlo[2], xhi[2], coord(g.y_org, g.y_dx, 2, yl2), coord(g.y_org, g.y_dx, 2, yh2));
        const double d2 = g0 * g0 + g1 * g1 + g2 * g2;
        // every term of the tile has log value <= amax + tmax - d2/eps (slack 1 for rounding)
        if (amax + tmax[t] - d2 / eps < cut_log - 1.0) continue;
        for (int y0 = yl0; y0 <= yh0; ++y0)
            for (int y1 = yl1; y1 <= yh1; ++y1)
                for (int y2 = yl2; y2 <= yh2; ++y2) {
                    const int64_t id = ((int64_t)y0 * g.ny[1] + y1) * g.ny[2] + y2;
                    const double nu = s.nu[id];
                    const double col = cut_col(
                        g, xs_c0, xs_c1, xs_c2, xs_a, xs_lm, xs_mu, nxn,
                        coord(g.y_org, g.y_dx, 0, y0), coord(g.y_org, g.y_dx, 1, y1),
                        coord(g.y_org, g.y_dx, 2, y2), nu, s.log_nu[id], beta[id], cut_log, &tr,
                        &klp, xacc);
                    mass += col;
                    if (col >= trunc) {
                        lo0 = min(lo0, y0); hi0 = max(hi0, y0);
                        lo1 = min(lo1, y1); hi1 = max(hi1, y1);
                        lo2 = min(lo2, y2); hi2 = max(hi2, y2);
                    } else {
                        rem += col;
                    }
                }
    }
    mass = bsum(mass, red);
    tr = bsum(tr, red);
    klp = bsum(klp, red);
    rem = bsum(rem, red);
    lo0 = bmin_i(lo0, redi); lo1 = bmin_i(lo1, redi); lo2 = bmin_i(lo2, redi);
    hi0 = bmax_i(hi0, redi); hi1 = bmax_i(hi1, redi); hi2 = bmax_i(hi2, redi);
    for (int k = threadIdx.x; k < bs; k += NT) s.x_marg[(int64_t)i * bs + k] = 0.0;
    __syncthreads();
    for (int k = 0; k < nxn; ++k) {
        const double v = bsum(xacc[k], red);
        if (threadIdx.x == 0) s.x_marg[(int64_t)i * bs + xs_t[k]] = v;
    }
    __syncthreads();
    int ne0 = 0, ne1 = 0, ne2 = 0;
    if (hi0 >= 0) { ne0 = hi0 - lo0 + 1; ne1 = hi1 - lo1 + 1; ne2 = hi2 - lo2 + 1; }
    if (threadIdx.x == 0) {
        double mmu = 0.0;
        for (int k = 0; k < nxn; ++k) mmu += xs_mu[k];
        s.transport[i] = tr;
        s.kl[i] = klp - mass + mmu * g.nu_total;
        trunc_out[i] = rem;
        int32_t* ob = boxes_out + (int64_t)i * 6;
        ob[0] = hi0 >= 0 ? lo0 : 0; ob[1] = ne0;
        ob[2] = hi0 >= 0 ? lo1 : 0; ob[3] = ne1;
        ob[4] = hi0 >= 0 ? lo2 : 0; ob[5] = ne2;
    }
    const int64_t nn = (int64_t)ne0 * ne1 * ne2;
    if (s.yval == nullptr || nn > s.cap) return;
    double* v = s.yval + (int64_t)i * s.cap;
    for (int64_t t = threadIdx.x; t < nn; t += NT) {
        int a0, a1, a2;
        unflat(t, ne1, ne2, a0, a1, a2);
        const int y0 = lo0 + a0, y1 = lo1 + a1, y2 = lo2 + a2;
        const int64_t id = ((int64_t)y0 * g.ny[1] + y1) * g.ny[2] + y2;
        const double col = cut_col(g, xs_c0, xs_c1, xs_c2, xs_a, xs_lm, xs_mu, nxn,
                                   coord(g.y_org, g.y_dx, 0, y0), coord(g.y_org, g.y_dx, 1, y1),
                                   coord(g.y_org, g.y_dx, 2, y2), s.nu[id], s.log_nu[id],
                                   beta[id], cut_log, nullptr, nullptr, nullptr);
        v[t] = col >= trunc ? col : 0.0;
    }
    if (threadIdx.x < 6) s.ybox[(int64_t)i * 6 + threadIdx.x] = boxes_out[(int64_t)i * 6 + threadIdx.x];
}

// Factorised plan cut (same outputs as cut_plan3_kernel, to rounding).  With
// a(x) = alpha/eps + log mu on the block's retained nodes, A = max a, and Y-normalised
// per-axis tables Kn_a = exp(-d_a^2/eps - c_a(y_a)) (c_a = the column max), every term is
//   exp((alpha + beta - c)/eps) mu nu = F(y) t(x, y),
//   F(y) = exp(beta/eps + log nu + A + sum_a c_a(y_a)),  t = exp(a - A) prod_a Kn_a,
// so a node's column sum, transport and entropy pieces are table products and FMAs
// instead of one exp per term.  A node whose normalised sum S = sum_x t is below kTiny
// (its dominant terms may have underflowed) or whose scale F would overflow takes the
// per-term exact path of cut_plan3_kernel.  Tables live in dynamic shared memory:
// per axis block_a x ny_a entries of Kn_a and d_a^2, and ny_a column shifts.
struct CutTabs {
    const double* K[3];
    const double* D[3];
    const double* c[3];
    int n[3];
};

__device__ __forceinline__ bool cut_fast(const CutTabs& T, const double* xs_ex, const double* xs_ae,
                                         const int* xi0, const int* xi1, const int* xi2, int nxn,
                                         double A, double eps, int y0, int y1, int y2, double bt,
                                         double lnu, bool stats, double& col, double& trc,
                                         double& klc, double* xacc) {
    const double logF = bt / eps + lnu + A + (T.c[0][y0] + T.c[1][y1] + T.c[2][y2]);
    if (!(logF <= 700.0)) return false;
    const double* K0 = T.K[0] + y0;
    const double* K1 = T.K[1] + y1;
    const double* K2 = T.K[2] + y2;
    const int n0 = T.n[0], n1 = T.n[1], n2 = T.n[2];
    double S = 0.0;
    for (int k = 0; k < nxn; ++k)
        S += xs_ex[k] * K0[xi0[k] * n0] * K1[xi1[k] * n1] * K2[xi2[k] * n2];
    if (!(S >= kTiny)) return false;
    const double F = exp(logF);
    col = F * S;
    if (!stats) return true;
    const double* D0 = T.D[0] + y0;
    const double* D1 = T.D[1] + y1;
    const double* D2 = T.D[2] + y2;
    double Sc = 0.0, Sa = 0.0;
    for (int k = 0; k < nxn; ++k) {
        const int i0 = xi0[k] * n0, i1 = xi1[k] * n1, i2 = xi2[k] * n2;
        const double t = xs_ex[k] * K0[i0] * K1[i1] * K2[i2];
        Sc = fma(t, D0[i0] + D1[i1] + D2[i2], Sc);
        Sa = fma(t, xs_ae[k], Sa);
        xacc[k] = fma(t, F, xacc[k]);
    }
    trc = F * Sc;
    klc = F * Sa + col * (bt / eps) - trc / eps;   // sum_x blk (alpha + beta - c) / eps
    return true;
}

// bv = beta / eps + log nu (the global X sweep's input for the separable cut's X-marginals)
__global__ void cut_bv_kernel(int64_t n, const double* beta, const double* log_nu, double eps,
                              double* bv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bv[i] = beta[i] / eps + log_nu[i];
}

// Separable plan cut.  Per basic cell: the 4^3 Y tiles whose bound clears cut_log give a
// candidate Y box; over it the column sums S(y) = sum_x t(x, y) and the cost-weighted sums
// Sc(y) = sum_x t c are three-stage contractions of the block weights exp(a - A) against
// the Y-normalised tables (axis 2, then 1, then 0; Sc through the d_a^2-weighted tables),
// so a node costs a few FMAs.  col(y) = F(y) S(y), transport = sum F Sc; the X-marginal of
// the cut is mu exp(alpha/eps + L) with L the global X sweep of beta/eps + log nu (every
// term of the block's rows), and the entropy piece follows from
//   sum blk (alpha + beta - c)/eps = sum_x xm alpha/eps + sum_y col beta/eps - transport/eps.
// A node whose normalised sum is below kTiny or whose scale would overflow takes the exact
// per-term path; a cell whose candidate box does not fit shared memory takes the per-node
// factorised path (cut_fast) for every node.
__global__ void __launch_bounds__(NT) cut_plan3s_kernel(dd3_geom g, dd3_state s,
                                                        const double* alpha, const double* beta,
                                                        const double* Lx, double trunc,
                                                        double cut_log, const double* tmax,
                                                        double* trunc_out, int32_t* boxes_out,
                                                        int smem_doubles) {
    extern __shared__ double dsm[];
    __shared__ double red[NW];
    __shared__ int redi[NW];
    __shared__ double xs_a[64], xs_lm[64], xs_mu[64], xs_c0[64], xs_c1[64], xs_c2[64];
    __shared__ double xs_ex[64], xs_ae[64], exb[64];
    __shared__ int xs_t[64], xs_i0[64], xs_i1[64], xs_i2[64];
    __shared__ int n_sh;
    __shared__ double s_amax;
    const int i = blockIdx.x;
    const B3 bx = ldbox(s.basic_xbox + (int64_t)i * 6);
    const int bs = s.block[0] * s.block[1] * s.block[2];
    const double eps = g.eps;
    if (threadIdx.x == 0) {
        int n = 0;
        double am = kNegInf;
        for (int t = 0; t < bs && t < 64; ++t) {
            exb[t] = 0.0;
            int t0, t1, t2;
            unflat(t, bx.e[1], bx.e[2], t0, t1, t2);
            const int xi0 = bx.o[0] + t0, xi1 = bx.o[1] + t1, xi2 = bx.o[2] + t2;
            const int64_t id = ((int64_t)xi0 * g.nx[1] + xi1) * g.nx[2] + xi2;
            const double mu = s.mu[id];
            if (mu > 0) {
                xs_a[n] = alpha[id];
                xs_lm[n] = log(mu);
                xs_mu[n] = mu;
                xs_c0[n] = coord(g.x_org, g.x_dx, 0, xi0);
                xs_c1[n] = coord(g.x_org, g.x_dx, 1, xi1);
                xs_c2[n] = coord(g.x_org, g.x_dx, 2, xi2);
                xs_i0[n] = t0; xs_i1[n] = t1; xs_i2[n] = t2;
                xs_t[n] = t;
                xs_ae[n] = alpha[id] / eps;
                am = fmax(am, alpha[id] / eps + xs_lm[n]);
                ++n;
            }
        }
        n_sh = n;
        s_amax = am;
        for (int k = 0; k < n; ++k) {
            xs_ex[k] = exp(xs_ae[k] + xs_lm[k] - am);
            exb[xs_t[k]] = xs_ex[k];
        }
    }
    __syncthreads();
    const int nxn = n_sh;
    const double amax = s_amax;
    double xlo[3], xhi[3];
    for (int a = 0; a < 3; ++a) {
        xlo[a] = coord(g.x_org, g.x_dx, a, bx.o[a]);
        xhi[a] = coord(g.x_org, g.x_dx, a, bx.o[a] + bx.e[a] - 1);
    }
    const int tn0 = (g.ny[0] + kCutTile - 1) / kCutTile, tn1 = (g.ny[1] + kCutTile - 1) / kCutTile,
              tn2 = (g.ny[2] + kCutTile - 1) / kCutTile;
    const int64_t ntile = (int64_t)tn0 * tn1 * tn2;
    // ---- candidate box: the surviving tiles' bounding box
    int cl0 = INT_MAX, cl1 = INT_MAX, cl2 = INT_MAX, ch0 = -1, ch1 = -1, ch2 = -1;
    for (int64_t t = threadIdx.x; t < ntile; t += NT) {
        int ta0, ta1, ta2;
        unflat(t, tn1, tn2, ta0, ta1, ta2);
        const int yl0 = ta0 * kCutTile, yl1 = ta1 * kCutTile, yl2 = ta2 * kCutTile;
        const int yh0 = min(g.ny[0], yl0 + kCutTile) - 1, yh1 = min(g.ny[1], yl1 + kCutTile) - 1,
                  yh2 = min(g.ny[2], yl2 + kCutTile) - 1;
        const double g0 = gap1(xlo[0], xhi[0], coord(g.y_org, g.y_dx, 0, yl0), coord(g.y_org, g.y_dx, 0, yh0));
        const double g1 = gap1(xlo[1], xhi[1], coord(g.y_org, g.y_dx, 1, yl1), coord(g.y_org, g.y_dx, 1, yh1));
        const double g2 = gap1(xlo[2], xhi[2], coord(g.y_org, g.y_dx, 2, yl2), coord(g.y_org, g.y_dx, 2, yh2));
        const double d2 = g0 * g0 + g1 * g1 + g2 * g2;
        if (amax + tmax[t] - d2 / eps < cut_log - 1.0) continue;
        cl0 = min(cl0, yl0); ch0 = max(ch0, yh0);
        cl1 = min(cl1, yl1); ch1 = max(ch1, yh1);
        cl2 = min(cl2, yl2); ch2 = max(ch2, yh2);
    }
    cl0 = bmin_i(cl0, redi); cl1 = bmin_i(cl1, redi); cl2 = bmin_i(cl2, redi);
    ch0 = bmax_i(ch0, redi); ch1 = bmax_i(ch1, redi); ch2 = bmax_i(ch2, redi);
    const int m0 = ch0 >= 0 ? ch0 - cl0 + 1 : 0, m1 = ch0 >= 0 ? ch1 - cl1 + 1 : 0,
              m2 = ch0 >= 0 ? ch2 - cl2 + 1 : 0;
    const int s0 = bx.e[0], s1 = bx.e[1], s2 = bx.e[2];
    // per-axis tables over the candidate ranges only (base pointers shifted so they are
    // indexed by absolute Y node): Kn_a, d_a^2, column shifts
    const int mm[3] = {m0, m1, m2};
    const int cl[3] = {cl0, cl1, cl2};
    const int64_t tabn = 2 * ((int64_t)s0 * m0 + (int64_t)s1 * m1 + (int64_t)s2 * m2) + m0 + m1 + m2;
    const bool tabs_fit = tabn <= smem_doubles;
    CutTabs T;
    double* free_sm = dsm;
    if (tabs_fit && m0 > 0) {
        double* p = dsm;
        double* Kb[3];
        double* Db[3];
        double* cb[3];
        for (int q = 0; q < 3; ++q) { Kb[q] = p; p += (int64_t)bx.e[q] * mm[q]; }
        for (int q = 0; q < 3; ++q) { Db[q] = p; p += (int64_t)bx.e[q] * mm[q]; }
        for (int q = 0; q < 3; ++q) { cb[q] = p; p += mm[q]; }
        free_sm = p;
        for (int q = 0; q < 3; ++q) {
            T.n[q] = mm[q];
            T.K[q] = Kb[q] - cl[q];
            T.D[q] = Db[q] - cl[q];
            T.c[q] = cb[q] - cl[q];
            for (int r = threadIdx.x; r < mm[q]; r += NT) {
                const double yc = coord(g.y_org, g.y_dx, q, cl[q] + r);
                double cm = kNegInf;
                for (int xq = 0; xq < bx.e[q]; ++xq) {
                    const double d = coord(g.x_org, g.x_dx, q, bx.o[q] + xq) - yc;
                    cm = fmax(cm, -(d * d) / eps);
                }
                cb[q][r] = cm;
                for (int xq = 0; xq < bx.e[q]; ++xq) {
                    const double d = coord(g.x_org, g.x_dx, q, bx.o[q] + xq) - yc;
                    Kb[q][xq * mm[q] + r] = exp(-(d * d) / eps - cm);
                    Db[q][xq * mm[q] + r] = d * d;
                }
            }
        }
    }
    __syncthreads();
    const int64_t used = free_sm - dsm;
    const int64_t need = 2 * (int64_t)s0 * s1 * m2 + 3 * (int64_t)s0 * m1 * m2;
    const bool sep = tabs_fit && need <= smem_doubles - used;
    double mass = 0.0, tr = 0.0, klp = 0.0, rem = 0.0;
    double xacc[64];   // per-term path scratch (the X-marginals come from the global sweep)
    for (int k = 0; k < 64; ++k) xacc[k] = 0.0;
    int lo0 = INT_MAX, lo1 = INT_MAX, lo2 = INT_MAX, hi0 = -1, hi1 = -1, hi2 = -1;
    double* U1 = free_sm;
    double* U1c = U1 + (int64_t)s0 * s1 * m2;
    double* U2 = U1c + (int64_t)s0 * s1 * m2;
    double* U2c2 = U2 + (int64_t)s0 * m1 * m2;
    double* U2c1 = U2c2 + (int64_t)s0 * m1 * m2;
    const double* K0 = T.K[0];
    const double* K1 = T.K[1];
    const double* K2 = T.K[2];
    const double* D0 = T.D[0];
    const double* D1 = T.D[1];
    const double* D2 = T.D[2];
    const int n0 = g.ny[0], n1 = g.ny[1], n2 = g.ny[2];
    if (sep && m0 > 0) {
        // stage 1 (axis 2): U1[x0][x1][y2] = sum_x2 exb K2, U1c with K2 d2^2
        const int nu1 = s0 * s1 * m2;
        for (int t = threadIdx.x; t < nu1; t += NT) {
            const int q = t / m2, y2 = t - q * m2;
            const double* e = exb + q * s2;
            double u = 0.0, uc = 0.0;
            for (int x2 = 0; x2 < s2; ++x2) {
                const double kv = e[x2] * K2[x2 * m2 + cl2 + y2];
                u += kv;
                uc = fma(kv, D2[x2 * m2 + cl2 + y2], uc);
            }
            U1[t] = u;
            U1c[t] = uc;
        }
        __syncthreads();
        // stage 2 (axis 1): U2[x0][y1][y2] = sum_x1 U1 K1; U2c2 from U1c; U2c1 with K1 d1^2
        const int nu2 = s0 * m1 * m2;
        for (int t = threadIdx.x; t < nu2; t += NT) {
            const int x0 = t / (m1 * m2), r = t - x0 * m1 * m2;
            const int y1 = r / m2, y2 = r - y1 * m2;
            double u = 0.0, uc2 = 0.0, uc1 = 0.0;
            for (int x1 = 0; x1 < s1; ++x1) {
                const double kv = K1[x1 * m1 + cl1 + y1];
                const double a1 = U1[(x0 * s1 + x1) * m2 + y2];
                u = fma(a1, kv, u);
                uc2 = fma(U1c[(x0 * s1 + x1) * m2 + y2], kv, uc2);
                uc1 = fma(a1 * kv, D1[x1 * m1 + cl1 + y1], uc1);
            }
            U2[t] = u;
            U2c2[t] = uc2;
            U2c1[t] = uc1;
        }
        __syncthreads();
        // stage 3 (axis 0) per candidate node
        const int nc = m0 * m1 * m2;
        Step3<NT> p(threadIdx.x, m1, m2);
        for (int t = threadIdx.x; t < nc; t += NT, p.next()) {
            const int y0 = cl0 + p.i0, y1 = cl1 + p.i1, y2 = cl2 + p.i2;
            const int64_t id = ((int64_t)y0 * n1 + y1) * n2 + y2;
            const double bt = beta[id];
            const double lnu = s.log_nu[id];
            const double logF = bt / eps + lnu + amax + (T.c[0][y0] + T.c[1][y1] + T.c[2][y2]);
            const int r = p.i1 * m2 + p.i2;
            double S = 0.0, Sc = 0.0;
            for (int x0 = 0; x0 < s0; ++x0) {
                const double kv = K0[x0 * m0 + y0];
                const int q = x0 * m1 * m2 + r;
                S = fma(U2[q], kv, S);
                Sc = fma(U2c2[q] + U2c1[q] + U2[q] * D0[x0 * m0 + y0], kv, Sc);
            }
            double col, trc;
            if (logF <= 700.0 && S >= kTiny) {
                const double F = exp(logF);
                col = F * S;
                trc = F * Sc;
            } else {
                trc = 0.0;
                double scratch = 0.0;   // per-term entropy pieces: the formula below covers them
                col = cut_col(g, xs_c0, xs_c1, xs_c2, xs_a, xs_lm, xs_mu, nxn,
                              coord(g.y_org, g.y_dx, 0, y0), coord(g.y_org, g.y_dx, 1, y1),
                              coord(g.y_org, g.y_dx, 2, y2), s.nu[id], lnu, bt, cut_log, &trc,
                              &scratch, xacc);
            }
            tr += trc;
            klp += col * (bt / eps);
            mass += col;
            if (col >= trunc) {
                lo0 = min(lo0, y0); hi0 = max(hi0, y0);
                lo1 = min(lo1, y1); hi1 = max(hi1, y1);
                lo2 = min(lo2, y2); hi2 = max(hi2, y2);
            } else {
                rem += col;
            }
        }
    } else if (m0 > 0) {
        // the candidate box exceeds shared memory: per-node factorised path over the tiles
        // (per-term exact path when not even the tables fit)
        for (int64_t t = threadIdx.x; t < ntile; t += NT) {
            int ta0, ta1, ta2;
            unflat(t, tn1, tn2, ta0, ta1, ta2);
            const int yl0 = ta0 * kCutTile, yl1 = ta1 * kCutTile, yl2 = ta2 * kCutTile;
            const int yh0 = min(n0, yl0 + kCutTile) - 1, yh1 = min(n1, yl1 + kCutTile) - 1,
                      yh2 = min(n2, yl2 + kCutTile) - 1;
            const double g0 = gap1(xlo[0], xhi[0], coord(g.y_org, g.y_dx, 0, yl0), coord(g.y_org, g.y_dx, 0, yh0));
            const double g1 = gap1(xlo[1], xhi[1], coord(g.y_org, g.y_dx, 1, yl1), coord(g.y_org, g.y_dx, 1, yh1));
            const double g2 = gap1(xlo[2], xhi[2], coord(g.y_org, g.y_dx, 2, yl2), coord(g.y_org, g.y_dx, 2, yh2));
            if (amax + tmax[t] - (g0 * g0 + g1 * g1 + g2 * g2) / eps < cut_log - 1.0) continue;
            for (int y0 = yl0; y0 <= yh0; ++y0)
                for (int y1 = yl1; y1 <= yh1; ++y1)
                    for (int y2 = yl2; y2 <= yh2; ++y2) {
                        const int64_t id = ((int64_t)y0 * n1 + y1) * n2 + y2;
                        const double bt = beta[id];
                        const double lnu = s.log_nu[id];
                        double col, trc = 0.0, klc = 0.0, scratch = 0.0;
                        if (!tabs_fit ||
                            !cut_fast(T, xs_ex, xs_ae, xs_i0, xs_i1, xs_i2, nxn, amax, eps, y0,
                                      y1, y2, bt, lnu, true, col, trc, klc, xacc))
                            col = cut_col(g, xs_c0, xs_c1, xs_c2, xs_a, xs_lm, xs_mu, nxn,
                                          coord(g.y_org, g.y_dx, 0, y0),
                                          coord(g.y_org, g.y_dx, 1, y1),
                                          coord(g.y_org, g.y_dx, 2, y2), s.nu[id], lnu, bt,
                                          cut_log, &trc, &scratch, xacc);
                        tr += trc;
                        klp += col * (bt / eps);
                        mass += col;
                        if (col >= trunc) {
                            lo0 = min(lo0, y0); hi0 = max(hi0, y0);
                            lo1 = min(lo1, y1); hi1 = max(hi1, y1);
                            lo2 = min(lo2, y2); hi2 = max(hi2, y2);
                        } else {
                            rem += col;
                        }
                    }
        }
    }
    // klp holds sum_y col beta/eps; the entropy piece adds the X side and the transport
    mass = bsum(mass, red);
    tr = bsum(tr, red);
    klp = bsum(klp, red);
    rem = bsum(rem, red);
    lo0 = bmin_i(lo0, redi); lo1 = bmin_i(lo1, redi); lo2 = bmin_i(lo2, redi);
    hi0 = bmax_i(hi0, redi); hi1 = bmax_i(hi1, redi); hi2 = bmax_i(hi2, redi);
    // X-marginals from the global X sweep: xm = mu exp(alpha/eps + L)
    double xa = 0.0;
    for (int k = threadIdx.x; k < bs; k += NT) {
        int t0, t1, t2;
        unflat(k, bx.e[1], bx.e[2], t0, t1, t2);
        const int64_t id = ((int64_t)(bx.o[0] + t0) * g.nx[1] + bx.o[1] + t1) * g.nx[2] + bx.o[2] + t2;
        const double mu = s.mu[id];
        double xm = 0.0;
        if (mu > 0) {
            xm = mu * exp(alpha[id] / eps + Lx[id]);
            xa += xm * (alpha[id] / eps);
        }
        s.x_marg[(int64_t)i * bs + k] = xm;
    }
    xa = bsum(xa, red);
    int ne0 = 0, ne1 = 0, ne2 = 0;
    if (hi0 >= 0) { ne0 = hi0 - lo0 + 1; ne1 = hi1 - lo1 + 1; ne2 = hi2 - lo2 + 1; }
    if (threadIdx.x == 0) {
        double mmu = 0.0;
        for (int k = 0; k < nxn; ++k) mmu += xs_mu[k];
        s.transport[i] = tr;
        s.kl[i] = (xa + klp - tr / eps) - mass + mmu * g.nu_total;
        trunc_out[i] = rem;
        int32_t* ob = boxes_out + (int64_t)i * 6;
        ob[0] = hi0 >= 0 ? lo0 : 0; ob[1] = ne0;
        ob[2] = hi0 >= 0 ? lo1 : 0; ob[3] = ne1;
        ob[4] = hi0 >= 0 ? lo2 : 0; ob[5] = ne2;
    }
    const int64_t nn = (int64_t)ne0 * ne1 * ne2;
    if (s.yval == nullptr || nn > s.cap) return;
    double* v = s.yval + (int64_t)i * s.cap;
    double dummy[1];
    for (int64_t t = threadIdx.x; t < nn; t += NT) {
        int a0, a1, a2;
        unflat(t, ne1, ne2, a0, a1, a2);
        const int y0 = lo0 + a0, y1 = lo1 + a1, y2 = lo2 + a2;
        const int64_t id = ((int64_t)y0 * n1 + y1) * n2 + y2;
        double col = -1.0;
        if (sep) {
            const double logF = beta[id] / eps + s.log_nu[id] + amax +
                                (T.c[0][y0] + T.c[1][y1] + T.c[2][y2]);
            const int r = (y1 - cl1) * m2 + (y2 - cl2);
            double S = 0.0;
            for (int x0 = 0; x0 < s0; ++x0) S = fma(U2[x0 * m1 * m2 + r], K0[x0 * m0 + y0], S);
            if (logF <= 700.0 && S >= kTiny) col = exp(logF) * S;
        } else if (tabs_fit) {
            double trc, klc;
            if (!cut_fast(T, xs_ex, xs_ae, xs_i0, xs_i1, xs_i2, nxn, amax, eps, y0, y1, y2,
                          beta[id], s.log_nu[id], false, col, trc, klc, dummy))
                col = -1.0;
        }
        if (col < 0.0)
            col = cut_col(g, xs_c0, xs_c1, xs_c2, xs_a, xs_lm, xs_mu, nxn,
                          coord(g.y_org, g.y_dx, 0, y0), coord(g.y_org, g.y_dx, 1, y1),
                          coord(g.y_org, g.y_dx, 2, y2), s.nu[id], s.log_nu[id], beta[id],
                          cut_log, nullptr, nullptr, nullptr);
        v[t] = col >= trunc ? col : 0.0;
    }
    if (threadIdx.x < 6) s.ybox[(int64_t)i * 6 + threadIdx.x] = boxes_out[(int64_t)i * 6 + threadIdx.x];
}

__global__ void __launch_bounds__(NT) seed_duals3_kernel(dd3_geom g, dd3_state s, int w0, int w1,
                                                         int w2, const int32_t* xbox,
                                                         const int32_t* ybox, const double* alpha,
                                                         const double* beta) {
    const int j = blockIdx.x;
    const B3 xb = ldbox(xbox + (int64_t)j * 6);
    const B3 yb = ldbox(ybox + (int64_t)j * 6);
    const int64_t nx = (int64_t)w0 * w1 * w2;
    for (int64_t x = threadIdx.x; x < nx; x += NT) {
        int x0, x1, x2;
        unflat(x, w1, w2, x0, x1, x2);
        const int r0 = xb.o[0] + x0, r1 = xb.o[1] + x1, r2 = xb.o[2] + x2;
        double a = 0.0;
        if (r0 >= 0 && r0 < g.nx[0] && r1 >= 0 && r1 < g.nx[1] && r2 >= 0 && r2 < g.nx[2])
            a = alpha[((int64_t)r0 * g.nx[1] + r1) * g.nx[2] + r2];
        s.d_alpha[(int64_t)j * nx + x] = a;
    }
    const int64_t ny = bsize(yb);
    for (int64_t y = threadIdx.x; y < ny; y += NT) {
        int y0, y1, y2;
        unflat(y, yb.e[1], yb.e[2], y0, y1, y2);
        s.d_beta[(int64_t)j * s.d_cap + y] =
            beta[((int64_t)(yb.o[0] + y0) * g.ny[1] + yb.o[1] + y1) * g.ny[2] + yb.o[2] + y2];
    }
    if (threadIdx.x < 6) s.d_box[(int64_t)j * 6 + threadIdx.x] = ybox[(int64_t)j * 6 + threadIdx.x];
    if (threadIdx.x == 0) s.d_has[j] = 1;
}

}  // namespace v3

// ---- host wrappers ------------------------------------------------------------------------

static int v3_blocks(int64_t n) {
    int64_t b = (n + v3::NT - 1) / v3::NT;
    if (b > 8192) b = 8192;
    if (b < 1) b = 1;
    return (int)b;
}

struct GridWs {
    int64_t wmax, t1, t2;
};

static GridWs grid_ws_parts(const dd3_geom* g) {
    const int64_t X = (int64_t)g->nx[0] * g->nx[1] * g->nx[2];
    const int64_t Y = (int64_t)g->ny[0] * g->ny[1] * g->ny[2];
    const int64_t i1 = (int64_t)g->ny[0] * g->ny[1] * g->nx[2];
    const int64_t i2 = (int64_t)g->ny[0] * g->nx[1] * g->nx[2];
    const int64_t j1 = (int64_t)g->nx[0] * g->nx[1] * g->ny[2];
    const int64_t j2 = (int64_t)g->nx[0] * g->ny[1] * g->ny[2];
    GridWs w;
    w.t1 = i1 > j1 ? i1 : j1;
    w.t2 = i2 > j2 ? i2 : j2;
    int64_t m = X > Y ? X : Y;
    m = m > w.t1 ? m : w.t1;
    w.wmax = m > w.t2 ? m : w.t2;
    return w;
}

extern "C" int64_t dd3_grid_ws(const dd3_geom* g) {
    const GridWs w = grid_ws_parts(g);
    int64_t tab = 0;
    for (int a = 0; a < 3; ++a) tab += (int64_t)g->nx[a] * g->ny[a];
    return 2 * w.wmax + w.t1 + w.t2 + 2 * tab + 16;
}

static int grid_lse3(const dd3_geom* g, const double* v, double* out, int to_x, double* work,
                     int tables_ready, const int* stop, cudaStream_t st) {
    const int* in = to_x ? g->ny : g->nx;
    const int* on = to_x ? g->nx : g->ny;
    const double* in_org = to_x ? g->y_org : g->x_org;
    const double* on_org = to_x ? g->x_org : g->y_org;
    const double in_dx = to_x ? g->y_dx : g->x_dx, on_dx = to_x ? g->x_dx : g->y_dx;
    const GridWs ws = grid_ws_parts(g);
    double* w = work;
    double* rmax = w + ws.wmax;
    double* T1 = rmax + ws.wmax;
    double* T2 = T1 + ws.t1;
    int64_t tabn = 0;
    for (int a = 0; a < 3; ++a) tabn += (int64_t)g->nx[a] * g->ny[a];
    double* tab[3];
    tab[0] = T2 + ws.t2 + (to_x ? 0 : tabn);     // one table set per direction
    tab[1] = tab[0] + (int64_t)on[0] * in[0];
    tab[2] = tab[1] + (int64_t)on[1] * in[1];
    if (!tables_ready)
        for (int a = 0; a < 3; ++a)
            v3::g_table_kernel<<<v3_blocks((int64_t)on[a] * in[a]), v3::NT, 0, st>>>(
                on[a], in[a], on_org[a], on_dx, in_org[a], in_dx, g->eps, tab[a]);
    // axis 2: (in0*in1, in2, 1) -> (in0*in1, on2, 1); axis 1: (in0, in1, on2) -> (in0, on1,
    // on2); axis 0: (1, in0, on1*on2) -> (1, on0, on1*on2)  (sinkhorn.py:159-175 order)
    const v3::GStage stages[3] = {
        {v, T1, w, rmax, tab[2], in[0] * in[1], in[2], 1, on[2], on_org[2], on_dx, in_org[2],
         in_dx, g->eps, stop},
        {T1, T2, w, rmax, tab[1], in[0], in[1], on[2], on[1], on_org[1], on_dx, in_org[1], in_dx,
         g->eps, stop},
        {T2, out, w, rmax, tab[0], 1, in[0], on[1] * on[2], on[0], on_org[0], on_dx, in_org[0],
         in_dx, g->eps, stop}};
    for (int k = 0; k < 3; ++k) {
        const v3::GStage& S = stages[k];
        v3::g_rows_kernel<<<v3_blocks((int64_t)S.A * S.B * (S.B == 1 ? 32 : 1)), v3::NT, 0, st>>>(S);
        v3::g_contract_kernel<<<v3_blocks((int64_t)S.A * S.O * S.B), v3::NT, 0, st>>>(S);
    }
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_grid_lse(const dd3_geom* g, const double* v, double* out, int to_x, double* work,
                            int tables_ready, void* stream) {
    return grid_lse3(g, v, out, to_x, work, tables_ready, nullptr, (cudaStream_t)stream);
}

extern "C" int64_t dd3_sinkhorn_ws(const dd3_geom* g) {
    return dd3_grid_ws(g) + dd_sk_partial_doubles() + 16;
}

// Global unbalanced Sinkhorn iterations k0 .. k0+n_iters-1 enqueued without host
// synchronisation (dd_sinkhorn_run over three axes): the stopping test runs on the device
// (ctl_i[0]), every later launch of the chunk is a no-op once it is set.
extern "C" int dd3_sinkhorn_run(const dd3_geom* g, double* alpha, double* beta, const double* mu,
                                const double* log_mu, const double* log_nu, double* L, double* z,
                                double* bv, double* av, double* px, double* work, int* ctl_i,
                                double* ctl_d, double thr, int k0, int n_iters, int tables_ready,
                                void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nx = (int64_t)g->nx[0] * g->nx[1] * g->nx[2];
    const int64_t ny = (int64_t)g->ny[0] * g->ny[1] * g->ny[2];
    double* partial = work + dd3_grid_ws(g);
    const double eps = g->eps, lam = g->lam;
    const double ratio = eps * lam / (eps + lam);
    const int* stop = ctl_i;
    int rc;
    for (int k = k0; k < k0 + n_iters; ++k) {
        const int ready = (tables_ready || k > k0) ? 1 : 0;
        if ((rc = dd_sk_axpb(ny, beta, eps, log_nu, bv, 1, stop, st))) return rc;
        if ((rc = grid_lse3(g, bv, L, 1, work, ready, stop, st))) return rc;
        if (k >= 2 && (rc = dd_sk_gap(nx, alpha, L, mu, eps, lam, px, partial, thr, ctl_i, ctl_d, st)))
            return rc;
        if ((rc = dd_sk_axpb(nx, L, -ratio, nullptr, alpha, 0, stop, st))) return rc;
        if ((rc = dd_sk_axpb(nx, alpha, eps, log_mu, av, 1, stop, st))) return rc;
        if ((rc = grid_lse3(g, av, z, 0, work, ready, stop, st))) return rc;
        if ((rc = dd_sk_newton(ny, z, ratio, lam, beta, ctl_i, k, st))) return rc;
    }
    return 0;
}

extern "C" int dd3_prolong(const int32_t* nf, const int32_t* nc, const double* coarse, double* fine,
                           void* stream) {
    const int64_t n = (int64_t)nf[0] * nf[1] * nf[2];
    v3::prolong3_kernel<<<v3_blocks(n), v3::NT, 0, (cudaStream_t)stream>>>(
        nf[0], nf[1], nf[2], nc[0], nc[1], nc[2], coarse, fine);
    return dd_set_error(cudaGetLastError());
}

extern "C" int64_t dd3_cell_ws_size(const int32_t* w, const int32_t* n) {
    const int ww[3] = {w[0], w[1], w[2]}, nn[3] = {n[0], n[1], n[2]};
    return v3::ws_layout(ww, nn).total;
}

extern "C" int dd3_cell_solve(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                              void* stream) {
    if (b->n_cells <= 0) return 0;
    // dynamic shared memory for the hot per-cell arrays (the kernel falls back to the
    // global workspace for a cell whose arrays do not fit)
    if (b->precision != 0 && b->precision != 1) return dd_set_error(cudaErrorInvalidValue);
    auto kern = b->precision ? v3::cell_solve3_kernel<v3::CELL_NT, 1>
                             : v3::cell_solve3_kernel<v3::CELL_NT, 0>;
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return dd_set_error(e);
    const int64_t cap = 227 * 1024 - (int64_t)fa.sharedSizeBytes - 1024;
    int64_t bytes = (int64_t)b->smem_doubles * (int64_t)sizeof(double);
    if (bytes > cap) bytes = cap;
    if (bytes < 0) bytes = 0;
    dd3_batch bb = *b;
    bb.smem_doubles = (int32_t)(bytes / (int64_t)sizeof(double));
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return dd_set_error(e);
    kern<<<b->n_cells, v3::CELL_NT, (size_t)bytes, (cudaStream_t)stream>>>(*g, *s, bb);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_cell_delta(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                              double theta_safe, double* dy, double* cd, void* stream) {
    if (b->n_cells <= 0) return 0;
    v3::cell_delta3_kernel<<<b->n_cells, v3::NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, theta_safe,
                                                                           dy, cd);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_blend_d1(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                            const double* theta, double* out, void* stream) {
    if (b->n_cells <= 0) return 0;
    v3::blend_d1_3_kernel<<<b->n_cells, v3::NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, theta, out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_opt_gh(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                          const double* dy, int c, double th, double th_cur, const double* ycur,
                          double* out, void* stream) {
    if (c < 0 || c >= b->n_cells) return dd_set_error(cudaErrorInvalidValue);
    v3::opt_gh3_kernel<<<1, v3::NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, dy, c, th, th_cur,
                                                               ycur, out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_opt_set(const dd3_geom* g, const dd3_batch* b, const double* dy, int c,
                           double dth, double* ycur, void* stream) {
    if (c < 0 || c >= b->n_cells) return dd_set_error(cudaErrorInvalidValue);
    v3::opt_set3_kernel<<<1, v3::NT, 0, (cudaStream_t)stream>>>(*g, *b, dy, c, dth, ycur);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_cell_commit(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                               const double* theta, double* alpha_grid, double* yrun,
                               double* errs, void* stream) {
    if (b->n_cells <= 0) return 0;
    v3::cell_commit3_kernel<<<b->n_cells, v3::NT, 0, (cudaStream_t)stream>>>(*g, *s, *b, theta,
                                                                            alpha_grid, yrun, errs);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_gather(const dd3_geom* g, int n, const int32_t* box, int bstride,
                          const double* vals, int64_t vstride, const int64_t* voff,
                          const double* scale, const double* base, double* out, int kl_mode,
                          const double* nu, double* partial, int* n_partial, void* stream) {
    const int n0 = g->ny[0], n1 = g->ny[1], n2 = g->ny[2];
    const int T2 = n2 < 32 ? n2 : 32;
    int T1 = v3::NT / T2;
    if (T1 > n1) T1 = n1;
    int T0 = v3::NT / (T1 * T2);
    if (T0 > n0) T0 = n0;
    if (T0 < 1) T0 = 1;
    const int tiles = ((n0 + T0 - 1) / T0) * ((n1 + T1 - 1) / T1) * ((n2 + T2 - 1) / T2);
    v3::GItems it{n, box, bstride, vals, vstride, voff, scale};
    v3::gather3_kernel<<<tiles, v3::NT, 0, (cudaStream_t)stream>>>(*g, it, T0, T1, T2, base, out,
                                                                   kl_mode, nu, partial);
    if (n_partial) *n_partial = tiles;
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_cell_terms(const dd3_geom* g, const dd3_state* s, double* out, void* stream) {
    v3::cell_terms3_kernel<<<s->n_basic, v3::NT, 0, (cudaStream_t)stream>>>(*g, *s, out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_product_init(const dd3_geom* g, const dd3_state* s, double mu_total,
                                void* stream) {
    v3::product_init3_kernel<<<s->n_basic, v3::NT, 0, (cudaStream_t)stream>>>(*g, *s, mu_total);
    return dd_set_error(cudaGetLastError());
}

static int64_t cut_tile_count(const dd3_geom* g) {
    const int k = v3::kCutTile;
    return (int64_t)((g->ny[0] + k - 1) / k) * ((g->ny[1] + k - 1) / k) * ((g->ny[2] + k - 1) / k);
}

extern "C" int64_t dd3_cut_tiles(const dd3_geom* g) {
    // workspace of dd3_cut_plan: tile maxima, beta/eps + log nu (Y grid), the global X
    // sweep (X grid) and its grid-LSE workspace
    const int64_t nx = (int64_t)g->nx[0] * g->nx[1] * g->nx[2];
    const int64_t ny = (int64_t)g->ny[0] * g->ny[1] * g->ny[2];
    return cut_tile_count(g) + ny + nx + dd3_grid_ws(g) + 16;
}

extern "C" int dd3_cut_plan(const dd3_geom* g, const dd3_state* s, const double* alpha,
                            const double* beta, double trunc, double cut_log, double* tile_max,
                            double* trunc_out, int32_t* boxes_out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nx = (int64_t)g->nx[0] * g->nx[1] * g->nx[2];
    const int64_t ny = (int64_t)g->ny[0] * g->ny[1] * g->ny[2];
    double* tmax = tile_max;
    double* bv = tmax + cut_tile_count(g);
    double* Lx = bv + ny;
    double* lws = Lx + nx;
    v3::cut_tiles_kernel<<<v3_blocks(cut_tile_count(g)), v3::NT, 0, st>>>(*g, beta, s->log_nu,
                                                                           tmax);
    const int64_t static_b = 8 * 1024;   // the kernel's static shared arrays (< 8 KB)
    const int64_t avail = 227 * 1024 - static_b;
    if (s->block[0] * s->block[1] * s->block[2] <= 64) {
        v3::cut_bv_kernel<<<v3_blocks(ny), v3::NT, 0, st>>>(ny, beta, s->log_nu, g->eps, bv);
        int rc = grid_lse3(g, bv, Lx, 1, lws, 0, nullptr, st);
        if (rc) return rc;
        cudaError_t e = cudaFuncSetAttribute(v3::cut_plan3s_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)avail);
        if (e != cudaSuccess) return dd_set_error(e);
        v3::cut_plan3s_kernel<<<s->n_basic, v3::NT, (size_t)avail, st>>>(
            *g, *s, alpha, beta, Lx, trunc, cut_log, tmax, trunc_out, boxes_out,
            (int)(avail / sizeof(double)));
    } else {
        v3::cut_plan3_kernel<<<s->n_basic, v3::NT, 0, st>>>(*g, *s, alpha, beta, trunc, cut_log,
                                                             tmax, trunc_out, boxes_out);
    }
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd3_seed_duals(const dd3_geom* g, const dd3_state* s, int n_comp, const int32_t* nxw,
                              const int32_t* xbox, const int32_t* ybox, const double* alpha,
                              const double* beta, void* stream) {
    if (n_comp <= 0) return 0;
    v3::seed_duals3_kernel<<<n_comp, v3::NT, 0, (cudaStream_t)stream>>>(
        *g, *s, nxw[0], nxw[1], nxw[2], xbox, ybox, alpha, beta);
    return dd_set_error(cudaGetLastError());
}
