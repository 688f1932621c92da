// Shared device helpers for the domdec B200 library.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <limits.h>

#ifndef DD_NT
#define DD_NT 512
#endif
#define DD_NW (DD_NT / 32)

namespace dd {

constexpr double kNegInf = -__builtin_huge_val();
constexpr double kDegenerateBetaScale = 700.0;  // sinkhorn.py:54

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block reductions (fixed tree). `red` is __shared__ double[DD_NW+1].
// All threads of the block must call; all receive the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < DD_NW ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) red[DD_NW] = t;
    }
    __syncthreads();
    return red[DD_NW];
}
__device__ __forceinline__ double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < DD_NW ? red[lane] : kNegInf;
        t = warp_max(t);
        if (lane == 0) red[DD_NW] = t;
    }
    __syncthreads();
    return red[DD_NW];
}
__device__ __forceinline__ int block_min_i(int v, int* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_min_i(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int t = lane < DD_NW ? red[lane] : 0x7fffffff;
        t = warp_min_i(t);
        if (lane == 0) red[DD_NW] = t;
    }
    __syncthreads();
    return red[DD_NW];
}
__device__ __forceinline__ int block_max_i(int v, int* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_max_i(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int t = lane < DD_NW ? red[lane] : -0x7fffffff;
        t = warp_max_i(t);
        if (lane == 0) red[DD_NW] = t;
    }
    __syncthreads();
    return red[DD_NW];
}

// Single-barrier deterministic block sum.  `red2` is __shared__ double[2*DD_NW];
// successive calls must alternate `parity` (the next call's barrier orders the
// re-use of a buffer).  Every thread sums the per-warp partials in warp order.
__device__ __forceinline__ double block_sum1(double v, double* red2, int parity) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    double* r = red2 + parity * DD_NW;
    if (lane == 0) r[wid] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < DD_NW; ++k) t += r[k];
    return t;
}

// Single-barrier block max (same double-buffer protocol as block_sum1).
__device__ __forceinline__ double block_max1(double v, double* red2, int parity) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_max(v);
    double* r = red2 + parity * DD_NW;
    if (lane == 0) r[wid] = v;
    __syncthreads();
    // every warp folds the DD_NW partials across its lanes (max is exact, so the
    // result does not depend on the order): one shared load per thread instead of DD_NW
    double t = r[lane & (DD_NW - 1)];
#pragma unroll
    for (int o = DD_NW / 2; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    return t;
}

__device__ __forceinline__ double warp_max_all(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// numpy.logaddexp semantics (npymath npy_logaddexp)
__device__ __forceinline__ double logaddexp(double x, double y) {
    if (x == y) return x + 0.693147180559945309417232121458176568;
    const double t = x - y;
    if (t > 0) return x + log1p(exp(-t));
    if (t <= 0) return y + log1p(exp(t));
    return t;  // nan
}

// scipy.special.expit
__device__ __forceinline__ double expit(double u) { return 1.0 / (1.0 + exp(-u)); }

// scipy.special.xlogy
__device__ __forceinline__ double xlogy(double x, double y) {
    return x == 0.0 ? 0.0 : x * log(y);
}

// Per-node KL contribution sigma*(r log r - r + 1) (measures.py:326-334)
__device__ __forceinline__ double kl_term(double rho, double sigma) {
    if (sigma > 0) return xlogy(rho, rho / sigma) - rho + sigma;
    return rho > 0 ? __builtin_huge_val() : 0.0;
}

constexpr double kRelaxedStep2 = 2e-6;   // fp32 mode: (step/eps)^2 bound of the early exit

// Unbalanced Y step for one node (sinkhorn.py:230-333 restated per node).
// Returns beta; *deg set when the node is degenerate (m == 0, z == -inf).
__device__ __forceinline__ double newton_node(double z, double m, bool has_m, double beta0,
                                              double eps, double lam, double tol, int max_iters,
                                              int* deg, long long* steps = nullptr,
                                              int* nstat = nullptr,
                                              double lm_cached = __builtin_nan(""),
                                              const bool relaxed = false) {
    const double ratio = eps * lam / (eps + lam);
    const bool fz = z > kNegInf;
    if (!has_m || !(m > 0)) {
        if (fz) return -ratio * z;
        *deg = 1;
        return lam * kDegenerateBetaScale;
    }
    if (!fz) return -lam * log(m);
    const double inv_eps = 1.0 / eps, inv_lam = 1.0 / lam;
    const double lm = lm_cached == lm_cached ? lm_cached : log(m);   // NaN: not cached
    const double b2 = -ratio * z;
    // Safeguard bracket, evaluated lazily.  The computed logaddexp(lm, z) lies in
    // [M, M + 0.7] with M = max(lm, z) (its log1p term is in [0, ln 2]), so
    //   lo <= loU = min(-lam M, b2) - lam   and   hi >= hiL = max(-lam (M + 0.7), b2) + lam
    // in floating point (each operation is monotone).  While beta0 and every iterate
    // stay inside (loU, hiL) the exact bracket cannot change the result, so its two
    // transcendentals are only paid when a value reaches the conservative edge.
    const double M = fmax(lm, z);
    double lo = fmin(-lam * M, b2) - lam;
    double hi = fmax(-lam * (M + 0.7), b2) + lam;
    bool exact = false;
    auto make_exact = [&]() {
        const double b1 = -lam * logaddexp(lm, z);
        lo = fmin(b1, b2) - lam;
        hi = fmax(b1, b2) + lam;
        exact = true;
    };
    if (!((beta0 > lo) && (beta0 < hi))) make_exact();
    double b = fmin(fmax(beta0, lo), hi);  // np.clip
    if (nstat && b != beta0) nstat[0] += 1;
    int nev = 0;
    for (int it = 0; it < max_iters; ++it) {
        if (steps) ++*steps;
        ++nev;
        const double w = b * inv_eps + z;
        // logaddexp(lm, w) and expit(w - lm) from one exponential, without branches:
        // lanes of a warp fall on both sides of t = 0, and a divergent if/else made the
        // warp issue both exp/log1p chains.  Same values as the two-sided form
        // (t > 0: exp(-t), w + log1p(e), 1/(1+e); t <= 0: exp(t), lm + log1p(e), e/(1+e)).
        const double t = w - lm;
        const bool pos = t > 0;
        double e, l1, sig;
        if (relaxed) {
            // fp32 mode: the transcendental part log1p(exp(-|t|)) in [0, ln 2] and the
            // slope factor in fp32; w, lm, the sum g and the iterate stay fp64.  The
            // error of l1 is relative (~1e-7 (1 + |t|)), and l1 / sig ~ 1 + e, so the
            // root moves by ~1e-7 (1 + |t|) in beta/eps: inside the 1e-4 bar.  sig only
            // sets the Newton slope (convergence rate, not the root).
            const float ef = expf((float)(pos ? -t : t));
            e = (double)ef;
            l1 = (double)log1pf(ef);
            sig = (double)((pos ? 1.0f : ef) * __frcp_rn(1.0f + ef));
        } else {
            e = exp(pos ? -t : t);
            l1 = log1p(e);
            sig = (pos ? 1.0 : e) / (1.0 + e);
        }
        double la = (pos ? w : lm) + l1;
        if (t == 0) la = w + 0.693147180559945309417232121458176568;
        if (t != t) { la = t; sig = t; }
        const double g = la + b * inv_lam;
        if (g == 0.0) break;   // step 0: inactive (avoids the division's slow path)
        const double gp = sig * inv_eps + inv_lam;
        const double step = relaxed ? g * (double)__frcp_rn((float)gp) : g / gp;
        const bool active = (fabs(g) > tol) || (fabs(step) > 4e-16 * (1.0 + fabs(b)));
        if (!active) break;
        double nb = b - step;
        if (!exact && !((nb > lo) && (nb < hi))) make_exact();
        bool safeguarded = false;
        if (!((nb > lo) && (nb < hi))) {
            safeguarded = true;
            if (g > 0) hi = fmin(hi, b);
            else lo = fmax(lo, b);
            if ((nb <= lo) || (nb >= hi)) {
                nb = 0.5 * (lo + hi);
                if (nstat) nstat[1] += 1;
            }
        }
        // fixed point of the iteration (the step is below half an ulp of b): every
        // further pass of the reference loop recomputes the same g and step and
        // leaves b unchanged until max_iters, so stopping here returns the same b.
        // Exception (batch coupling of the reference's vectorised loop,
        // sinkhorn.py:320-326): if a batch-mate leaves its bracket in a later pass,
        // the reference shrinks every active node's bracket to b and bisects this
        // stuck node once; it then re-converges to within the tolerance, so the two
        // results agree to the Newton tolerance, not bitwise, in that case.
        if (nb == b) break;
        // Converged step.  Newton's next correction is at most
        //   |g''| step^2 / (2 g') <= (1 - sig) step^2 / (2 eps)   (g'' = sig(1-sig)/eps^2),
        // so once step^2/eps <= 2^-52 |nb| it is below one ulp of nb and the confirming
        // evaluation the reference loop spends to observe that is skipped.  The result
        // differs from running it by at most that ulp (well inside the 1e-9 parity bar).
        if (!safeguarded && step * step * inv_eps <= 2.220446049250313e-16 * fabs(nb)) {
            b = nb;
            break;
        }
        // fp32 mode only (relaxed): the same bound in the units that matter for the
        // 1e-4 parity bar.  beta enters every exponent as beta/eps, and the correction
        // left after this step is at most (step/eps)^2 / 2 there, so a step with
        // (step/eps)^2 <= kRelaxedStep2 leaves the node within 1e-6 of the root in the
        // exponent (1e-6 relative on the plan entries) and the confirming evaluation is
        // skipped.  The next Sinkhorn iteration starts its Newton step from this value
        // with the fresh z, so the leftover does not accumulate.
        if (relaxed && !safeguarded) {
            const double se = step * inv_eps;
            if (se * se <= kRelaxedStep2) {
                b = nb;
                break;
            }
        }
        b = nb;
    }
    if (nstat) {
        nstat[2] = max(nstat[2], nev);
        if (nev >= 6) nstat[3] += 1;
    }
    return b;
}



// _move_mass (cells.py:483-502) across a thread block, same arithmetic as the reference's
// sequential walk: the donor row's running sum is accumulated by ONE thread in node
// order (numpy cumsum's order; chunks of S nodes staged through shared memory by the
// whole block, so the chain runs at the DADD latency instead of a global load per node),
// the first node whose running sum reaches `amount` is published, and the element-wise
// moves (rowr[y] += rowd[y]; rowd[y] = 0 below that node, the partial move on it) run
// across the block.  Returns 1 when the donor cannot cover the amount (everything is
// handed over: the reference's fallback).  Every thread of the block must call it;
// stage holds S (<= T) doubles and pub 4 doubles of shared memory.
template <int T, int S = T>
__device__ int move_mass_block(double* rowd, double* rowr, int64_t ny, double amount,
                               double* stage, double* pub) {
    static_assert(S <= T, "one staged node per thread");
    double cum = 0.0;   // thread 0 only
    if (threadIdx.x == 0) { pub[0] = -1.0; pub[1] = 0.0; pub[2] = 0.0; }
    __syncthreads();
    for (int64_t base = 0; base < ny; base += S) {
        const int64_t y = base + threadIdx.x;
        if (threadIdx.x < S) stage[threadIdx.x] = y < ny ? rowd[y] : 0.0;
        __syncthreads();
        if (threadIdx.x == 0) {
            const int n = (int)((ny - base) < (int64_t)S ? (ny - base) : (int64_t)S);
            for (int j = 0; j < n; ++j) {
                const double prev = cum;
                cum += stage[j];
                if (cum >= amount) {
                    pub[0] = (double)(base + j);
                    pub[1] = prev;
                    break;
                }
            }
            pub[2] = cum;
        }
        __syncthreads();
        if (pub[0] >= 0.0) break;
    }
    const int64_t kk = (int64_t)pub[0];
    const double prev = pub[1], total = pub[2];
    int fb = 0;
    if (kk < 0) {
        if (ny > 0 && total > 0) {
            for (int64_t y = threadIdx.x; y < ny; y += T) { rowr[y] += rowd[y]; rowd[y] = 0.0; }
        }
        fb = 1;
    } else {
        for (int64_t y = threadIdx.x; y < kk; y += T) { rowr[y] += rowd[y]; rowd[y] = 0.0; }
        if (threadIdx.x == 0) {
            const double part = amount - (kk ? prev : 0.0);
            rowd[kk] -= part;
            rowr[kk] += part;
        }
    }
    __syncthreads();
    return fb;
}

}  // namespace dd

// Deterministic boxed gather-sum (grid.cu): out = base + sum_i scale_i * v_i over
// the items' boxes, accumulated in item order; library-internal.
int dd_box_gather(int n, const int32_t* box, int bstride, const double* vals, int64_t vstride,
                  const int64_t* voff, int voff_stride, const double* scale, int ny0, int ny1,
                  const double* base, double* out, cudaStream_t st);

// Stop-aware element-wise pieces of one global Sinkhorn iteration (grid.cu), for the
// three-axis device loop (vol.cu); library-internal.
int dd_sk_axpb(int64_t n, const double* a, double s, const double* b, double* out, int divide,
               const int* stop, cudaStream_t st);
int dd_sk_gap(int64_t nx, const double* alpha, const double* L, const double* mu, double eps,
              double lam, double* px, double* partial, double thr, int* ctl_i, double* ctl_d,
              cudaStream_t st);
int dd_sk_newton(int64_t ny, const double* z, double ratio, double lam, double* beta, int* ctl_i,
                 int k, cudaStream_t st);
int64_t dd_sk_partial_doubles();
