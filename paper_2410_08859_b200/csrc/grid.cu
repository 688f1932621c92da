// Full-grid kernels: separable log-sum-exp sweeps, reductions, state setup.

#include <stdio.h>
#include <algorithm>
#include <string.h>

#include "common.cuh"
#include "domdec_b200.h"

static thread_local char g_err[512] = "";

extern "C" int dd_set_error(cudaError_t e) {
    if (e == cudaSuccess) return 0;
    snprintf(g_err, sizeof(g_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return -(int)e;
}

extern "C" const char* dd_last_error(void) { return g_err; }

extern "C" int dd_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

extern "C" int dd_abi_version(void) { return 1; }

namespace dd {

// Axis table in the reference's rounding, transposed: tab[m*N + n] = -(d*d)/eps with
// d = (p0 + pd*n) - (q0 + qd*m)  (sinkhorn.py:149-151 _neg_sq, computed once per sweep).
__global__ void neg_sq_table_kernel(int M, int N, double p0, double pd, double q0, double qd,
                                    double eps, double* tab) {
    const int64_t tot = (int64_t)M * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(i / N), n = (int)(i - (int64_t)m * N);
        const double d = (p0 + pd * (double)n) - (q0 + qd * (double)m);
        tab[i] = -(d * d) / eps;
    }
}

// One separable stage for kRows input rows at once (they share every table load):
//   out[r][n] = LSE_m(in[r][m] + tab[m][n])
// two passes (max, then sum of exp(t - max) over the terms with t - max > -760; the
// skipped ones are exactly 0 in double), the reference's _lse order per output.
// Table reads are coalesced over n and L2-resident; input rows live in shared memory.
template <int kRows>
__global__ void __launch_bounds__(256) row_lse_tab_kernel(int R, int M, int N,
                                                          const double* __restrict__ in,
                                                          const double* __restrict__ tab,
                                                          double* __restrict__ out, int transpose,
                                                          const int* stop) {
    extern __shared__ double rows[];   // [kRows][M]
    if (stop && *stop) return;
    const int r0 = blockIdx.x * kRows;
    const int nr = min(kRows, R - r0);
    for (int i = threadIdx.x; i < kRows * M; i += blockDim.x) {
        const int q = i / M, m = i - q * M;
        rows[i] = q < nr ? in[(int64_t)(r0 + q) * M + m] : kNegInf;
    }
    __syncthreads();
    const int n = blockIdx.y * blockDim.x + threadIdx.x;
    if (n >= N) return;
    double mx[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) mx[q] = kNegInf;
    for (int m = 0; m < M; ++m) {
        const double t = __ldg(tab + (int64_t)m * N + n);
#pragma unroll
        for (int q = 0; q < kRows; ++q) mx[q] = fmax(mx[q], rows[q * M + m] + t);
    }
    double sm[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) sm[q] = 0.0;
    for (int m = 0; m < M; ++m) {
        const double t = __ldg(tab + (int64_t)m * N + n);
#pragma unroll
        for (int q = 0; q < kRows; ++q) {
            const double u = rows[q * M + m] + t - mx[q];
            if (u > -760.0) sm[q] += exp(u);
        }
    }
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        if (q >= nr) break;
        const int r = r0 + q;
        const double res = isfinite(mx[q]) ? log(sm[q]) + mx[q] : kNegInf;
        if (transpose) out[(int64_t)n * R + r] = res;
        else out[(int64_t)r * N + n] = res;
    }
}

// divide == 0: out = a*s + b;  divide == 1: out = a/s + b  (b may be NULL)
__global__ void axpb_kernel(int64_t n, const double* a, double s, const double* b, double* out,
                            int divide, const int* stop = nullptr) {
    if (stop && *stop) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double t = divide ? a[i] / s : a[i] * s;
        out[i] = b ? t + b[i] : t;
    }
}

__global__ void newton_global_kernel(int64_t n, const double* z, double ratio, double lam,
                                     double* beta, int32_t* n_deg, const int* stop = nullptr,
                                     int* iters = nullptr, int k = 0) {
    if (stop && *stop) return;
    if (iters && blockIdx.x == 0 && threadIdx.x == 0) *iters = k;
    int cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double zz = z[i];
        if (zz > kNegInf) {
            beta[i] = -ratio * zz;
        } else {
            beta[i] = lam * kDegenerateBetaScale;
            ++cnt;
        }
    }
    if (cnt && n_deg) atomicAdd(n_deg, cnt);
}

// General per-node Y step (m may be NULL = zero background).
__global__ void newton_nodes_kernel(int64_t n, const double* z, const double* m,
                                    const double* beta0, const double* eps, const double* lam,
                                    double tol, int max_iters, double* beta, int32_t* n_deg) {
    int cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int dg = 0;
        beta[i] = newton_node(z[i], m ? m[i] : 0.0, m != nullptr, beta0 ? beta0[i] : 0.0, eps[i],
                              lam[i], tol, max_iters, &dg);
        cnt += dg;
    }
    if (cnt && n_deg) atomicAdd(n_deg, cnt);
}

constexpr int kRedBlocks = 1024;

// stage 1: per-block partial sums of up to 3 quantities, partial[q*kRedBlocks + block]
__global__ void __launch_bounds__(DD_NT) terms_kernel(int mode, int64_t n_x, int64_t n_y,
                                                      const double* a, const double* l,
                                                      const double* w, const double* b,
                                                      const double* z, const double* w2, double eps,
                                                      double lam, double* px, double* partial,
                                                      const int* stop = nullptr) {
    if (stop && *stop) return;
    __shared__ double red[DD_NW + 1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    const int64_t stride = (int64_t)gridDim.x * DD_NT;
    const int64_t t0 = blockIdx.x * (int64_t)DD_NT + threadIdx.x;
    if (mode == 0) {
        for (int64_t i = t0; i < n_x; i += stride) {
            const double mu = w[i];
            double p = 0.0;
            if (mu > 0) {
                const double al = a[i];
                const double lr = al / eps + l[i];
                p = mu * exp(lr);
                const double ref = mu * exp(-al / lam);
                s0 += p * (lr + al / lam) - p + ref;
            }
            if (px) px[i] = p;
        }
    } else if (mode == 1) {
        for (int64_t i = t0; i < n_y; i += stride) {
            const double nu = w2[i];
            s0 += nu * exp(b[i] / eps + z[i]);
            s2 += nu * (1.0 - exp(-b[i] / lam));
        }
        for (int64_t i = t0; i < n_x; i += stride) s1 += w[i] * (1.0 - exp(-a[i] / lam));
    } else if (mode == 2) {
        // KL(y | nu) with clipping at zero (a = y, w2 = nu), n_y entries
        for (int64_t i = t0; i < n_y; i += stride) {
            const double y = l ? fmax(a[i], 0.0) : a[i];
            s0 += kl_term(y, w2[i]);
        }
    }
    s0 = block_sum(s0, red);
    s1 = block_sum(s1, red);
    s2 = block_sum(s2, red);
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = s0;
        partial[kRedBlocks + blockIdx.x] = s1;
        partial[2 * kRedBlocks + blockIdx.x] = s2;
    }
}

// out[q] = sum_r in[r*width + q] in a fixed order (one block per q)
// Global Sinkhorn stopping test on the device (sinkhorn.py:361-432): the gap sum
// reduced exactly as reduce_rows_kernel does for dd_global_terms, gap = lam * sum,
// done when gap / lam <= thr (the host loop's arithmetic).  ctl_i = {done, iters},
// ctl_d = {gap}.
__global__ void __launch_bounds__(DD_NT) sk_check_kernel(const double* partial, double lam,
                                                         double thr, int* ctl_i, double* ctl_d) {
    __shared__ double red[DD_NW + 1];
    if (ctl_i[0]) return;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < kRedBlocks; r += DD_NT) s += partial[r];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
        const double gap = lam * s;
        ctl_d[0] = gap;
        if (gap / lam <= thr) ctl_i[0] = 1;
    }
}

__global__ void __launch_bounds__(DD_NT) reduce_rows_kernel(int64_t n_rows, int width,
                                                            const double* in, double* out) {
    __shared__ double red[DD_NW + 1];
    const int q = blockIdx.x;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < n_rows; r += DD_NT) s += in[r * width + q];
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[q] = s;
}

// ---- deterministic boxed gather-sum ------------------------------------------------
// out[y] = base[y] (or 0) + sum over items i in index order with y in box_i of
// scale_i * v_i[y - box_i], each product rounded before its add (no FMA), i.e.
// exactly the reference's sequential accumulation (measures.py:410-425
// assemble_y_marginal; engine.py:441-456 BlendScorer.energy_at y[ids] += th*dy).
// One CTA per Y tile: items are scanned in chunks of DD_NT; a chunk whose
// bounding box (precomputed) misses the tile is skipped; the hits of a chunk
// are compacted in index order (warp ballots) and every node of the tile
// accumulates them in that order.  No atomics: bitwise reproducible.
struct gather_items {
    int n;
    const int32_t* box;      // (o0, e0, o1, e1) at box + i*bstride
    int bstride;
    const double* vals;      // values of item i at vals + (voff ? voff[i*voff_stride] : i*vstride)
    int64_t vstride;
    const int64_t* voff;
    int voff_stride;
    const double* scale;     // nullable: plain sum
};

__device__ __forceinline__ bool item_live(const gather_items& it, int i, int4& b) {
    const int32_t* p = it.box + (int64_t)i * it.bstride;
    b = make_int4(p[0], p[1], p[2], p[3]);
    if (b.y <= 0 || b.w <= 0) return false;
    if (it.scale && it.scale[i] == 0.0) return false;
    return true;
}

__global__ void __launch_bounds__(DD_NT) chunk_bbox_kernel(gather_items it, int4* cb) {
    __shared__ int red[4][DD_NW];
    const int i = blockIdx.x * DD_NT + threadIdx.x;
    int lo0 = INT_MAX, hi0 = INT_MIN, lo1 = INT_MAX, hi1 = INT_MIN;
    int4 b;
    if (i < it.n && item_live(it, i, b)) {
        lo0 = b.x; hi0 = b.x + b.y; lo1 = b.z; hi1 = b.z + b.w;
    }
    for (int o = 16; o; o >>= 1) {
        lo0 = min(lo0, __shfl_xor_sync(0xffffffffu, lo0, o));
        hi0 = max(hi0, __shfl_xor_sync(0xffffffffu, hi0, o));
        lo1 = min(lo1, __shfl_xor_sync(0xffffffffu, lo1, o));
        hi1 = max(hi1, __shfl_xor_sync(0xffffffffu, hi1, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { red[0][w] = lo0; red[1][w] = hi0; red[2][w] = lo1; red[3][w] = hi1; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < DD_NW; ++k) {
            lo0 = min(lo0, red[0][k]); hi0 = max(hi0, red[1][k]);
            lo1 = min(lo1, red[2][k]); hi1 = max(hi1, red[3][k]);
        }
        cb[blockIdx.x] = make_int4(lo0, hi0, lo1, hi1);
    }
}

template <int TC>
__global__ void __launch_bounds__(DD_NT) box_gather_kernel(gather_items it, const int4* cb,
                                                           int nchunks, int ny0, int ny1,
                                                           const double* base, double* out) {
    constexpr int TR = DD_NT / TC;
    __shared__ int4 sbox[DD_NT];
    __shared__ int64_t soff[DD_NT];
    __shared__ double ssc[DD_NT];
    __shared__ int wcnt[DD_NW + 1];
    const int tiles1 = (ny1 + TC - 1) / TC;
    const int r0 = (blockIdx.x / tiles1) * TR, c0 = (blockIdx.x % tiles1) * TC;
    const int y0 = r0 + threadIdx.x / TC, y1 = c0 + threadIdx.x % TC;
    const bool valid = y0 < ny0 && y1 < ny1;
    const int64_t node = (int64_t)y0 * ny1 + y1;
    double acc = (valid && base) ? base[node] : 0.0;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int ch = 0; ch < nchunks; ++ch) {
        const int4 c = cb[ch];
        if (c.x >= r0 + TR || c.y <= r0 || c.z >= c0 + TC || c.w <= c0) continue;
        const int i = ch * DD_NT + threadIdx.x;
        int4 b = make_int4(0, 0, 0, 0);
        bool hit = false;
        if (i < it.n && item_live(it, i, b))
            hit = b.x < r0 + TR && b.x + b.y > r0 && b.z < c0 + TC && b.z + b.w > c0;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (l == 0) wcnt[w] = __popc(m);
        __syncthreads();
        int pre = 0, tot = 0;
        for (int k = 0; k < DD_NW; ++k) {
            pre += (k < w) ? wcnt[k] : 0;
            tot += wcnt[k];
        }
        if (hit) {
            const int pos = pre + __popc(m & ((1u << l) - 1u));
            sbox[pos] = b;
            soff[pos] = it.voff ? it.voff[(int64_t)i * it.voff_stride] : (int64_t)i * it.vstride;
            ssc[pos] = it.scale ? it.scale[i] : 1.0;
        }
        __syncthreads();
        if (valid) {
            for (int k = 0; k < tot; ++k) {
                const int4 bb = sbox[k];
                const int a0 = y0 - bb.x, a1 = y1 - bb.z;
                if (a0 >= 0 && a0 < bb.y && a1 >= 0 && a1 < bb.w) {
                    const double v = it.vals[soff[k] + (int64_t)a0 * bb.w + a1];
                    acc = it.scale ? __dadd_rn(acc, __dmul_rn(ssc[k], v)) : __dadd_rn(acc, v);
                }
            }
        }
        __syncthreads();
    }
    if (valid) out[node] = acc;
}

}  // namespace dd

// host launcher shared by dd_assemble and dd_blend_energy (cell.cu)
int dd_box_gather(int n, const int32_t* box, int bstride, const double* vals, int64_t vstride,
                  const int64_t* voff, int voff_stride, const double* scale, int ny0, int ny1,
                  const double* base, double* out, cudaStream_t st) {
    const int nchunks = (n + DD_NT - 1) / DD_NT;
    int4* cb = nullptr;
    cudaError_t e;
    static thread_local bool pool_kept = false;
    if (!pool_kept) {
        // keep freed stream-ordered allocations in the device pool (no OS round trip
        // for the per-call chunk table)
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_kept = true;
    }
    if (nchunks > 0) {
        e = cudaMallocAsync((void**)&cb, sizeof(int4) * nchunks, st);
        if (e != cudaSuccess) return dd_set_error(e);
        dd::gather_items it{n, box, bstride, vals, vstride, voff, voff_stride, scale};
        dd::chunk_bbox_kernel<<<nchunks, DD_NT, 0, st>>>(it, cb);
        e = cudaGetLastError();
        if (e != cudaSuccess) return dd_set_error(e);
    }
    dd::gather_items it{n, box, bstride, vals, vstride, voff, voff_stride, scale};
    if (ny0 == 1) {
        const int tiles = (ny1 + DD_NT - 1) / DD_NT;
        dd::box_gather_kernel<DD_NT><<<tiles, DD_NT, 0, st>>>(it, cb, nchunks, ny0, ny1, base, out);
    } else {
        const int tiles = ((ny0 + DD_NT / 32 - 1) / (DD_NT / 32)) * ((ny1 + 31) / 32);
        dd::box_gather_kernel<32><<<tiles, DD_NT, 0, st>>>(it, cb, nchunks, ny0, ny1, base, out);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return dd_set_error(e);
    if (cb) {
        e = cudaFreeAsync(cb, st);
        if (e != cudaSuccess) return dd_set_error(e);
    }
    return 0;
}

namespace dd {

// per basic cell: [transport, kl, d1_i, 0]
__global__ void __launch_bounds__(DD_NT) cell_terms_kernel(dd_geom g, dd_state s, double* pc,
                                                           const double* mask) {
    __shared__ double red[DD_NW + 1];
    const int i = blockIdx.x;
    if (mask && mask[i] == 0.0) {   // basic cell held by another rank (slab mode)
        if (threadIdx.x < 4) pc[(int64_t)i * 4 + threadIdx.x] = 0.0;
        return;
    }
    const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
    const int bs = s.block0 * s.block1;
    double p = 0.0;
    for (int t = threadIdx.x; t < bs; t += DD_NT) {
        const int a0 = t / bx[3], a1 = t - a0 * bx[3];
        const double mu = s.mu[(int64_t)(bx[0] + a0) * g.nx1 + (bx[2] + a1)];
        if (mu > 0) p += kl_term(s.x_marg[(int64_t)i * bs + t], mu);
    }
    p = block_sum(p, red);
    if (threadIdx.x == 0) {
        pc[(int64_t)i * 4 + 0] = s.transport[i];
        pc[(int64_t)i * 4 + 1] = s.kl[i];
        pc[(int64_t)i * 4 + 2] = p;
        pc[(int64_t)i * 4 + 3] = 0.0;
    }
}

// Product start (engine.py:234-257, cells.py:566-606)
__global__ void __launch_bounds__(DD_NT) product_init_kernel(dd_geom g, dd_state s,
                                                             double mu_total) {
    __shared__ double red[DD_NW + 1];
    const int i = blockIdx.x;
    const int64_t ny = (int64_t)g.ny0 * g.ny1;
    const double scale = s.basic_mass[i] / mu_total;
    const double ratio = g.nu_total / mu_total;
    double* v = s.yval + (int64_t)i * s.cap;
    double mnu = 0.0, sy1a = 0.0, sy2a = 0.0, sy1b = 0.0, sy2b = 0.0, ent = 0.0;
    for (int64_t t = threadIdx.x; t < ny; t += DD_NT) {
        const int y0 = (int)(t / g.ny1), y1 = (int)(t - (int64_t)y0 * g.ny1);
        const double nu = s.nu[t];
        const double val = nu * scale;
        v[t] = val;
        mnu += val;
        const double ya = g.y_org0 + g.y_dx * (double)y0;
        const double yb = g.y_org1 + g.y_dx * (double)y1;
        sy1a += val * ya;
        sy2a += val * (ya * ya);
        sy1b += val * yb;
        sy2b += val * (yb * yb);
        ent += xlogy(val, val / nu);
    }
    mnu = block_sum(mnu, red);
    sy1a = block_sum(sy1a, red);
    sy2a = block_sum(sy2a, red);
    sy1b = block_sum(sy1b, red);
    sy2b = block_sum(sy2b, red);
    ent = block_sum(ent, red);
    const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
    const int bs = s.block0 * s.block1;
    double mmu = 0.0, sx1a = 0.0, sx2a = 0.0, sx1b = 0.0, sx2b = 0.0;
    for (int t = threadIdx.x; t < bs; t += DD_NT) {
        const int a0 = t / bx[3], a1 = t - a0 * bx[3];
        const int r = bx[0] + a0, q = bx[2] + a1;
        const double mu = s.mu[(int64_t)r * g.nx1 + q];
        s.x_marg[(int64_t)i * bs + t] = mu > 0 ? mu * ratio : 0.0;
        if (mu > 0) {
            const double xa = g.x_org0 + g.x_dx * (double)r;
            const double xb = g.x_org1 + g.x_dx * (double)q;
            mmu += mu;
            sx1a += mu * xa;
            sx2a += mu * (xa * xa);
            sx1b += mu * xb;
            sx2b += mu * (xb * xb);
        }
    }
    mmu = block_sum(mmu, red);
    sx1a = block_sum(sx1a, red);
    sx2a = block_sum(sx2a, red);
    sx1b = block_sum(sx1b, red);
    sx2b = block_sum(sx2b, red);
    if (threadIdx.x == 0) {
        s.ybox[(int64_t)i * 4 + 0] = 0;
        s.ybox[(int64_t)i * 4 + 1] = g.ny0;
        s.ybox[(int64_t)i * 4 + 2] = 0;
        s.ybox[(int64_t)i * 4 + 3] = g.ny1;
        if (mnu == 0.0) {
            s.transport[i] = 0.0;
            s.kl[i] = mmu * g.nu_total;
        } else {
            double tr = 0.0;
            tr += sx2a * mnu - 2.0 * sx1a * sy1a + mmu * sy2a;
            tr += sx2b * mnu - 2.0 * sx1b * sy1b + mmu * sy2b;
            tr /= mmu;
            s.transport[i] = tr;
            s.kl[i] = ent - mnu * log(mmu) - mnu + mmu * g.nu_total;
        }
    }
}

// Plan cut of global duals along one basic cell (engine.py:307-322).
// pass 0: statistics + bounding box; pass 1: write truncated values.
__global__ void __launch_bounds__(DD_NT) cut_plan_kernel(dd_geom g, dd_state s,
                                                         const double* alpha, const double* beta,
                                                         double trunc, double* trunc_out,
                                                         int32_t* boxes_out) {
    __shared__ double red[DD_NW + 1];
    __shared__ int redi[DD_NW + 1];
    __shared__ double xs_a[256], xs_mu[256], xs_c0[256], xs_c1[256];
    __shared__ int xs_t[256];
    __shared__ int n_sh;
    const int i = blockIdx.x;
    const int32_t* bx = s.basic_xbox + (int64_t)i * 4;
    const int bs = s.block0 * s.block1;
    const double eps = g.eps;
    if (threadIdx.x == 0) {
        int n = 0;
        for (int t = 0; t < bs; ++t) {
            const int a0 = t / bx[3], a1 = t - a0 * bx[3];
            const int r = bx[0] + a0, q = bx[2] + a1;
            const int64_t id = (int64_t)r * g.nx1 + q;
            const double mu = s.mu[id];
            if (mu > 0) {
                xs_a[n] = alpha[id];
                xs_mu[n] = mu;
                xs_c0[n] = g.x_org0 + g.x_dx * (double)r;
                xs_c1[n] = g.x_org1 + g.x_dx * (double)q;
                xs_t[n] = t;
                ++n;
            }
        }
        n_sh = n;
    }
    __syncthreads();
    const int nxn = n_sh;
    const int64_t ny = (int64_t)g.ny0 * g.ny1;
    // num < -750 eps  =>  num / eps < -749.9...  =>  exp(num / eps) == 0 exactly
    const double zero_cut = -750.0 * eps;
    double xacc[64];
    for (int k = 0; k < 64; ++k) xacc[k] = 0.0;
    double mass = 0.0, tr = 0.0, klp = 0.0, rem = 0.0;
    int rmin = 0x7fffffff, rmax = -1, cmin = 0x7fffffff, cmax = -1;
    for (int64_t t = threadIdx.x; t < ny; t += DD_NT) {
        const int y0 = (int)(t / g.ny1), y1 = (int)(t - (int64_t)y0 * g.ny1);
        const double yc0 = g.y_org0 + g.y_dx * (double)y0;
        const double yc1 = g.y_org1 + g.y_dx * (double)y1;
        const double nu = s.nu[t];
        const double bt = beta[t];
        double col = 0.0;
        for (int k = 0; k < nxn; ++k) {
            const double d0 = xs_c0[k] - yc0, d1 = xs_c1[k] - yc1;
            const double cost = d0 * d0 + d1 * d1;
            const double num = xs_a[k] + bt - cost;
            // exp(num/eps) is exactly 0 in double below -745.14: such terms add
            // exact zeros to every sum, so the division and exp are skipped
            if (num < zero_cut) continue;
            const double lr = num / eps;
            const double blk = exp(lr) * xs_mu[k] * nu;
            col += blk;
            tr += cost * blk;
            klp += blk * lr;
            if (k < 64) xacc[k] += blk;
        }
        mass += col;
        if (col >= trunc) {
            rmin = min(rmin, y0); rmax = max(rmax, y0);
            cmin = min(cmin, y1); cmax = max(cmax, y1);
        } else {
            rem += col;
        }
    }
    mass = block_sum(mass, red);
    tr = block_sum(tr, red);
    klp = block_sum(klp, red);
    rem = block_sum(rem, red);
    rmin = block_min_i(rmin, redi);
    rmax = block_max_i(rmax, redi);
    cmin = block_min_i(cmin, redi);
    cmax = block_max_i(cmax, redi);
    // zero the block first: retained nodes are a subsequence, so zeroing slot k
    // while scattering xs_t[k] >= k would wipe earlier writes
    for (int k = threadIdx.x; k < bs; k += DD_NT) s.x_marg[(int64_t)i * bs + k] = 0.0;
    __syncthreads();
    for (int k = 0; k < nxn; ++k) {
        const double v = block_sum(xacc[k], red);
        if (threadIdx.x == 0) s.x_marg[(int64_t)i * bs + xs_t[k]] = v;
    }
    __syncthreads();
    int ne0 = 0, ne1 = 0;
    if (rmax >= 0) { ne0 = rmax - rmin + 1; ne1 = cmax - cmin + 1; }
    if (threadIdx.x == 0) {
        double mmu = 0.0;
        for (int k = 0; k < nxn; ++k) mmu += xs_mu[k];
        s.transport[i] = tr;
        s.kl[i] = klp - mass + mmu * g.nu_total;
        trunc_out[i] = rem;
        int32_t* ob = boxes_out + (int64_t)i * 4;
        if (rmax >= 0) { ob[0] = rmin; ob[1] = ne0; ob[2] = cmin; ob[3] = ne1; }
        else { ob[0] = 0; ob[1] = 0; ob[2] = 0; ob[3] = 0; }
    }
    if (s.yval == nullptr || (int64_t)ne0 * ne1 > s.cap) return;
    // pass 1: values inside the box
    double* v = s.yval + (int64_t)i * s.cap;
    for (int t = threadIdx.x; t < ne0 * ne1; t += DD_NT) {
        const int a0 = t / ne1, a1 = t - a0 * ne1;
        const int y0 = rmin + a0, y1 = cmin + a1;
        const int64_t id = (int64_t)y0 * g.ny1 + y1;
        const double yc0 = g.y_org0 + g.y_dx * (double)y0;
        const double yc1 = g.y_org1 + g.y_dx * (double)y1;
        const double nu = s.nu[id];
        const double bt = beta[id];
        double col = 0.0;
        for (int k = 0; k < nxn; ++k) {
            const double d0 = xs_c0[k] - yc0, d1 = xs_c1[k] - yc1;
            const double cost = d0 * d0 + d1 * d1;
            const double num = xs_a[k] + bt - cost;
            if (num < zero_cut) continue;
            col += exp(num / eps) * xs_mu[k] * nu;
        }
        v[t] = col >= trunc ? col : 0.0;
    }
    if (threadIdx.x < 4) s.ybox[(int64_t)i * 4 + threadIdx.x] = boxes_out[(int64_t)i * 4 + threadIdx.x];
}

// Seed cell duals of one partition from global duals.
__global__ void __launch_bounds__(DD_NT) seed_duals_kernel(dd_geom g, dd_state s, int nw0, int nw1,
                                                           const int32_t* xbox, const int32_t* ybox,
                                                           const double* alpha, const double* beta) {
    const int j = blockIdx.x;
    const int32_t* xb = xbox + (int64_t)j * 4;
    const int32_t* yb = ybox + (int64_t)j * 4;
    const int nx = nw0 * nw1;
    for (int x = threadIdx.x; x < nx; x += DD_NT) {
        const int x0 = x / nw1, x1 = x - x0 * nw1;
        const int r = xb[0] + x0, q = xb[2] + x1;
        double a = 0.0;
        if (r >= 0 && r < g.nx0 && q >= 0 && q < g.nx1) a = alpha[(int64_t)r * g.nx1 + q];
        s.d_alpha[(int64_t)j * nx + x] = a;
    }
    const int ny = yb[1] * yb[3];
    for (int y = threadIdx.x; y < ny; y += DD_NT) {
        const int y0 = y / yb[3], y1 = y - y0 * yb[3];
        s.d_beta[(int64_t)j * s.d_cap + y] = beta[(int64_t)(yb[0] + y0) * g.ny1 + (yb[2] + y1)];
    }
    if (threadIdx.x < 4) s.d_box[(int64_t)j * 4 + threadIdx.x] = yb[threadIdx.x];
    if (threadIdx.x == 0) s.d_has[j] = 1;
}

// Multiscale refinement of one fine basic cell j from its coarse parent
// (SPEC multiscale.refine_plan): nu_j(yf) = f_j nu_i(yf/2) nu_f(yf)/nu_c(yf/2),
// f_j = mu_f(X_j)/mu_c(X_i); truncated at `trunc`; product-plan fragments.
struct RefineArgs {
    const int32_t* parent;     // [n_fine] coarse cell id
    const int32_t* cbox;       // coarse Y boxes
    const double* cval;        // coarse slots
    int64_t ccap;
    const double* cmass;       // coarse basic masses
    const double* nu_c;        // coarse nu grid
    int32_t cny1;              // coarse Y dim 1
    double trunc;
    double* trunc_out;         // [n_fine]
};

__global__ void __launch_bounds__(DD_NT) refine_kernel(dd_geom g, dd_state s, RefineArgs a) {
    __shared__ double red[DD_NW + 1];
    __shared__ int redi[DD_NW + 1];
    const int j = blockIdx.x;
    const int i = a.parent[j];
    const int32_t* cb = a.cbox + (int64_t)i * 4;
    const double* cv = a.cval + (int64_t)i * a.ccap;
    const double f = s.basic_mass[j] / a.cmass[i];
    const int fo0 = 2 * cb[0], fe0 = 2 * cb[1], fo1 = 2 * cb[2], fe1 = 2 * cb[3];
    const int n = fe0 * fe1;
    // pass 0: bounding box and removed mass
    int rmin = 0x7fffffff, rmax = -1, cmin = 0x7fffffff, cmax = -1;
    double rem = 0.0;
    for (int t = threadIdx.x; t < n; t += DD_NT) {
        const int a0 = t / fe1, a1 = t - a0 * fe1;
        const int yf0 = fo0 + a0, yf1 = fo1 + a1;
        const int yc0 = yf0 >> 1, yc1 = yf1 >> 1;
        const double vc = cv[(int64_t)(yc0 - cb[0]) * cb[3] + (yc1 - cb[2])];
        const double v = f * vc * (s.nu[(int64_t)yf0 * g.ny1 + yf1] / a.nu_c[(int64_t)yc0 * a.cny1 + yc1]);
        if (v >= a.trunc) {
            rmin = min(rmin, a0); rmax = max(rmax, a0); cmin = min(cmin, a1); cmax = max(cmax, a1);
        } else {
            rem += v;
        }
    }
    rmin = block_min_i(rmin, redi);
    rmax = block_max_i(rmax, redi);
    cmin = block_min_i(cmin, redi);
    cmax = block_max_i(cmax, redi);
    rem = block_sum(rem, red);
    int ne0 = 0, ne1 = 0;
    if (rmax >= 0) { ne0 = rmax - rmin + 1; ne1 = cmax - cmin + 1; }
    double* out = s.yval + (int64_t)j * s.cap;
    double mnu = 0.0, sy1a = 0.0, sy2a = 0.0, sy1b = 0.0, sy2b = 0.0, ent = 0.0;
    for (int t = threadIdx.x; t < ne0 * ne1; t += DD_NT) {
        const int a0 = t / ne1, a1 = t - a0 * ne1;
        const int yf0 = fo0 + rmin + a0, yf1 = fo1 + cmin + a1;
        const int yc0 = yf0 >> 1, yc1 = yf1 >> 1;
        const double vc = cv[(int64_t)(yc0 - cb[0]) * cb[3] + (yc1 - cb[2])];
        const double nu = s.nu[(int64_t)yf0 * g.ny1 + yf1];
        double v = f * vc * (nu / a.nu_c[(int64_t)yc0 * a.cny1 + yc1]);
        v = v >= a.trunc ? v : 0.0;
        out[t] = v;
        mnu += v;
        const double ya = g.y_org0 + g.y_dx * (double)yf0;
        const double yb = g.y_org1 + g.y_dx * (double)yf1;
        sy1a += v * ya;
        sy2a += v * (ya * ya);
        sy1b += v * yb;
        sy2b += v * (yb * yb);
        ent += xlogy(v, v / nu);
    }
    mnu = block_sum(mnu, red);
    sy1a = block_sum(sy1a, red);
    sy2a = block_sum(sy2a, red);
    sy1b = block_sum(sy1b, red);
    sy2b = block_sum(sy2b, red);
    ent = block_sum(ent, red);
    const int32_t* bx = s.basic_xbox + (int64_t)j * 4;
    const int bs = s.block0 * s.block1;
    double mmu = 0.0, sx1a = 0.0, sx2a = 0.0, sx1b = 0.0, sx2b = 0.0;
    for (int t = threadIdx.x; t < bs; t += DD_NT) {
        const int a0 = t / bx[3], a1 = t - a0 * bx[3];
        const int r = bx[0] + a0, q = bx[2] + a1;
        const double mu = s.mu[(int64_t)r * g.nx1 + q];
        if (mu > 0) {
            const double xa = g.x_org0 + g.x_dx * (double)r;
            const double xb = g.x_org1 + g.x_dx * (double)q;
            mmu += mu;
            sx1a += mu * xa;
            sx2a += mu * (xa * xa);
            sx1b += mu * xb;
            sx2b += mu * (xb * xb);
        }
    }
    mmu = block_sum(mmu, red);
    sx1a = block_sum(sx1a, red);
    sx2a = block_sum(sx2a, red);
    sx1b = block_sum(sx1b, red);
    sx2b = block_sum(sx2b, red);
    for (int t = threadIdx.x; t < bs; t += DD_NT) {
        const int a0 = t / bx[3], a1 = t - a0 * bx[3];
        const double mu = s.mu[(int64_t)(bx[0] + a0) * g.nx1 + (bx[2] + a1)];
        s.x_marg[(int64_t)j * bs + t] = mu > 0 ? mu * (mnu / mmu) : 0.0;
    }
    if (threadIdx.x == 0) {
        int32_t* ob = s.ybox + (int64_t)j * 4;
        if (rmax >= 0) { ob[0] = fo0 + rmin; ob[1] = ne0; ob[2] = fo1 + cmin; ob[3] = ne1; }
        else { ob[0] = 0; ob[1] = 0; ob[2] = 0; ob[3] = 0; }
        a.trunc_out[j] = rem;
        if (mnu == 0.0) {
            s.transport[j] = 0.0;
            s.kl[j] = mmu * g.nu_total;
        } else {
            double tr = sx2a * mnu - 2.0 * sx1a * sy1a + mmu * sy2a;
            tr += sx2b * mnu - 2.0 * sx1b * sy1b + mmu * sy2b;
            s.transport[j] = tr / mmu;
            s.kl[j] = ent - mnu * log(mmu) - mnu + mmu * g.nu_total;
        }
    }
}


// Prolongation of a coarse cell-centred grid field to the fine grid (x2 per
// axis): bilinear in the coarse node positions, constant beyond the outer
// coarse centres.  Axes of length 1 (1D embedding) are copied.
__global__ void prolong_kernel(int nf0, int nf1, int nc0, int nc1, const double* c, double* f) {
    const int64_t n = (int64_t)nf0 * nf1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(t / nf1), q = (int)(t - (int64_t)r * nf1);
        int i0 = 0, i1 = 0, j0 = 0, j1 = 0;
        double w0 = 0.0, w1 = 0.0;
        if (nc0 > 1) {
            const double p = 0.5 * (double)r - 0.25;   // coarse index of fine centre r
            const double pc = fmin(fmax(p, 0.0), (double)(nc0 - 1));
            i0 = min((int)floor(pc), nc0 - 2);
            i1 = i0 + 1;
            w0 = pc - (double)i0;
        }
        if (nc1 > 1) {
            const double p = 0.5 * (double)q - 0.25;
            const double pc = fmin(fmax(p, 0.0), (double)(nc1 - 1));
            j0 = min((int)floor(pc), nc1 - 2);
            j1 = j0 + 1;
            w1 = pc - (double)j0;
        }
        const double c00 = c[(int64_t)i0 * nc1 + j0], c01 = c[(int64_t)i0 * nc1 + j1];
        const double c10 = c[(int64_t)i1 * nc1 + j0], c11 = c[(int64_t)i1 * nc1 + j1];
        f[t] = (1.0 - w0) * ((1.0 - w1) * c00 + w1 * c01) + w0 * ((1.0 - w1) * c10 + w1 * c11);
    }
}

}  // namespace dd

// ---- host wrappers ------------------------------------------------------------------

static int grid_blocks(int64_t n) {
    int64_t b = (n + DD_NT - 1) / DD_NT;
    if (b > 4096) b = 4096;
    if (b < 1) b = 1;
    return (int)b;
}

static int row_lse_apply(int R, int M, int N, const double* in, const double* tab, double* out,
                         int transpose, const int* stop, cudaStream_t st) {
    // threads per block: the outputs of one row (rounded to warps, <= 256)
    const int nt = std::min(256, (N + 31) / 32 * 32);
    auto launch = [&](auto kern, int rows) -> int {
        const size_t smem = (size_t)rows * M * sizeof(double);
        if (smem > 48 * 1024) {
            cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)smem);
            if (e2 != cudaSuccess) return dd_set_error(e2);
        }
        dim3 grid((R + rows - 1) / rows, (N + nt - 1) / nt);
        kern<<<grid, nt, smem, st>>>(R, M, N, in, tab, out, transpose, stop);
        return dd_set_error(cudaGetLastError());
    };
    // rows per block: as many as keep >= 2 blocks per SM (148 SMs) and fit 200 KB of
    // shared memory; small grids get one row per block (parallelism over reuse)
    const int64_t col_blocks = (N + nt - 1) / nt;
    auto fits = [&](int rows) {
        return (size_t)rows * M * sizeof(double) <= 200 * 1024 &&
               ((R + rows - 1) / rows) * col_blocks >= 2 * 148;
    };
    if (fits(8)) return launch(dd::row_lse_tab_kernel<8>, 8);
    if (fits(2)) return launch(dd::row_lse_tab_kernel<2>, 2);
    return launch(dd::row_lse_tab_kernel<1>, 1);
}

static int neg_sq_table(int M, int N, double p0, double pd, double q0, double qd, double eps,
                        double* tab, cudaStream_t st) {
    const int64_t nt = (int64_t)M * N;
    dd::neg_sq_table_kernel<<<grid_blocks(nt), DD_NT, 0, st>>>(M, N, p0, pd, q0, qd, eps, tab);
    return dd_set_error(cudaGetLastError());
}

static int row_lse(int R, int M, int N, const double* in, double p0, double pd, double q0,
                   double qd, double eps, double* out, int transpose, double* tab,
                   cudaStream_t st) {
    const int rc = neg_sq_table(M, N, p0, pd, q0, qd, eps, tab, st);
    if (rc) return rc;
    return row_lse_apply(R, M, N, in, tab, out, transpose, nullptr, st);
}

extern "C" int dd_grid_lse(const dd_geom* g, const double* v, double* out, int to_x, double* work,
                           void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t mid = std::max((int64_t)g->ny0 * g->nx1, (int64_t)g->nx0 * g->ny1);
    double* tab = work + mid;   // axis table of the current stage (reused by both)
    int rc;
    if (to_x) {
        // stage A: rows y0 of v (over y1) -> x1, stored transposed [nx1][ny0]
        rc = row_lse(g->ny0, g->ny1, g->nx1, v, g->x_org1, g->x_dx, g->y_org1, g->y_dx, g->eps,
                     work, 1, tab, st);
        if (rc) return rc;
        // stage B: rows x1 (over y0) -> x0, stored transposed [nx0][nx1]
        return row_lse(g->nx1, g->ny0, g->nx0, work, g->x_org0, g->x_dx, g->y_org0, g->y_dx,
                       g->eps, out, 1, tab, st);
    }
    rc = row_lse(g->nx0, g->nx1, g->ny1, v, g->y_org1, g->y_dx, g->x_org1, g->x_dx, g->eps, work,
                 1, tab, st);
    if (rc) return rc;
    return row_lse(g->ny1, g->nx0, g->ny0, work, g->y_org0, g->y_dx, g->x_org0, g->x_dx, g->eps,
                   out, 1, tab, st);
}

extern "C" int64_t dd_sinkhorn_ws(const dd_geom* g) {
    const int64_t mid = std::max((int64_t)g->ny0 * g->nx1, (int64_t)g->nx0 * g->ny1);
    return mid + 2 * ((int64_t)g->nx1 * g->ny1 + (int64_t)g->nx0 * g->ny0) + 5 * 1024;
}

// n_iters iterations k = k0 .. k0+n_iters-1 of the global unbalanced Sinkhorn with
// zero background (sinkhorn.py:361-432), enqueued without host synchronisation:
// the stopping test runs on the device and every later kernel of the chunk exits at
// once after it fires.  Same operations, in the same order, as the host loop in
// sinkhorn.sinkhorn_solve (gap at the top of iteration k >= 2 from the X sweep the
// next alpha reuses; the loop always ends after a Y half-step).
extern "C" int dd_sinkhorn_run(const dd_geom* g, double* alpha, double* beta, const double* mu,
                               const double* log_mu, const double* log_nu, double* L, double* z,
                               double* bv, double* av, double* px, double* work, int* ctl_i,
                               double* ctl_d, double thr, int k0, int n_iters, int tables_ready,
                               void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nx = (int64_t)g->nx0 * g->nx1, ny = (int64_t)g->ny0 * g->ny1;
    const int64_t mid = std::max((int64_t)g->ny0 * g->nx1, (int64_t)g->nx0 * g->ny1);
    double* tmid = work;
    double* tXa = work + mid;                               // [ny1][nx1]
    double* tXb = tXa + (int64_t)g->nx1 * g->ny1;           // [ny0][nx0]
    double* tYa = tXb + (int64_t)g->nx0 * g->ny0;           // [nx1][ny1]
    double* tYb = tYa + (int64_t)g->nx1 * g->ny1;           // [nx0][ny0]
    double* partial = tYb + (int64_t)g->nx0 * g->ny0;       // 3 * kRedBlocks
    const double eps = g->eps, lam = g->lam;
    const double ratio = eps * lam / (eps + lam);
    int rc;
    if (!tables_ready) {
        if ((rc = neg_sq_table(g->ny1, g->nx1, g->x_org1, g->x_dx, g->y_org1, g->y_dx, eps, tXa, st))) return rc;
        if ((rc = neg_sq_table(g->ny0, g->nx0, g->x_org0, g->x_dx, g->y_org0, g->y_dx, eps, tXb, st))) return rc;
        if ((rc = neg_sq_table(g->nx1, g->ny1, g->y_org1, g->y_dx, g->x_org1, g->x_dx, eps, tYa, st))) return rc;
        if ((rc = neg_sq_table(g->nx0, g->ny0, g->y_org0, g->y_dx, g->x_org0, g->x_dx, eps, tYb, st))) return rc;
    }
    const int* stop = ctl_i;
    for (int k = k0; k < k0 + n_iters; ++k) {
        dd::axpb_kernel<<<grid_blocks(ny), DD_NT, 0, st>>>(ny, beta, eps, log_nu, bv, 1, stop);
        if ((rc = row_lse_apply(g->ny0, g->ny1, g->nx1, bv, tXa, tmid, 1, stop, st))) return rc;
        if ((rc = row_lse_apply(g->nx1, g->ny0, g->nx0, tmid, tXb, L, 1, stop, st))) return rc;
        if (k >= 2) {
            dd::terms_kernel<<<dd::kRedBlocks, DD_NT, 0, st>>>(0, nx, 0, alpha, L, mu, nullptr,
                                                              nullptr, nullptr, eps, lam, px,
                                                              partial, stop);
            dd::sk_check_kernel<<<1, DD_NT, 0, st>>>(partial, lam, thr, ctl_i, ctl_d);
        }
        dd::axpb_kernel<<<grid_blocks(nx), DD_NT, 0, st>>>(nx, L, -ratio, nullptr, alpha, 0, stop);
        dd::axpb_kernel<<<grid_blocks(nx), DD_NT, 0, st>>>(nx, alpha, eps, log_mu, av, 1, stop);
        if ((rc = row_lse_apply(g->nx0, g->nx1, g->ny1, av, tYa, tmid, 1, stop, st))) return rc;
        if ((rc = row_lse_apply(g->ny1, g->nx0, g->ny0, tmid, tYb, z, 1, stop, st))) return rc;
        dd::newton_global_kernel<<<grid_blocks(ny), DD_NT, 0, st>>>(ny, z, ratio, lam, beta,
                                                                    nullptr, stop, ctl_i + 1, k);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return dd_set_error(e);
    }
    return 0;
}

// Library-internal (vol.cu, the three-axis device loop): the element-wise pieces of one
// global Sinkhorn iteration, with the device stop flag of dd_sinkhorn_run.
int dd_sk_axpb(int64_t n, const double* a, double s, const double* b, double* out, int divide,
               const int* stop, cudaStream_t st) {
    dd::axpb_kernel<<<grid_blocks(n), DD_NT, 0, st>>>(n, a, s, b, out, divide, stop);
    return dd_set_error(cudaGetLastError());
}

int dd_sk_gap(int64_t nx, const double* alpha, const double* L, const double* mu, double eps,
              double lam, double* px, double* partial, double thr, int* ctl_i, double* ctl_d,
              cudaStream_t st) {
    dd::terms_kernel<<<dd::kRedBlocks, DD_NT, 0, st>>>(0, nx, 0, alpha, L, mu, nullptr, nullptr,
                                                      nullptr, eps, lam, px, partial, ctl_i);
    dd::sk_check_kernel<<<1, DD_NT, 0, st>>>(partial, lam, thr, ctl_i, ctl_d);
    return dd_set_error(cudaGetLastError());
}

int dd_sk_newton(int64_t ny, const double* z, double ratio, double lam, double* beta, int* ctl_i,
                 int k, cudaStream_t st) {
    dd::newton_global_kernel<<<grid_blocks(ny), DD_NT, 0, st>>>(ny, z, ratio, lam, beta, nullptr,
                                                                ctl_i, ctl_i + 1, k);
    return dd_set_error(cudaGetLastError());
}

int64_t dd_sk_partial_doubles() { return 3 * (int64_t)dd::kRedBlocks; }

extern "C" int dd_axpb(int64_t n, const double* a, double s, const double* b, double* out,
                       int divide, void* stream) {
    dd::axpb_kernel<<<grid_blocks(n), DD_NT, 0, (cudaStream_t)stream>>>(n, a, s, b, out, divide);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_newton_global(int64_t n, const double* z, double ratio, double lam, double* beta,
                                int32_t* n_deg, void* stream) {
    dd::newton_global_kernel<<<grid_blocks(n), DD_NT, 0, (cudaStream_t)stream>>>(n, z, ratio, lam,
                                                                                 beta, n_deg);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_newton_nodes(int64_t n, const double* z, const double* m, const double* beta0,
                               const double* eps, const double* lam, double tol, int max_iters,
                               double* beta, int32_t* n_deg, void* stream) {
    dd::newton_nodes_kernel<<<grid_blocks(n), DD_NT, 0, (cudaStream_t)stream>>>(
        n, z, m, beta0, eps, lam, tol, max_iters, beta, n_deg);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_reduce_rows(int64_t n_rows, int width, const double* in, double* out,
                              void* stream) {
    dd::reduce_rows_kernel<<<width, DD_NT, 0, (cudaStream_t)stream>>>(n_rows, width, in, out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_global_terms(int mode, int64_t n_x, int64_t n_y, const double* a,
                               const double* l, const double* w, const double* b, const double* z,
                               const double* w2, double eps, double lam, double* px,
                               double* partial, double* sums, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    dd::terms_kernel<<<dd::kRedBlocks, DD_NT, 0, st>>>(mode, n_x, n_y, a, l, w, b, z, w2, eps, lam,
                                                      px, partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dd_set_error(e);
    // partial is [3][kRedBlocks] -> sums[0..2]: view it as rows of width 1 per quantity
    for (int q = 0; q < 3; ++q) {
        dd::reduce_rows_kernel<<<1, DD_NT, 0, st>>>(dd::kRedBlocks, 1, partial + q * dd::kRedBlocks,
                                                   sums + q);
    }
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_grid_kl(int64_t n, const double* y, const double* nu, int clip, double* partial,
                          double* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    dd::terms_kernel<<<dd::kRedBlocks, DD_NT, 0, st>>>(2, 0, n, y, clip ? y : nullptr, nullptr,
                                                      nullptr, nullptr, nu, 1.0, 1.0, nullptr,
                                                      partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dd_set_error(e);
    dd::reduce_rows_kernel<<<1, DD_NT, 0, st>>>(dd::kRedBlocks, 1, partial, out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_assemble(const dd_geom* g, const dd_state* s, double* out, void* stream) {
    return dd_box_gather(s->n_basic, s->ybox, 4, s->yval, s->cap, nullptr, 0, nullptr, g->ny0,
                         g->ny1, nullptr, out, (cudaStream_t)stream);
}

extern "C" int dd_assemble_masked(const dd_geom* g, const dd_state* s, const double* mask,
                                  double* out, void* stream) {
    // mask entries are exactly 1 or 0: 1 * v is v, 0 skips the cell
    return dd_box_gather(s->n_basic, s->ybox, 4, s->yval, s->cap, nullptr, 0, mask, g->ny0,
                         g->ny1, nullptr, out, (cudaStream_t)stream);
}

extern "C" int dd_energy_terms_masked(const dd_geom* g, const dd_state* s, const double* y,
                                      const double* mask, double* partial, double* sums,
                                      void* stream);

extern "C" int dd_energy_terms(const dd_geom* g, const dd_state* s, const double* y,
                               double* partial, double* sums, void* stream) {
    return dd_energy_terms_masked(g, s, y, nullptr, partial, sums, stream);
}

extern "C" int dd_energy_terms_masked(const dd_geom* g, const dd_state* s, const double* y,
                                      const double* mask, double* partial, double* sums,
                                      void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    double* pc = partial + 4096;
    dd::cell_terms_kernel<<<s->n_basic, DD_NT, 0, st>>>(*g, *s, pc, mask);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dd_set_error(e);
    int rc = dd_reduce_rows(s->n_basic, 4, pc, sums, stream);
    if (rc) return rc;
    return dd_grid_kl((int64_t)g->ny0 * g->ny1, y, s->nu, 0, partial, sums + 3, stream);
}

extern "C" int dd_product_init(const dd_geom* g, const dd_state* s, double mu_total, void* stream) {
    dd::product_init_kernel<<<s->n_basic, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, mu_total);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_cut_plan(const dd_geom* g, const dd_state* s, const double* alpha,
                           const double* beta, double trunc, double* trunc_out, int32_t* boxes_out,
                           void* stream) {
    if (s->block0 * s->block1 > 64) return -1000;
    dd::cut_plan_kernel<<<s->n_basic, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, alpha, beta, trunc,
                                                                       trunc_out, boxes_out);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_seed_duals(const dd_geom* g, const dd_state* s, int n_comp, int nw0, int nw1,
                             const int32_t* xbox, const int32_t* ybox, const double* alpha,
                             const double* beta, void* stream) {
    if (n_comp <= 0) return 0;
    dd::seed_duals_kernel<<<n_comp, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, nw0, nw1, xbox, ybox,
                                                                      alpha, beta);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_refine(const dd_geom* g, const dd_state* s, const int32_t* parent,
                         const int32_t* cbox, const double* cval, int64_t ccap, const double* cmass,
                         const double* nu_c, int cny1, double trunc, double* trunc_out,
                         void* stream) {
    if (s->n_basic <= 0) return 0;
    dd::RefineArgs a{parent, cbox, cval, ccap, cmass, nu_c, cny1, trunc, trunc_out};
    dd::refine_kernel<<<s->n_basic, DD_NT, 0, (cudaStream_t)stream>>>(*g, *s, a);
    return dd_set_error(cudaGetLastError());
}

extern "C" int dd_prolong(int nf0, int nf1, int nc0, int nc1, const double* coarse, double* fine,
                          void* stream) {
    const int64_t n = (int64_t)nf0 * nf1;
    dd::prolong_kernel<<<grid_blocks(n), DD_NT, 0, (cudaStream_t)stream>>>(nf0, nf1, nc0, nc1,
                                                                          coarse, fine);
    return dd_set_error(cudaGetLastError());
}

