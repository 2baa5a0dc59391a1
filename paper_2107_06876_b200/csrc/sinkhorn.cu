// Log-stabilised Sinkhorn over the bucket-blocked operators
// (sinkhorn.cpp:104-188, operator.cpp:123-224).
//
// One iteration = the reference's s-update, K^T application, t-update, K
// application and marginal error (sinkhorn.cpp:149-168). On the device it is a
// fixed sequence of kernels, all enqueued ahead and gated by a device-side
// `done` flag, so the host never waits inside the loop:
//   col side  : [band blocks: K_sp^T / Delta^T over each bucket] -> col finalize
//               (low-rank W^T mid, positivity, log t = log q - K^T(log s),
//               finiteness, and - LCN - the partial W tt of the next half)
//               -> low-rank reduce (global shift H_t, mid_t = W tt)
//   row side  : [band blocks] -> row finalize (U mid, kt, row marginal, err
//               partial, next log s, partial U^T ss) -> iteration end
//               (err, convergence, error precedence, next shift H_s).
// Low-rank shifts: the reference shifts by the global max of the input log
// vector (operator.cpp:147-151); here each warp keeps a running max with
// online rescaling and the reduce rescales block partials to the global max,
// which is the same product in exact arithmetic and needs no extra pass.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "op.cuh"

namespace lcnb {

namespace {

enum : unsigned {
    F_LOGS = 1u,      // next log s non-finite
    F_LOGT = 2u,      // log t non-finite
    F_NEG_ROW = 4u,   // K(log t): y <= 0
    F_NYS_ROW = 8u,   // K(log t): nystrom part <= 0 (checked only for positive input)
    F_NEG_COL = 16u,  // K^T(log s): y <= 0
    F_NYS_COL = 32u,
};

struct DevState {
    int done;
    int status;     // 0, 3 (StabilizationError), 4 (NegativeKernelError)
    int which;      // 0 "log s", 1 "log t", 2 K, 3 K^T
    int iters;
    int converged;
    unsigned flags;
    double err;
    double H_s, H_t;  // low-rank shifts
    int allpos_s, allpos_t;
};

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 4096;  // bucket-side vector tile staged in shared memory

__device__ __forceinline__ double ld_val(const float* p, unsigned long long i) { return static_cast<double>(__ldg(p + i)); }
__device__ __forceinline__ double ld_val(const double* p, unsigned long long i) { return __ldg(p + i); }

// ---------------------------------------------------------------------------
// Sparse (log-domain) band kernels: per bucket block, per row / column online
// log-sum-exp, merged across bands as (max, sum) pairs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lse_merge(double& M, double& S, double m2, double s2) {
    if (m2 == kNegInf) return;
    if (M == kNegInf) { M = m2; S = s2; return; }
    if (m2 > M) { S = S * exp(M - m2) + s2; M = m2; }
    else S = S + s2 * exp(m2 - M);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) sparse_row_band_kernel(const DevState* __restrict__ st, BandView bv,
                                                                   const uint32_t* __restrict__ work,
                                                                   const T* __restrict__ vals,
                                                                   const double* __restrict__ log_t,
                                                                   double* __restrict__ Mrow, double* __restrict__ Srow) {
    if (st->done) return;
    __shared__ double lt[kTile];
    const uint32_t b = work[blockIdx.x];
    const uint32_t sb = bv.src_start[b], nb = bv.src_start[b + 1] - sb;
    const uint32_t tb = bv.tgt_start[b], mb = bv.tgt_start[b + 1] - tb;
    const unsigned long long off = bv.blk_off[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c0 = 0; c0 < mb; c0 += kTile) {
        const uint32_t cn = min(mb - c0, static_cast<uint32_t>(kTile));
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < cn; c += kThreads) lt[c] = log_t[bv.tgt_order[tb + c0 + c]];
        __syncthreads();
        for (uint32_t r = warp; r < nb; r += kWarps) {
            const unsigned long long row = off + static_cast<unsigned long long>(r) * mb + c0;
            double hi = kNegInf;
            for (uint32_t c = lane; c < cn; c += 32) hi = fmax(hi, ld_val(vals, row + c) + lt[c]);
            hi = warp_max(hi);
            double acc = 0.0;
            if (hi != kNegInf)
                for (uint32_t c = lane; c < cn; c += 32) acc += exp(ld_val(vals, row + c) + lt[c] - hi);
            acc = warp_sum(acc);
            if (lane == 0) {
                const uint32_t i = bv.src_order[sb + r];
                double M = Mrow[i], S = Srow[i];
                lse_merge(M, S, hi, acc);
                Mrow[i] = M;
                Srow[i] = S;
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) sparse_col_band_kernel(const DevState* __restrict__ st, BandView bv,
                                                                   const uint32_t* __restrict__ work,
                                                                   const T* __restrict__ vals,
                                                                   const double* __restrict__ log_s,
                                                                   double* __restrict__ Mcol, double* __restrict__ Scol) {
    if (st->done) return;
    __shared__ double ls[kTile];
    const uint32_t b = work[blockIdx.x];
    const uint32_t sb = bv.src_start[b], nb = bv.src_start[b + 1] - sb;
    const uint32_t tb = bv.tgt_start[b], mb = bv.tgt_start[b + 1] - tb;
    const unsigned long long off = bv.blk_off[b];
    for (uint32_t r0 = 0; r0 < nb; r0 += kTile) {
        const uint32_t rn = min(nb - r0, static_cast<uint32_t>(kTile));
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < rn; r += kThreads) ls[r] = log_s[bv.src_order[sb + r0 + r]];
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < mb; c += kThreads) {
            double hi = kNegInf;
            for (uint32_t r = 0; r < rn; ++r) hi = fmax(hi, ld_val(vals, off + static_cast<unsigned long long>(r0 + r) * mb + c) + ls[r]);
            double acc = 0.0;
            if (hi != kNegInf)
                for (uint32_t r = 0; r < rn; ++r)
                    acc += exp(ld_val(vals, off + static_cast<unsigned long long>(r0 + r) * mb + c) + ls[r] - hi);
            const uint32_t j = bv.tgt_order[tb + c];
            double M = Mcol[j], S = Scol[j];
            lse_merge(M, S, hi, acc);
            Mcol[j] = M;
            Scol[j] = S;
        }
    }
}

__global__ void lse_init_kernel(const DevState* __restrict__ st, double* __restrict__ M, double* __restrict__ S, long long n) {
    if (st->done) return;
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) { M[i] = kNegInf; S[i] = 0.0; }
}

// kts = M + log S (empty -> -inf, sparse_kernel.cpp:129); log t = log q - kts.
__global__ void sparse_col_finalize_kernel(DevState* __restrict__ st, const double* __restrict__ M,
                                           const double* __restrict__ S, const double* __restrict__ log_q, long long m,
                                           double* __restrict__ log_t) {
    if (st->done) return;
    long long j = blockIdx.x * 256LL + threadIdx.x;
    bool bad = false;
    if (j < m) {
        double kts = M[j] == kNegInf ? kNegInf : M[j] + log(S[j]);
        double v = log_q[j] - kts;
        log_t[j] = v;
        bad = !isfinite(v);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->flags, F_LOGT);
}

// kt, row marginal and error partial (sinkhorn.cpp:157-162), next log s.
__global__ void sparse_row_finalize_kernel(DevState* __restrict__ st, const double* __restrict__ M,
                                           const double* __restrict__ S, const double* __restrict__ log_p,
                                           const double* __restrict__ p, long long n, const double* __restrict__ log_s_cur,
                                           double* __restrict__ log_s_next, double* __restrict__ kt_out,
                                           double* __restrict__ row_marg, double* __restrict__ err_part, int with_err) {
    if (st->done) return;
    __shared__ double red[kWarps];
    long long i = blockIdx.x * 256LL + threadIdx.x;
    double e = 0.0;
    bool bad = false;
    if (i < n) {
        double kt = M[i] == kNegInf ? kNegInf : M[i] + log(S[i]);
        if (kt_out) kt_out[i] = kt;
        if (with_err) {
            double rm = exp(log_s_cur[i] + kt);
            row_marg[i] = rm;
            e = fabs(rm - p[i]);
        }
        double v = log_p[i] - kt;
        log_s_next[i] = v;
        bad = !isfinite(v);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->flags, F_LOGS);
    e = warp_sum(e);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0 && with_err) {
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += red[w];
        err_part[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// LCN (linear-space) band kernels: correction products Delta tt / Delta^T ss.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) lcn_row_band_kernel(const DevState* __restrict__ st, BandView bv,
                                                                const uint32_t* __restrict__ work,
                                                                const T* __restrict__ vals,
                                                                const double* __restrict__ log_t,
                                                                double* __restrict__ corr) {
    if (st->done) return;
    __shared__ double tt[kTile];
    const double H = st->H_t;
    const uint32_t b = work[blockIdx.x];
    const uint32_t sb = bv.src_start[b], nb = bv.src_start[b + 1] - sb;
    const uint32_t tb = bv.tgt_start[b], mb = bv.tgt_start[b + 1] - tb;
    const unsigned long long off = bv.blk_off[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c0 = 0; c0 < mb; c0 += kTile) {
        const uint32_t cn = min(mb - c0, static_cast<uint32_t>(kTile));
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < cn; c += kThreads) tt[c] = exp(log_t[bv.tgt_order[tb + c0 + c]] - H);
        __syncthreads();
        for (uint32_t r = warp; r < nb; r += kWarps) {
            const unsigned long long row = off + static_cast<unsigned long long>(r) * mb + c0;
            double acc = 0.0;
            for (uint32_t c = lane; c < cn; c += 32) acc += ld_val(vals, row + c) * tt[c];
            acc = warp_sum(acc);
            if (lane == 0) corr[bv.src_order[sb + r]] += acc;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) lcn_col_band_kernel(const DevState* __restrict__ st, BandView bv,
                                                                const uint32_t* __restrict__ work,
                                                                const T* __restrict__ vals,
                                                                const double* __restrict__ log_s,
                                                                double* __restrict__ corr) {
    if (st->done) return;
    __shared__ double ss[kTile];
    const double H = st->H_s;
    const uint32_t b = work[blockIdx.x];
    const uint32_t sb = bv.src_start[b], nb = bv.src_start[b + 1] - sb;
    const uint32_t tb = bv.tgt_start[b], mb = bv.tgt_start[b + 1] - tb;
    const unsigned long long off = bv.blk_off[b];
    for (uint32_t r0 = 0; r0 < nb; r0 += kTile) {
        const uint32_t rn = min(nb - r0, static_cast<uint32_t>(kTile));
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < rn; r += kThreads) ss[r] = exp(log_s[bv.src_order[sb + r0 + r]] - H);
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < mb; c += kThreads) {
            double acc = 0.0;
            for (uint32_t r = 0; r < rn; ++r) acc += ld_val(vals, off + static_cast<unsigned long long>(r0 + r) * mb + c) * ss[r];
            corr[bv.tgt_order[tb + c]] += acc;
        }
    }
}

__global__ void zero_kernel(const DevState* __restrict__ st, double* __restrict__ p, long long n) {
    if (st->done) return;
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) p[i] = 0.0;
}

// ---------------------------------------------------------------------------
// Low-rank passes. A warp owns a row of the tall factor F (U: n x l, or W^T:
// m x l); lane a-slices are a = lane + 32 k. The finalize kernel computes
// y = F_row . mid + corr, checks it, produces the new log vector, and folds
// F_row * exp(v - h) into the warp's running partial of the next product,
// rescaling when the running max h grows.
// ---------------------------------------------------------------------------
template <int LPL>
struct Partial {
    double h;
    double acc[LPL];
    __device__ void init() {
        h = kNegInf;
#pragma unroll
        for (int k = 0; k < LPL; ++k) acc[k] = 0.0;
    }
    template <typename T>
    __device__ void add(const T* __restrict__ row, int l, int lane, double v) {
        if (!(v > kNegInf && v < kPosInf)) return;  // non-finite inputs are flagged elsewhere
        if (v > h) {
            double sc = h == kNegInf ? 0.0 : exp(h - v);
#pragma unroll
            for (int k = 0; k < LPL; ++k) acc[k] *= sc;
            h = v;
        }
        const double w = exp(v - h);
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
            int a = lane + 32 * k;
            if (a < l) acc[k] += static_cast<double>(row[a]) * w;
        }
    }
};

// Combine the warps' partials of a block into one (h_b, partial_b[l]).
template <int LPL>
__device__ void block_combine(Partial<LPL>& P, int l, double* __restrict__ part_out, double* __restrict__ h_out,
                              double vmin, double vmax, double* __restrict__ min_out, double* __restrict__ max_out) {
    extern __shared__ double sm[];  // [kWarps * l] + [kWarps] h + 2*kWarps
    double* sp = sm;
    double* sh = sm + kWarps * l;
    double* smin = sh + kWarps;
    double* smax = smin + kWarps;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    vmin = -warp_max(-vmin);
    vmax = warp_max(vmax);
#pragma unroll
    for (int k = 0; k < LPL; ++k) {
        int a = lane + 32 * k;
        if (a < l) sp[warp * l + a] = P.acc[k];
    }
    if (lane == 0) {
        sh[warp] = P.h;
        smin[warp] = vmin;
        smax[warp] = vmax;
    }
    __syncthreads();
    double H = kNegInf;
    for (int w = 0; w < kWarps; ++w) H = fmax(H, sh[w]);
    for (int a = threadIdx.x; a < l; a += kThreads) {
        double s = 0.0;
        if (H != kNegInf)
            for (int w = 0; w < kWarps; ++w)
                if (sh[w] != kNegInf) s += sp[w * l + a] * exp(sh[w] - H);
        part_out[static_cast<long long>(blockIdx.x) * l + a] = s;
    }
    if (threadIdx.x == 0) {
        h_out[blockIdx.x] = H;
        double mn = kPosInf, mx = kNegInf;
        for (int w = 0; w < kWarps; ++w) { mn = fmin(mn, smin[w]); mx = fmax(mx, smax[w]); }
        min_out[blockIdx.x] = mn;
        max_out[blockIdx.x] = mx;
    }
}

// Partial F^T exp(v - h) for an arbitrary input vector (initial t = 0 and
// the log_matvec API).
template <typename T, int LPL>
__global__ void __launch_bounds__(kThreads) lowrank_accum_kernel(const DevState* __restrict__ st, const double* __restrict__ v,
                                                                 long long rows, const T* __restrict__ F, int l,
                                                                 double* __restrict__ part, double* __restrict__ hpart,
                                                                 double* __restrict__ mnp, double* __restrict__ mxp) {
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    Partial<LPL> P;
    P.init();
    double vmin = kPosInf, vmax = kNegInf;
    const long long gw = (static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const long long nw = static_cast<long long>(gridDim.x) * kWarps;
    for (long long i = gw; i < rows; i += nw) {
        double x = v ? v[i] : 0.0;
        vmin = fmin(vmin, x);
        vmax = fmax(vmax, x);
        P.add(F + i * l, l, lane, x);
    }
    block_combine<LPL>(P, l, part, hpart, vmin, vmax, mnp, mxp);
}

// Global shift and mid = sum_b exp(h_b - H) part_b; which: 0 -> t side, 1 -> s side.
__global__ void lowrank_reduce_kernel(DevState* __restrict__ st, const double* __restrict__ part,
                                      const double* __restrict__ hpart, const double* __restrict__ mnp,
                                      const double* __restrict__ mxp, int G, int l, double* __restrict__ mid, int which) {
    if (st->done) return;
    double H = kNegInf, mn = kPosInf;
    for (int b = 0; b < G; ++b) {
        H = fmax(H, hpart[b]);
        mn = fmin(mn, mnp[b]);
    }
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < l; a += gridDim.x * blockDim.x) {
        double s = 0.0;
        if (H != kNegInf)
            for (int b = 0; b < G; ++b)
                if (hpart[b] != kNegInf) s += part[static_cast<long long>(b) * l + a] * exp(hpart[b] - H);
        mid[a] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // positive_input of nys_matvec(_t) (nystrom.cpp:139-141): every exp(v - H) > 0.
        int allpos = H != kNegInf && exp(mn - H) > 0.0;
        if (which == 0) { st->H_t = H; st->allpos_t = allpos; }
        else { st->H_s = H; st->allpos_s = allpos; }
    }
}

// Column finalize (K^T side): y_j = W^T_j . mid_s + corr_t[j]; kts, log t,
// and the partial of W tt for the row side.
template <typename T, int LPL>
__global__ void __launch_bounds__(kThreads) lcn_col_finalize_kernel(
    DevState* __restrict__ st, const T* __restrict__ Wt, int l, long long m, const double* __restrict__ mid_s,
    const double* __restrict__ corr, const double* __restrict__ log_q, double* __restrict__ log_t,
    double* __restrict__ part, double* __restrict__ hpart, double* __restrict__ mnp, double* __restrict__ mxp, int mode,
    double* __restrict__ out) {
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    const double H = st->H_s;
    const int allpos = st->allpos_s;
    double mids[LPL];
#pragma unroll
    for (int k = 0; k < LPL; ++k) mids[k] = lane + 32 * k < l ? mid_s[lane + 32 * k] : 0.0;
    Partial<LPL> P;
    P.init();
    double vmin = kPosInf, vmax = kNegInf;
    unsigned fl = 0;
    const long long gw = (static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const long long nw = static_cast<long long>(gridDim.x) * kWarps;
    for (long long j = gw; j < m; j += nw) {
        const T* row = Wt + j * l;
        double nys = 0.0;
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
            int a = lane + 32 * k;
            if (a < l) nys += static_cast<double>(row[a]) * mids[k];
        }
        nys = warp_sum(nys);
        double y = nys + (corr ? corr[j] : 0.0);
        if (allpos && !(nys > 0.0)) fl |= F_NYS_COL;
        if (!(y > 0.0)) fl |= F_NEG_COL;
        double kts = H + log(y);
        if (mode == 1) {
            if (lane == 0) out[j] = kts;
            continue;
        }
        double v = log_q[j] - kts;
        if (lane == 0) log_t[j] = v;
        if (!isfinite(v)) fl |= F_LOGT;
        vmin = fmin(vmin, v);
        vmax = fmax(vmax, v);
        P.add(row, l, lane, v);
    }
    if (fl && lane == 0) atomicOr(&st->flags, fl);
    if (mode == 0) block_combine<LPL>(P, l, part, hpart, vmin, vmax, mnp, mxp);
}

// Row finalize (K side): y_i = U_i . mid_t + corr_s[i]; kt, row marginal,
// error partial, next log s and the partial of U^T ss for the next K^T.
template <typename T, int LPL>
__global__ void __launch_bounds__(kThreads) lcn_row_finalize_kernel(
    DevState* __restrict__ st, const T* __restrict__ U, int l, long long n, const double* __restrict__ mid_t,
    const double* __restrict__ corr, const double* __restrict__ log_p, const double* __restrict__ p,
    const double* __restrict__ log_s_cur, double* __restrict__ log_s_next, double* __restrict__ row_marg,
    double* __restrict__ err_part, int with_err, double* __restrict__ part, double* __restrict__ hpart,
    double* __restrict__ mnp, double* __restrict__ mxp, int mode, double* __restrict__ out) {
    if (st->done) return;
    __shared__ double red[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double H = st->H_t;
    const int allpos = st->allpos_t;
    double mids[LPL];
#pragma unroll
    for (int k = 0; k < LPL; ++k) mids[k] = lane + 32 * k < l ? mid_t[lane + 32 * k] : 0.0;
    Partial<LPL> P;
    P.init();
    double vmin = kPosInf, vmax = kNegInf, e = 0.0;
    unsigned fl = 0;
    const long long gw = (static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const long long nw = static_cast<long long>(gridDim.x) * kWarps;
    for (long long i = gw; i < n; i += nw) {
        const T* row = U + i * l;
        double nys = 0.0;
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
            int a = lane + 32 * k;
            if (a < l) nys += static_cast<double>(row[a]) * mids[k];
        }
        nys = warp_sum(nys);
        double y = nys + (corr ? corr[i] : 0.0);
        if (allpos && !(nys > 0.0)) fl |= F_NYS_ROW;
        if (!(y > 0.0)) fl |= F_NEG_ROW;
        double kt = H + log(y);
        if (mode == 1) {
            if (lane == 0) out[i] = kt;
            continue;
        }
        if (with_err) {
            double rm = exp(log_s_cur[i] + kt);
            if (lane == 0) row_marg[i] = rm;
            e += fabs(rm - p[i]);
        }
        double v = log_p[i] - kt;
        if (lane == 0) log_s_next[i] = v;
        if (!isfinite(v)) fl |= F_LOGS;
        vmin = fmin(vmin, v);
        vmax = fmax(vmax, v);
        P.add(row, l, lane, v);
    }
    if (fl && lane == 0) atomicOr(&st->flags, fl);
    if (mode == 1) return;
    if (lane == 0) red[warp] = e;
    block_combine<LPL>(P, l, part, hpart, vmin, vmax, mnp, mxp);
    if (threadIdx.x == 0 && with_err) {
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += red[w];
        err_part[blockIdx.x] = s;
    }
}

// End of iteration `it` (0 = the initial K(log t = 0)): error precedence in
// the reference's order, marginal error, trace, convergence.
__global__ void iter_end_kernel(DevState* __restrict__ st, const double* __restrict__ err_part, int G, int it,
                                int max_iters, double tol, double* __restrict__ trace) {
    if (st->done) return;
    const unsigned f = st->flags;
    auto fail = [&](int status, int which) {
        st->status = status;
        st->which = which;
        st->done = 1;
    };
    if (it > 0) {
        if (f & (F_NEG_COL | F_NYS_COL)) return fail(4, 3);
        if (f & F_LOGT) return fail(3, 1);
    }
    if (f & (F_NEG_ROW | F_NYS_ROW)) return fail(4, 2);
    if (it > 0) {
        double e = 0.0;
        for (int b = 0; b < G; ++b) e += err_part[b];
        st->err = e;
        trace[it - 1] = e;
        st->iters = it;
        if (e <= tol) {
            st->converged = 1;
            st->done = 1;
            return;
        }
        if (it >= max_iters) {
            st->done = 1;
            return;
        }
    }
    if (f & F_LOGS) return fail(3, 0);
    st->flags = 0;
}

// Distance identity (sinkhorn.cpp:178-183) partials.
__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                   double* __restrict__ out) {
    __shared__ double red[kWarps];
    double s = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) s += a[i] * b[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        out[blockIdx.x] = t;
    }
}

__global__ void sum_partial_kernel(const double* __restrict__ a, long long n, double* __restrict__ out) {
    __shared__ double red[kWarps];
    double s = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) s += a[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        out[blockIdx.x] = t;
    }
}

__global__ void log_kernel(const double* __restrict__ in, double* __restrict__ out, long long n) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) out[i] = log(in[i]);
}

int lpl_of(size_t l) {
    int k = static_cast<int>((l + 31) / 32);
    int p = 1;
    while (p < k) p <<= 1;
    return p;
}

}  // namespace

// ---------------------------------------------------------------------------
// Host driver
// ---------------------------------------------------------------------------
struct Solver {
    Op& op;
    Ctx& ctx;
    cudaStream_t s;
    long long n, m;
    int l, G, LPL;
    DevBuf<DevState> st;
    DevBuf<double> log_p, log_q, pv, qv, log_s[2], log_t, row_marg, err_part, trace;
    DevBuf<double> Mr, Sr, Mc, Sc, corr_s, corr_t;                  // sparse / lcn band accumulators
    DevBuf<double> part, hpart, mnp, mxp, mid_s, mid_t;             // low-rank reductions
    DevBuf<double> dpart;                                           // distance / mass partials
    size_t smem = 0;
    bool attrs_set = false;
    std::vector<cudaEvent_t> evs;                                   // phase events (profiling)
    ~Solver() {
        for (auto e : evs) cudaEventDestroy(e);
    }
    cudaEvent_t ev(size_t i) {
        while (evs.size() <= i) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            evs.push_back(e);
        }
        return evs[i];
    }

    explicit Solver(Op& o) : op(o), ctx(*o.ctx), s(o.ctx->stream), n(o.n), m(o.m), l(static_cast<int>(o.l)) {
        G = 4 * ctx.num_sms;
        LPL = lpl_of(std::max(l, 1));
        smem = (kWarps * static_cast<size_t>(std::max(l, 1)) + 3 * kWarps) * sizeof(double);
    }

    template <typename T>
    const T* band_vals(int b) const {
        if constexpr (std::is_same_v<T, float>) return op.val32[b].get();
        else return op.val64[b].get();
    }
    template <typename T>
    const T* U() const {
        if constexpr (std::is_same_v<T, float>) return op.U32.get();
        else return op.U64.get();
    }
    template <typename T>
    const T* Wt() const {
        if constexpr (std::is_same_v<T, float>) return op.Wt32.get();
        else return op.Wt64.get();
    }

    template <typename T, int LPLc>
    void launch_accum(const double* v, long long rows, const T* F) {
        lowrank_accum_kernel<T, LPLc><<<G, kThreads, smem, s>>>(st.get(), v, rows, F, l, part.get(), hpart.get(),
                                                               mnp.get(), mxp.get());
    }
    template <typename T, int LPLc>
    void launch_colfin(int mode, double* out) {
        lcn_col_finalize_kernel<T, LPLc><<<G, kThreads, smem, s>>>(st.get(), Wt<T>(), l, m, mid_s.get(),
                                                                  op.kind == 3 ? corr_t.get() : nullptr, log_q.get(),
                                                                  log_t.get(), part.get(), hpart.get(), mnp.get(),
                                                                  mxp.get(), mode, out);
    }
    template <typename T, int LPLc>
    void launch_rowfin(int it, int mode, double* out) {
        const int cur = it % 2, nxt = (it + 1) % 2;
        lcn_row_finalize_kernel<T, LPLc><<<G, kThreads, smem, s>>>(
            st.get(), U<T>(), l, n, mid_t.get(), op.kind == 3 ? corr_s.get() : nullptr, log_p.get(), pv.get(),
            log_s[cur].get(), log_s[nxt].get(), row_marg.get(), err_part.get(), it > 0, part.get(), hpart.get(),
            mnp.get(), mxp.get(), mode, out);
    }

#define LCNB_LPL_DISPATCH(CALL)                        \
    switch (LPL) {                                     \
        case 1: CALL(1); break;                        \
        case 2: CALL(2); break;                        \
        case 4: CALL(4); break;                        \
        case 8: CALL(8); break;                        \
        case 16: CALL(16); break;                      \
        case 32: CALL(32); break;                      \
        default: throw Status(2, "lcn: landmark count above 1024 is not supported on this path"); \
    }

    void alloc() {
        s = ctx.stream;
        st.resize(1);
        st.zero(s);
        dpart.resize(256);
        log_p.resize(n); log_q.resize(m); pv.resize(n); qv.resize(m);
        log_s[0].resize(n); log_s[1].resize(n); log_t.resize(m); row_marg.resize(n);
        err_part.resize(std::max<long long>(G, ceil_div(n, 256)));
        if (op.kind == 1) {
            Mr.resize(n); Sr.resize(n); Mc.resize(m); Sc.resize(m);
        } else {
            corr_s.resize(n); corr_t.resize(m);
            part.resize(static_cast<size_t>(G) * l); hpart.resize(G); mnp.resize(G); mxp.resize(G);
            mid_s.resize(l); mid_t.resize(l);
        }
    }

    // -------- sparse -------------------------------------------------------
    template <typename T>
    void sparse_rows(const double* lt) {
        lse_init_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), Mr.get(), Sr.get(), n);
        for (size_t b = 0; b < op.bands.size(); ++b)
            if (op.bands[b].n_work)
                sparse_row_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                    st.get(), op.view(b), op.bands[b].work.get(), band_vals<T>(b), lt, Mr.get(), Sr.get());
    }
    template <typename T>
    void sparse_cols(const double* ls) {
        lse_init_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), Mc.get(), Sc.get(), m);
        for (size_t b = 0; b < op.bands.size(); ++b)
            if (op.bands[b].n_work)
                sparse_col_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                    st.get(), op.view(b), op.bands[b].work.get(), band_vals<T>(b), ls, Mc.get(), Sc.get());
    }
    template <typename T>
    void sparse_iteration(int it, double tol, int max_iters) {
        const int cur = it % 2, nxt = (it + 1) % 2;
        mark(it, 0);
        if (it > 0) {
            sparse_cols<T>(log_s[cur].get());
            mark(it, 1);
            sparse_col_finalize_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), Mc.get(), Sc.get(), log_q.get(), m,
                                                                        log_t.get());
        } else {
            mark(it, 1);
        }
        mark(it, 2);
        sparse_rows<T>(log_t.get());
        mark(it, 3);
        sparse_row_finalize_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), Mr.get(), Sr.get(), log_p.get(), pv.get(),
                                                                    n, log_s[cur].get(), log_s[nxt].get(), nullptr,
                                                                    row_marg.get(), err_part.get(), it > 0);
        iter_end_kernel<<<1, 1, 0, s>>>(st.get(), err_part.get(), ceil_div(n, 256), it, max_iters, tol, trace.get());
        mark(it, 4);
    }

    // -------- lcn / nystrom ------------------------------------------------
    template <typename T>
    void lcn_rows(const double* lt) {
        if (op.kind != 3) return;
        zero_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), corr_s.get(), n);
        for (size_t b = 0; b < op.bands.size(); ++b)
            if (op.bands[b].n_work)
                lcn_row_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                    st.get(), op.view(b), op.bands[b].work.get(), band_vals<T>(b), lt, corr_s.get());
    }
    template <typename T>
    void lcn_cols(const double* ls) {
        if (op.kind != 3) return;
        zero_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), corr_t.get(), m);
        for (size_t b = 0; b < op.bands.size(); ++b)
            if (op.bands[b].n_work)
                lcn_col_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                    st.get(), op.view(b), op.bands[b].work.get(), band_vals<T>(b), ls, corr_t.get());
    }
    template <typename T>
    void lcn_iteration(int it, double tol, int max_iters) {
        const int cur = it % 2;
        mark(it, 0);
        if (it == 0) {
            // kt = K(log t = 0) (sinkhorn.cpp:145): partial W^T 1 with shift 0.
#define ACC0(L) launch_accum<T, L>(nullptr, m, Wt<T>())
            LCNB_LPL_DISPATCH(ACC0)
#undef ACC0
            lowrank_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(st.get(), part.get(), hpart.get(), mnp.get(),
                                                                  mxp.get(), G, l, mid_t.get(), 0);
            mark(it, 1);
        } else {
            lcn_cols<T>(log_s[cur].get());
            mark(it, 1);
#define COLF(L) launch_colfin<T, L>(0, nullptr)
            LCNB_LPL_DISPATCH(COLF)
#undef COLF
            lowrank_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(st.get(), part.get(), hpart.get(), mnp.get(),
                                                                  mxp.get(), G, l, mid_t.get(), 0);
        }
        mark(it, 2);
        lcn_rows<T>(log_t.get());
        mark(it, 3);
#define ROWF(L) launch_rowfin<T, L>(it, 0, nullptr)
        LCNB_LPL_DISPATCH(ROWF)
#undef ROWF
        lowrank_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(st.get(), part.get(), hpart.get(), mnp.get(), mxp.get(),
                                                              G, l, mid_s.get(), 1);
        iter_end_kernel<<<1, 1, 0, s>>>(st.get(), err_part.get(), G, it, max_iters, tol, trace.get());
        mark(it, 4);
    }

    template <typename T>
    void set_smem_attrs() {
        if (attrs_set) return;
        attrs_set = true;
        if (op.kind == 1 || smem <= 48 * 1024) return;
#define ATTR(L)                                                                                                    \
    CUDA_OK(cudaFuncSetAttribute(lowrank_accum_kernel<T, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    CUDA_OK(cudaFuncSetAttribute(lcn_col_finalize_kernel<T, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    CUDA_OK(cudaFuncSetAttribute(lcn_row_finalize_kernel<T, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
        LCNB_LPL_DISPATCH(ATTR)
#undef ATTR
    }

    // phase marks: 0 start of iteration, 1 after col bands, 2 after col
    // finalize+reduce, 3 after row bands, 4 after row finalize+reduce+end.
    size_t mark_base = 0;
    void mark(int it, int ph) {
        if (ctx.profile) CUDA_OK(cudaEventRecord(ev(mark_base + static_cast<size_t>(it) * 5 + ph), s));
    }

    template <typename T>
    void run(const double* in_p, const double* in_q, bool device_ptrs, const SolveOptions& o, Result& res) {
        set_smem_attrs<T>();
        alloc();
        trace.resize(std::max<size_t>(std::max(o.max_iters, 1), trace.size()));
        const cudaMemcpyKind kind = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        CUDA_OK(cudaMemcpyAsync(pv.get(), in_p, n * 8, kind, s));
        CUDA_OK(cudaMemcpyAsync(qv.get(), in_q, m * 8, kind, s));
        log_kernel<<<ceil_div(n, 256), 256, 0, s>>>(pv.get(), log_p.get(), n);
        log_kernel<<<ceil_div(m, 256), 256, 0, s>>>(qv.get(), log_q.get(), m);
        CUDA_OK(cudaMemsetAsync(log_s[0].get(), 0, n * 8, s));
        CUDA_OK(cudaMemsetAsync(log_s[1].get(), 0, n * 8, s));
        CUDA_OK(cudaMemsetAsync(log_t.get(), 0, m * 8, s));
        CUDA_OK(cudaMemsetAsync(row_marg.get(), 0, n * 8, s));
        // tol: default 1e-6 * (sum p + sum q) (sinkhorn.cpp:130-133).
        double tol = o.tol;
        if (tol < 0.0) {
            double mass = 0.0;
            if (device_ptrs) {
                sum_partial_kernel<<<64, 256, 0, s>>>(pv.get(), n, dpart.get());
                sum_partial_kernel<<<64, 256, 0, s>>>(qv.get(), m, dpart.get() + 64);
                std::vector<double> hp(128);
                dpart.download(hp.data(), 128, s);
                ctx.sync();
                for (double v : hp) mass += v;
            } else {
                for (long long i = 0; i < n; ++i) mass += in_p[i];
                for (long long j = 0; j < m; ++j) mass += in_q[j];
            }
            tol = 1e-6 * mass;
        }
        cudaEvent_t e0 = ev(0), e1 = ev(1);
        mark_base = 2;
        CUDA_OK(cudaEventRecord(e0, s));
        const int chunk = tol > 0.0 ? 8 : o.max_iters + 1;
        DevState h{};
        for (int it0 = 0; it0 <= o.max_iters; it0 += chunk) {
            for (int it = it0; it < std::min(it0 + chunk, o.max_iters + 1); ++it) {
                if (op.kind == 1) sparse_iteration<T>(it, tol, o.max_iters);
                else lcn_iteration<T>(it, tol, o.max_iters);
            }
            LAUNCH_OK("sinkhorn iteration");
            st.download(&h, 1, s);
            ctx.sync();
            if (h.done) break;
        }
        CUDA_OK(cudaEventRecord(e1, s));
        CUDA_OK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        res.device_ms = ms;
        res.phase_ms.assign(4, 0.0);
        res.phase_iters = 0;
        if (ctx.profile) {
            // iterations 1..iters ran all phases (iteration 0 has no column side)
            for (int it = 1; it <= h.iters; ++it) {
                for (int ph = 0; ph < 4; ++ph) {
                    float t = 0.f;
                    CUDA_OK(cudaEventElapsedTime(&t, ev(mark_base + it * 5 + ph), ev(mark_base + it * 5 + ph + 1)));
                    res.phase_ms[ph] += t;
                }
            }
            res.phase_iters = h.iters;
        }
        if (h.status) {
            std::string name = op.name();
            if (h.status == 3)
                throw Status(3, std::string("sinkhorn: non-finite scaling (") + (h.which == 0 ? "log s" : "log t") +
                                    ") under the " + name + " operator");
            throw Status(4, name + (h.which == 3 ? " transposed matvec" : " matvec") + " produced a nonpositive entry");
        }
        res.iters = h.iters;
        res.converged = h.converged != 0;
        res.marginal_err_final = h.err;
        res.n = n;
        res.m = m;
        const int fin = h.iters % 2;
        res.log_s.resize(n);
        res.log_t.resize(m);
        res.row_marg.resize(n);
        res.err_trace.resize(h.iters);
        log_s[fin].download(res.log_s.data(), n, s);
        log_t.download(res.log_t.data(), m, s);
        row_marg.download(res.row_marg.data(), n, s);
        if (h.iters) trace.download(res.err_trace.data(), h.iters, s);
        // distance = lambda (<log s, P1> + <log t, q>) (sinkhorn.cpp:178-183)
        const int DB = 64;
        double* dp = dpart.get();
        dot_partial_kernel<<<DB, 256, 0, s>>>(log_s[fin].get(), row_marg.get(), n, dp);
        dot_partial_kernel<<<DB, 256, 0, s>>>(log_t.get(), qv.get(), m, dp + DB);
        std::vector<double> hp(2 * DB);
        dpart.download(hp.data(), 2 * DB, s);
        ctx.sync();
        double acc = 0.0;
        for (double v : hp) acc += v;
        res.distance = op.lambda * acc;
    }

    // log_matvec / log_matvec_t (operator.cpp:226-252) on a host vector.
    template <typename T>
    void matvec(const double* h_in, bool transposed, double* h_out) {
        set_smem_attrs<T>();
        alloc();
        const long long len_in = transposed ? n : m, len_out = transposed ? m : n;
        DevBuf<double> vin(len_in), vout(len_out);
        vin.upload(h_in, len_in, s);
        if (op.kind == 1) {
            if (!transposed) {
                sparse_rows<T>(vin.get());
                sparse_row_finalize_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), Mr.get(), Sr.get(), log_p.get(),
                                                                            pv.get(), n, nullptr, log_s[1].get(),
                                                                            vout.get(), nullptr, nullptr, 0);
            } else {
                sparse_cols<T>(vin.get());
                // kts only: reuse the finalize with log_q = 0 and read M/S directly
                DevBuf<double> zq(m);
                zq.zero(s);
                sparse_col_finalize_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), Mc.get(), Sc.get(), zq.get(), m,
                                                                            vout.get());
                // vout = 0 - kts -> negate on host below
            }
        } else {
            if (!transposed) {
#define ACC1(L) launch_accum<T, L>(vin.get(), m, Wt<T>())
                LCNB_LPL_DISPATCH(ACC1)
#undef ACC1
                lowrank_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(st.get(), part.get(), hpart.get(), mnp.get(),
                                                                      mxp.get(), G, l, mid_t.get(), 0);
                lcn_rows<T>(vin.get());
#define ROWM(L) launch_rowfin<T, L>(0, 1, vout.get())
                LCNB_LPL_DISPATCH(ROWM)
#undef ROWM
            } else {
#define ACC2(L) launch_accum<T, L>(vin.get(), n, U<T>())
                LCNB_LPL_DISPATCH(ACC2)
#undef ACC2
                lowrank_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(st.get(), part.get(), hpart.get(), mnp.get(),
                                                                      mxp.get(), G, l, mid_s.get(), 1);
                lcn_cols<T>(vin.get());
#define COLM(L) launch_colfin<T, L>(1, vout.get())
                LCNB_LPL_DISPATCH(COLM)
#undef COLM
            }
        }
        LAUNCH_OK("log_matvec");
        DevState h{};
        st.download(&h, 1, s);
        vout.download(h_out, len_out, s);
        ctx.sync();
        if (op.kind == 1 && transposed)
            for (long long j = 0; j < len_out; ++j) h_out[j] = -h_out[j];
        if (op.kind != 1) {
            // all -inf input -> all -inf output (operator.cpp:148-149)
            double hi = kNegInf;
            for (long long i = 0; i < len_in; ++i) hi = std::max(hi, h_in[i]);
            if (hi == kNegInf) {
                for (long long i = 0; i < len_out; ++i) h_out[i] = kNegInf;
                return;
            }
            const unsigned f = h.flags;
            std::string name = op.name();
            if (!transposed && (f & (F_NEG_ROW | F_NYS_ROW))) throw Status(4, name + " matvec produced a nonpositive entry");
            if (transposed && (f & (F_NEG_COL | F_NYS_COL)))
                throw Status(4, name + " transposed matvec produced a nonpositive entry");
        }
    }
};

Solver& solver_of(Op& op) {
    if (!op.ws) op.ws = std::make_shared<Solver>(op);
    return *op.ws;
}

void sinkhorn_solve(Op& op, const double* p, const double* q, bool device_ptrs, const SolveOptions& o, Result& res) {
    if (o.max_iters < 1) throw Status(2, "sinkhorn: max_iters must be >= 1");
    Solver& sv = solver_of(op);
    if (op.fp64) sv.run<double>(p, q, device_ptrs, o, res);
    else sv.run<float>(p, q, device_ptrs, o, res);
}

void op_log_matvec(Op& op, const double* h_in, bool transposed, double* h_out) {
    Solver& sv = solver_of(op);
    if (op.fp64) sv.matvec<double>(h_in, transposed, h_out);
    else sv.matvec<float>(h_in, transposed, h_out);
}

// distance_lcn (sinkhorn.cpp:222-261), from the fp64 factors on the device
// (host-side reduction order).
double distance_lcn_device(Op& op, const Result& res) {
    Ctx& ctx = *op.ctx;
    const size_t n = op.n, m = op.m, l = op.l;
    std::vector<double> U(n * l), Wt(m * l);
    op.U64.download(U.data(), n * l, ctx.stream);
    op.Wt64.download(Wt.data(), m * l, ctx.stream);
    ctx.sync();
    std::vector<double> s_lin(n), t_lin(m), wt(l, 0.0), su(l, 0.0);
    for (size_t i = 0; i < n; ++i) s_lin[i] = std::exp(res.log_s[i]);
    for (size_t j = 0; j < m; ++j) t_lin[j] = std::exp(res.log_t[j]);
    for (size_t j = 0; j < m; ++j)
        for (size_t a = 0; a < l; ++a) wt[a] += Wt[j * l + a] * t_lin[j];
    for (size_t i = 0; i < n; ++i)
        for (size_t a = 0; a < l; ++a) su[a] += U[i * l + a] * s_lin[i];
    double term = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double row = 0.0;
        for (size_t a = 0; a < l; ++a) row += U[i * l + a] * wt[a];
        term += res.log_s[i] * (s_lin[i] * row);
    }
    for (size_t j = 0; j < m; ++j) {
        double col = 0.0;
        for (size_t a = 0; a < l; ++a) col += su[a] * Wt[j * l + a];
        term += res.log_t[j] * (col * t_lin[j]);
    }
    if (op.kind == 3 && op.nnz) {
        std::vector<uint32_t> rp(n + 1), col(op.nnz);
        std::vector<double> dl(op.nnz);
        export_csr(op, 1, rp.data(), col.data(), dl.data());
        for (size_t i = 0; i < n; ++i)
            for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
                double mass = s_lin[i] * dl[e] * t_lin[col[e]];
                term += mass * (res.log_s[i] + res.log_t[col[e]]);
            }
    }
    return op.lambda * term;
}

}  // namespace lcnb
