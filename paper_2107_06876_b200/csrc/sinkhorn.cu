// Log-stabilised Sinkhorn over the bucket-blocked operators
// (sinkhorn.cpp:104-188, operator.cpp:123-224).
//
// One iteration = the reference's s-update, K^T application, t-update, K
// application and marginal error (sinkhorn.cpp:149-168). On the device it is a
// fixed sequence of kernels, all enqueued ahead and gated by a device-side
// `done` flag, so the host never waits inside the loop:
//   col side : band blocks (Delta^T ss per band / sparse column LSE)  ->
//              low-rank pass over W^T rows (W^T_j . mid_s + corrections,
//              positivity, log t = log q - K^T(log s), finiteness, and the
//              partial W tt of the next half)  ->  reduce (H_t, mid_t)
//   row side : band blocks  ->  low-rank pass over U rows (kt, row marginal,
//              error partial, next log s, partial U^T ss)  ->  reduce + end
// Low-rank shifts: the reference shifts by the global max of the input log
// vector (operator.cpp:147-151); each CTA keeps a running max with online
// rescaling and the reduce rescales the CTA partials to the global max — the
// same product in exact arithmetic, with no extra pass over the factors.
//
// Streaming design (HBM-bound passes). Loaded HBM latency on this part is a
// few microseconds, so an SM needs ~200 KB of reads in flight to approach
// peak (Little's law). Both the low-rank pass and the band passes are
// warp-specialized: producer warps keep a shared-memory ring full with
// cp.async.bulk copies (SASS UBLKCP) tracked by mbarriers, consumer warps
// only wait on `full` barriers and compute from shared memory. Block rows are
// padded to 16-byte multiples and blocks start on 128-byte lines (build.cu),
// factor rows to lp = round_up(l, 4).
#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <utility>
#include <type_traits>


#include "async.cuh"
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

constexpr int kThreads = 256;  // consumer threads per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 4096;    // bucket-side vector tile of the per-bucket kernels

template <typename T>
struct Raw4 {
    T v[4];
};
__device__ __forceinline__ Raw4<float> raw4(const float* p) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    return {{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ Raw4<double> raw4(const double* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return {{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ double ld1(const float* p) { return static_cast<double>(__ldg(p)); }
__device__ __forceinline__ double ld1(const double* p) { return __ldg(p); }

// consumer-only barrier (producer warps never join)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }


// ---------------------------------------------------------------------------
// Sparse (log-domain) band kernels: per bucket block, per row / column
// log-sum-exp (sparse_kernel.cpp:119-155), merged across bands as (max, sum).
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
    const unsigned long long ms = row_stride(mb);
    const unsigned long long off = bv.blk_off[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c0 = 0; c0 < mb; c0 += kTile) {
        const uint32_t cn = min(mb - c0, static_cast<uint32_t>(kTile));
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < cn; c += kThreads) lt[c] = log_t[bv.tgt_order[tb + c0 + c]];
        __syncthreads();
        if constexpr (sizeof(T) == 4) {
            // fp32 storage: the tile's log t as fp32 in shared memory (-inf
            // past the bucket, so padded row ends drop out), 16-byte loads,
            // 4 rows per warp at a time (4 x the loads in flight), exponents
            // in fp32 (MUFU), each row's sum widened once; the second read of
            // the rows hits L1 / L2
            __shared__ __align__(16) float ltf[kTile];
            const uint32_t cn4 = (cn + 3) & ~3u;
            for (uint32_t c = threadIdx.x; c < cn4; c += kThreads)
                ltf[c] = c < cn ? static_cast<float>(lt[c]) : -CUDART_INF_F;
            __syncthreads();
            constexpr int kRW = 4;
            for (uint32_t r0w = warp * kRW; r0w < nb; r0w += kWarps * kRW) {
                const float* rp[kRW];
                bool rv[kRW];
#pragma unroll
                for (int k = 0; k < kRW; ++k) {
                    rv[k] = r0w + k < nb;
                    rp[k] = vals + off + static_cast<unsigned long long>(rv[k] ? r0w + k : r0w) * ms + c0;
                }
                // one read: per lane an online (max, sum) per row, merged
                // across the warp at the end
                float hf[kRW], af[kRW];
#pragma unroll
                for (int k = 0; k < kRW; ++k) {
                    hf[k] = -CUDART_INF_F;
                    af[k] = 0.0f;
                }
                for (uint32_t c = 4 * lane; c < cn4; c += 128) {
                    const float4 l4 = *reinterpret_cast<const float4*>(ltf + c);
#pragma unroll
                    for (int k = 0; k < kRW; ++k) {
                        const float4 v = __ldg(reinterpret_cast<const float4*>(rp[k] + c));
                        const float x0 = v.x + l4.x, x1 = v.y + l4.y, x2 = v.z + l4.z, x3 = v.w + l4.w;
                        const float mx = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
                        if (mx > hf[k]) {  // new running max: rescale the sum once
                            af[k] *= __expf(hf[k] - mx);
                            hf[k] = mx;
                        }
                        if (hf[k] != -CUDART_INF_F)
                            af[k] += (__expf(x0 - hf[k]) + __expf(x1 - hf[k])) + (__expf(x2 - hf[k]) + __expf(x3 - hf[k]));
                    }
                }
#pragma unroll
                for (int k = 0; k < kRW; ++k) {  // warp merge of the lanes' (max, sum)
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        const float ho = __shfl_xor_sync(0xffffffffu, hf[k], o);
                        const float ao = __shfl_xor_sync(0xffffffffu, af[k], o);
                        const float hn = fmaxf(hf[k], ho);
                        if (hn != -CUDART_INF_F) {
                            af[k] = af[k] * __expf(hf[k] - hn) + ao * __expf(ho - hn);
                            hf[k] = hn;
                        }
                    }
                }
                if (lane < kRW && rv[lane & (kRW - 1)]) {
                    float h = hf[0], a = af[0];
#pragma unroll
                    for (int k = 1; k < kRW; ++k)
                        if (lane == k) {
                            h = hf[k];
                            a = af[k];
                        }
                    const uint32_t i = bv.src_order[sb + r0w + lane];
                    double M = Mrow[i], S = Srow[i];
                    lse_merge(M, S, h == -CUDART_INF_F ? kNegInf : static_cast<double>(h), static_cast<double>(a));
                    Mrow[i] = M;
                    Srow[i] = S;
                }
            }
            continue;
        }
        for (uint32_t r = warp; r < nb; r += kWarps) {
            const T* row = vals + off + r * ms + c0;
            double hi = kNegInf, acc = 0.0;
            {
                for (uint32_t c = lane; c < cn; c += 32) hi = fmax(hi, ld1(row + c) + lt[c]);
                hi = warp_max(hi);
                if (hi != kNegInf)
                    for (uint32_t c = lane; c < cn; c += 32) acc += exp(ld1(row + c) + lt[c] - hi);
                acc = warp_sum(acc);
            }
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
    const unsigned long long ms = row_stride(mb);
    const unsigned long long off = bv.blk_off[b];
    for (uint32_t r0 = 0; r0 < nb; r0 += kTile) {
        const uint32_t rn = min(nb - r0, static_cast<uint32_t>(kTile));
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < rn; r += kThreads) ls[r] = log_s[bv.src_order[sb + r0 + r]];
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < mb; c += kThreads) {
            double hi = kNegInf, acc = 0.0;
            if constexpr (sizeof(T) == 4) {  // fp32 storage: fp32 exponents (MUFU); the second pass hits L2
                const T* col = vals + off + static_cast<unsigned long long>(r0) * ms + c;
                float h4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
                uint32_t r = 0;
                for (; r + 4 <= rn; r += 4)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        h4[k] = fmaxf(h4[k], col[static_cast<unsigned long long>(r + k) * ms] + static_cast<float>(ls[r + k]));
                for (; r < rn; ++r) h4[0] = fmaxf(h4[0], col[static_cast<unsigned long long>(r) * ms] + static_cast<float>(ls[r]));
                const float hf = fmaxf(fmaxf(h4[0], h4[1]), fmaxf(h4[2], h4[3]));
                float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                if (hf != -CUDART_INF_F) {
                    r = 0;
                    for (; r + 4 <= rn; r += 4)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            a4[k] += __expf(col[static_cast<unsigned long long>(r + k) * ms] + static_cast<float>(ls[r + k]) - hf);
                    for (; r < rn; ++r) a4[0] += __expf(col[static_cast<unsigned long long>(r) * ms] + static_cast<float>(ls[r]) - hf);
                }
                hi = hf == -CUDART_INF_F ? kNegInf : static_cast<double>(hf);
                acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
            } else {
                for (uint32_t r = 0; r < rn; ++r) hi = fmax(hi, ld1(vals + off + (r0 + r) * ms + c) + ls[r]);
                if (hi != kNegInf)
                    for (uint32_t r = 0; r < rn; ++r) acc += exp(ld1(vals + off + (r0 + r) * ms + c) + ls[r] - hi);
            }
            const uint32_t j = bv.tgt_order[tb + c];
            double M = Mcol[j], S = Scol[j];
            lse_merge(M, S, hi, acc);
            Mcol[j] = M;
            Scol[j] = S;
        }
    }
}

// ---- general CSR patterns (KernelOperator::sparse / ::lcn from host structs) ----
// Row (or, on the CSC view, column) log-sum-exp of a sparse kernel
// (sparse_log_matvec, sparse_kernel.cpp:119-155): (max, sum exp(. - max)) per
// row, the pair the band kernels produce. One warp per row.
__global__ void csr_lse_kernel(const DevState* __restrict__ st, const uint32_t* __restrict__ ptr,
                               const uint32_t* __restrict__ idx, const double* __restrict__ val,
                               const double* __restrict__ lv, long long rows, double* __restrict__ M,
                               double* __restrict__ S) {
    if (st->done) return;
    const long long r = (blockIdx.x * 256LL + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const uint32_t b = ptr[r], e = ptr[r + 1];
    double hi = kNegInf;
    for (uint32_t k = b + lane; k < e; k += 32) hi = fmax(hi, val[k] + lv[idx[k]]);
    hi = warp_max(hi);
    double acc = 0.0;
    if (hi != kNegInf)
        for (uint32_t k = b + lane; k < e; k += 32) acc += exp(val[k] + lv[idx[k]] - hi);
    acc = warp_sum(acc);
    if (lane == 0) {
        M[r] = hi;
        S[r] = hi == kNegInf ? 0.0 : acc;
    }
}

// Linear-space correction product (correction_matvec(_t), sparse_kernel.cpp:
// 157-185) in the band kernels' convention: out[r] = sum delta * exp(lv - H).
__global__ void csr_corr_kernel(const DevState* __restrict__ st, const uint32_t* __restrict__ ptr,
                                const uint32_t* __restrict__ idx, const double* __restrict__ val,
                                const double* __restrict__ lv, long long rows, int rows_pass,
                                double* __restrict__ out) {
    if (st->done) return;
    const long long r = (blockIdx.x * 256LL + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const double H = rows_pass ? st->H_t : st->H_s;
    double acc = 0.0;
    for (uint32_t k = ptr[r] + lane; k < ptr[r + 1]; k += 32) acc += val[k] * exp(lv[idx[k]] - H);
    acc = warp_sum(acc);
    if (lane == 0) out[r] = acc;
}

__global__ void lse_init_kernel(const DevState* __restrict__ st, double* __restrict__ M, double* __restrict__ S, long long n) {
    if (st->done) return;
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) { M[i] = kNegInf; S[i] = 0.0; }
}

// Dense log-domain matvec (operator.cpp:125-140 / 178-192), as (max, sum)
// pairs for the finalize kernels: for each of 8 rows per CTA, threads stream
// the row (coalesced) against the shared vector with an online max-shifted
// sum, then a warp / shared-memory merge. 8 rows per CTA share every read of
// the vector. fp32 storage: exp of the shifted value on the fp32 MUFU path.
constexpr int kDenseRows = 8;

template <typename T>
__device__ __forceinline__ double lse_exp(double x) {  // x <= 0
    if constexpr (sizeof(T) == 4) return x < -87.0 ? 0.0 : static_cast<double>(__expf(static_cast<float>(x)));
    else return exp(x);
}

template <typename T>
__device__ __forceinline__ void lse_push(double& m, double& s, double v) {
    if (v == kNegInf) return;
    if (v > m) {
        s = (m == kNegInf ? 0.0 : s * lse_exp<T>(m - v)) + 1.0;
        m = v;
    } else {
        s += lse_exp<T>(v - m);
    }
}

__device__ __forceinline__ void lse_pair_merge(double& m, double& s, double om, double os) {
    const double mm = fmax(m, om);
    if (mm == kNegInf) return;
    s = (m == kNegInf ? 0.0 : s * exp(m - mm)) + (om == kNegInf ? 0.0 : os * exp(om - mm));
    m = mm;
}

template <typename T>
__global__ void __launch_bounds__(256) dense_lse_kernel(const DevState* __restrict__ st, const T* __restrict__ logk,
                                                        long long rows, long long cols,
                                                        const double* __restrict__ logv, double* __restrict__ M,
                                                        double* __restrict__ S) {
    if (st->done) return;
    __shared__ double wm[kWarps][kDenseRows], ws[kWarps][kDenseRows];
    const long long i0 = static_cast<long long>(blockIdx.x) * kDenseRows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double m[kDenseRows], sm[kDenseRows];
#pragma unroll
    for (int r = 0; r < kDenseRows; ++r) { m[r] = kNegInf; sm[r] = 0.0; }
    const int nr = static_cast<int>(rows - i0 < kDenseRows ? rows - i0 : kDenseRows);
    if constexpr (sizeof(T) == 4) {
        // fp32 storage: the online max-shifted sum runs in fp32 (v = log K + log v
        // has ~1e-6 relative error on the exponent already); widened per thread
        float mf[kDenseRows], sf[kDenseRows];
#pragma unroll
        for (int r = 0; r < kDenseRows; ++r) { mf[r] = -INFINITY; sf[r] = 0.0f; }
        // batches of 4 strided columns: one max, at most one rescale, then
        // unconditional exps (no per-element divergence)
        constexpr int kB = 4;
        long long j0 = threadIdx.x;
        for (; j0 + (kB - 1) * 256 < cols; j0 += kB * 256) {
            float lv[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) lv[u] = static_cast<float>(logv[j0 + u * 256]);
#pragma unroll
            for (int r = 0; r < kDenseRows; ++r) {
                if (r < nr) {
                    const float* row = logk + (i0 + r) * cols + j0;
                    float v[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) v[u] = row[u * 256] + lv[u];
                    const float bm = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
                    if (bm > mf[r]) {
                        sf[r] *= __expf(mf[r] - bm);  // exp(-inf) = 0 for the first batch
                        mf[r] = bm;
                    }
                    if (mf[r] != -INFINITY) {
#pragma unroll
                        for (int u = 0; u < kB; ++u) sf[r] += __expf(v[u] - mf[r]);
                    }
                }
            }
        }
        for (long long j = j0; j < cols; j += 256) {  // tail
            const float lv = static_cast<float>(logv[j]);
#pragma unroll
            for (int r = 0; r < kDenseRows; ++r) {
                if (r < nr) {
                    const float v = logk[(i0 + r) * cols + j] + lv;
                    if (v > mf[r]) {
                        sf[r] = sf[r] * __expf(mf[r] - v) + 1.0f;
                        mf[r] = v;
                    } else if (v != -INFINITY) {
                        sf[r] += __expf(v - mf[r]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kDenseRows; ++r) {
            m[r] = mf[r] == -INFINITY ? kNegInf : static_cast<double>(mf[r]);
            sm[r] = static_cast<double>(sf[r]);
        }
    } else {
        for (long long j = threadIdx.x; j < cols; j += 256) {
            const double lv = logv[j];
#pragma unroll
            for (int r = 0; r < kDenseRows; ++r)
                if (r < nr) lse_push<T>(m[r], sm[r], static_cast<double>(logk[(i0 + r) * cols + j]) + lv);
        }
    }
#pragma unroll
    for (int r = 0; r < kDenseRows; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double om = __shfl_xor_sync(0xffffffffu, m[r], o), os = __shfl_xor_sync(0xffffffffu, sm[r], o);
            lse_pair_merge(m[r], sm[r], om, os);
        }
        if (lane == 0) { wm[warp][r] = m[r]; ws[warp][r] = sm[r]; }
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        const int r = threadIdx.x;
        double mm = kNegInf, ss = 0.0;
        for (int w = 0; w < kWarps; ++w) lse_pair_merge(mm, ss, wm[w][r], ws[w][r]);
        M[i0 + r] = mm;
        S[i0 + r] = ss;
    }
}

constexpr float kL2E = 1.4426950408889634f;  // log2(e)
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// fp32 storage, cols % 4 == 0: the same (max, sum) pairs, streamed through
// shared memory by the bulk-copy engine. Persistent CTAs walk (row group of 8,
// column chunk of 512) units in order; warp 8 bulk-copies each unit's 8 row
// chunks and the matching log v chunk into a ring of kLseStages stages
// (mbarrier transaction counts), so ~80 KB per CTA are in flight without
// registers. Consumer thread t owns column quad t & 127 of rows
// 4 (t >> 7) .. 4 (t >> 7) + 3 and keeps an online (max, sum) per row in fp32;
// at the end of a row group the 128 threads of each row set merge them.
constexpr int kLseChunk = 512;   // columns per unit
constexpr int kLseStages = 4;
struct LseSmem {
    float rows[kLseStages][kDenseRows][kLseChunk];
    double lv[kLseStages][kLseChunk];
    double wm[kWarps][4], ws[kWarps][4];
    uint64_t full[kLseStages], empty[kLseStages];
};

__global__ void __launch_bounds__(kThreads + 32, 2) dense_lse_tma_kernel(const DevState* __restrict__ st,
                                                                         const float* __restrict__ logk,
                                                                         long long rows, long long cols,
                                                                         const double* __restrict__ logv,
                                                                         double* __restrict__ M, double* __restrict__ S) {
    if (st->done) return;
    extern __shared__ __align__(128) unsigned char dyn[];
    LseSmem& sm = *reinterpret_cast<LseSmem*>(dyn);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long groups = (rows + kDenseRows - 1) / kDenseRows;
    const int nch = static_cast<int>((cols + kLseChunk - 1) / kLseChunk);
    if (tid == 0) {
        for (int k = 0; k < kLseStages; ++k) {
            mbar_init(&sm.full[k], 1);
            mbar_init(&sm.empty[k], kWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kWarps) {  // producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            bool wrapped = false;
            for (long long g = blockIdx.x; g < groups; g += gridDim.x) {
                const long long i0 = g * kDenseRows;
                const int nr = static_cast<int>(rows - i0 < kDenseRows ? rows - i0 : kDenseRows);
                for (int c = 0; c < nch; ++c) {
                    const long long j0 = static_cast<long long>(c) * kLseChunk;
                    const uint32_t w = static_cast<uint32_t>(cols - j0 < kLseChunk ? cols - j0 : kLseChunk);
                    if (wrapped) mbar_wait(&sm.empty[stage], phase ^ 1u);
                    mbar_arrive_expect_tx(&sm.full[stage], w * (4u * nr + 8u));
                    for (int r = 0; r < nr; ++r) bulk_g2s(sm.rows[stage][r], logk + (i0 + r) * cols + j0, w * 4u, &sm.full[stage]);
                    bulk_g2s(sm.lv[stage], logv + j0, w * 8u, &sm.full[stage]);
                    if (++stage == kLseStages) {
                        stage = 0;
                        phase ^= 1u;
                        wrapped = true;
                    }
                }
            }
        }
        return;
    }
    const int qi = tid & 127, h = tid >> 7;  // column quad, row set
    int stage = 0;
    uint32_t phase = 0;
    for (long long g = blockIdx.x; g < groups; g += gridDim.x) {
        const long long i0 = g * kDenseRows;
        const int nr = static_cast<int>(rows - i0 < kDenseRows ? rows - i0 : kDenseRows);
        float mf[4], sf[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) { mf[r] = -INFINITY; sf[r] = 0.0f; }
        for (int c = 0; c < nch; ++c) {
            const long long j0 = static_cast<long long>(c) * kLseChunk;
            const int w = static_cast<int>(cols - j0 < kLseChunk ? cols - j0 : kLseChunk);
            mbar_wait(&sm.full[stage], phase);
            if (4 * qi < w) {
                const double2 a0 = *reinterpret_cast<const double2*>(&sm.lv[stage][4 * qi]);
                const double2 a1 = *reinterpret_cast<const double2*>(&sm.lv[stage][4 * qi + 2]);
                const float l0 = static_cast<float>(a0.x), l1 = static_cast<float>(a0.y);
                const float l2 = static_cast<float>(a1.x), l3 = static_cast<float>(a1.y);
                // rows past nr (last group) reduce stale stage data; their pairs are dropped
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    {
                        const float4 x = *reinterpret_cast<const float4*>(&sm.rows[stage][4 * h + r][4 * qi]);
                        const float v0 = x.x + l0, v1 = x.y + l1, v2 = x.z + l2, v3 = x.w + l3;
                        const float bm = fmaxf(fmaxf(v0, v1), fmaxf(v2, v3));
                        if (bm > mf[r]) {
                            sf[r] *= ex2_ftz((mf[r] - bm) * kL2E);  // 2^-inf = 0 for the first batch
                            mf[r] = bm;
                        }
                        if (mf[r] != -INFINITY) {
                            const float ms = mf[r] * kL2E;
                            sf[r] += (ex2_ftz(fmaf(v0, kL2E, -ms)) + ex2_ftz(fmaf(v1, kL2E, -ms))) +
                                     (ex2_ftz(fmaf(v2, kL2E, -ms)) + ex2_ftz(fmaf(v3, kL2E, -ms)));
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (++stage == kLseStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        // merge the 128 threads of each row set: warps, then 4 warps via smem
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double m = mf[r] == -INFINITY ? kNegInf : static_cast<double>(mf[r]);
            double sv = static_cast<double>(sf[r]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sv, o);
                lse_pair_merge(m, sv, om, os);
            }
            if (lane == 0) { sm.wm[warp][r] = m; sm.ws[warp][r] = sv; }
        }
        consumers_sync();
        if (tid < nr) {
            const int hh = tid >> 2, r = tid & 3;
            double mm = kNegInf, ss = 0.0;
            for (int w = 4 * hh; w < 4 * hh + 4; ++w) lse_pair_merge(mm, ss, sm.wm[w][r], sm.ws[w][r]);
            M[i0 + tid] = mm;
            S[i0 + tid] = ss;
        }
        consumers_sync();  // wm / ws are rewritten by the next group
    }
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
// Streaming band kernels (warp-specialized). Both half-iterations stream
// bucket blocks along their reduction dimension and keep the outputs in
// registers ("output-stationary"):
//   column pass (K^T s): blocks n_b x row_stride(m_b), stream = sources,
//                        outputs = targets; corr_t[tgt] = sum_r delta ss_r
//   row pass (K t):      transposed blocks m_b x row_stride(n_b), stream =
//                        targets, outputs = sources; corr_s[src] = sum_c delta tt_c
// The band's work is a list of items (panel p of op.iter, stream rows s0 .. s0
// + ns, output columns o0 .. o0 + ow): wide panels are cut into <= kBandVec
// output tiles, long ones into stream pieces; the CTAs claim items largest
// first from a global counter (LCN_BAND_STATIC: host LPT ranges per CTA).
// Per CTA:
//   warp kWarps     bulk-copies the item's rows (one copy per chunk of whole
//                   rows, one per row for an output tile) through a ring of
//                   kBandStages shared stages (mbarrier transaction counts);
//   warp kWarps + 1 loads the item's stream scalings (exp(log v - H)), output
//                   indices and metadata into one of two slots;
//   8 consumer warps: thread (g, q) owns output quad q of stream rows g, g+ng,
//                   ... of every chunk, sums in registers; one shared-memory
//                   combine of the ng groups per item.
// An output split over K stream pieces goes through scratch: every piece writes
// its partials, the piece that finishes last (arrival counter) adds them in
// piece order, so results do not depend on CTA timing. Unsplit outputs are
// plain stores. Two CTAs per SM (112 KB smem each) keep 16 consumer warps.
// ---------------------------------------------------------------------------
constexpr int kBandStages = 5;
constexpr int kBandStageBytes = 16 * 1024;
constexpr int kBandVec = 1024;  // max item output width / item stream rows

// per item slot, resolved by producer 2 so consumers never touch global
// metadata (dependent L2 round trips at every item start otherwise)
struct ItemMeta {
    uint32_t ns, ow, split, pieces;
    double* part;  // this piece's scratch partials (split outputs), else null
};

constexpr int kBandQ = 8;     // item queue depth (producer 1 -> producer 2)
constexpr int kBandLook = 2;  // items claimed ahead of the one whose rows producer 1 copies

struct BandSmem {
    unsigned char ring[kBandStages][kBandStageBytes];
    uint32_t q[kBandQ];         // item indices in the order producer 1 claimed them
    uint64_t qfull[kBandQ], qempty[kBandQ];
    double vec[2][kBandVec];    // stream scalings per item slot (fp32 storage: float view)
    uint32_t out[2][kBandVec];  // output indices per item slot
    double red[kBandVec];       // per-group partial sums (groups x row width <= kBandVec)
    ItemMeta meta[2];
    uint64_t full[kBandStages], empty[kBandStages], vfull[2], vempty[2];
    uint32_t last;              // this CTA combines a split output
};

// One work item: stream rows [s0, s0 + ns) x outputs [o0, o0 + ow) of a panel,
// resolved on the host so the producers need no panel lookups.
struct BandItem {
    unsigned long long off;  // first stored entry (panel val_off + s0 * rs + o0)
    uint32_t rs;             // panel row stride (entries)
    uint32_t ns, ow, split;  // stream rows, outputs; split = sid << 8 | piece, or ~0u
    uint32_t va;             // bucket-ordered stream position of stored row s0
    uint32_t g0;             // stored rows of the item before the gap
    uint32_t gapn;           // stream rows in the gap
    uint32_t oa;             // o_order index of output o0
};

// Items are claimed dynamically (largest first): producer 1 of each CTA takes
// the next index from ctr[0]; the CTA that finishes last resets both counters.
struct BandWork {
    const BandItem* items;
    uint32_t nitems;
    uint32_t* ctr;            // [0] next item, [1] finished CTAs
    const uint32_t* cta_off;  // static mode (LCN_BAND_STATIC): CTA c takes items cta_off[c] .. cta_off[c + 1] - 1
    const uint2* splits;      // sid -> {scratch offset (doubles), pieces}
    uint32_t* counters;       // sid -> arrivals (reset by the combining CTA)
    double* scratch;
};

// rows per ring stage; a multiple of 8 keeps every chunk start 128-byte
// aligned (row bytes are a multiple of 16, block starts of 128)
template <typename T>
__device__ __forceinline__ int band_rows_per_stage(uint32_t ws) {
    int r = static_cast<int>(kBandStageBytes / (ws * sizeof(T)));
    if (r >= 8) r &= ~7;
    return r < 1 ? 1 : r;
}

// Split-output epilogue: partials of `count` outputs are in scratch at
// base + piece * count; the last piece to arrive sums them in order into
// corr[outi[c]]. Called by all consumer threads after they wrote their partials.
// log-sum-exp partials travel as a float2 (max, sum) in one double slot
__device__ __forceinline__ double pack_ms(float m, float s) {
    return __longlong_as_double(static_cast<long long>(__float_as_uint(m)) |
                                (static_cast<long long>(__float_as_uint(s)) << 32));
}
__device__ __forceinline__ float2 unpack_ms(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return make_float2(__uint_as_float(static_cast<unsigned>(b)), __uint_as_float(static_cast<unsigned>(b >> 32)));
}
// online log-sum-exp steps of the band consumers: fold entries d into the
// running (max m, sum s of exp(. - m)). An all -inf history keeps offset 0 so
// that exp(-inf - 0) = 0 (masked duplicates) instead of NaN.
__device__ __forceinline__ void lse_add4(float& m, float& s, float d0, float d1, float d2, float d3) {
    const float mn = fmaxf(fmaxf(m, fmaxf(d0, d1)), fmaxf(d2, d3));
    const float o = mn == -CUDART_INF_F ? 0.0f : mn;
    const float ol = o * kL2E;
    s = fmaf(s, ex2_ftz((m - o) * kL2E),
             (ex2_ftz(fmaf(d0, kL2E, -ol)) + ex2_ftz(fmaf(d1, kL2E, -ol))) +
                 (ex2_ftz(fmaf(d2, kL2E, -ol)) + ex2_ftz(fmaf(d3, kL2E, -ol))));
    m = mn;
}
__device__ __forceinline__ void lse_add1(float& m, float& s, float d) {
    const float mn = fmaxf(m, d);
    const float o = mn == -CUDART_INF_F ? 0.0f : mn;
    s = fmaf(s, ex2_ftz((m - o) * kL2E), ex2_ftz((d - o) * kL2E));
    m = mn;
}
// merge (m, s) into the output's running (M, S) (lse_merge in fp64)
__device__ __forceinline__ void lse_store(double* __restrict__ Mo, double* __restrict__ So, uint32_t i, float m, float s) {
    if (m == -CUDART_INF_F) return;
    double M = Mo[i], S = So[i];
    const double mm = static_cast<double>(m);
    if (mm > M) {
        S = S * exp(M - mm) + static_cast<double>(s);
        M = mm;
    } else {
        S += static_cast<double>(s) * exp(mm - M);
    }
    Mo[i] = M;
    So[i] = S;
}

template <bool LSE>
__device__ __forceinline__ void band_combine(BandSmem& sm, const BandWork& wk, const ItemMeta& mt, uint32_t count,
                                             const uint32_t* outi, double* __restrict__ corr, double* __restrict__ Sout,
                                             int tid) {
    __threadfence();
    consumers_sync();
    if (tid == 0) sm.last = atomicAdd(&wk.counters[mt.split >> 8], 1u) == mt.pieces - 1;
    consumers_sync();
    if (sm.last) {
        __threadfence();
        const double* base = mt.part - static_cast<size_t>(mt.split & 0xffu) * count;  // piece 0
        for (uint32_t c = tid; c < count; c += kThreads) {
            if constexpr (LSE) {
                float m = -CUDART_INF_F, sum = 0.0f;
                for (uint32_t k = 0; k < mt.pieces; ++k) {
                    const float2 ms = unpack_ms(__ldcg(base + static_cast<size_t>(k) * count + c));
                    if (ms.x == -CUDART_INF_F) continue;
                    if (ms.x > m) {
                        sum = sum * __expf(m - ms.x) + ms.y;
                        m = ms.x;
                    } else {
                        sum += ms.y * __expf(ms.x - m);
                    }
                }
                lse_store(corr, Sout, outi[c], m, sum);
            } else {
                double v = 0.0;
                for (uint32_t k = 0; k < mt.pieces; ++k) v += __ldcg(base + static_cast<size_t>(k) * count + c);
                corr[outi[c]] = v;
            }
        }
        if (tid == 0) wk.counters[mt.split >> 8] = 0u;
    }
}

// ROWS selects the row pass (transposed blocks). logv: the band's
// bucket-ordered copy of the stream side's log vector (log t for the row pass,
// log s for the column pass), written by the low-rank pass that produced it.
// LSE (the sparse operator's log-domain passes, sparse_kernel.cpp:119-155):
// vals are log K, the stream vector enters as log v, and each output gets a
// (max, sum exp(. - max)) merged into (corr = M, Sout = S); otherwise the
// linear LCN correction product.
template <typename T, bool ROWS, bool LSE = false>
__global__ void __launch_bounds__(kThreads + 64, 2) band_stream_kernel(const DevState* __restrict__ st,
                                                                      const uint32_t* __restrict__ o_order, BandWork wk, const T* __restrict__ vals,
                                                                      const double* __restrict__ logv,
                                                                      double* __restrict__ corr,
                                                                      double* __restrict__ Sout = nullptr,
                                                                      int late_wait = 0) {
    // Launched with programmatic serialisation inside the LCN iteration. A
    // later band of the same pass (late_wait) depends on nothing the band
    // before it writes: it starts as soon as that band's CTAs have all passed
    // their own wait (so everything earlier is complete), fills the SMs the
    // earlier band's tail leaves idle, and waits for it only before exiting,
    // which keeps "this grid complete" => "every earlier grid complete".
    // late_wait 2: no explicit trigger either; the dependent is launched when
    // this grid's CTAs exit, i.e. after their late wait (wait-then-trigger
    // order like every other kernel here).
    if (!late_wait) pdl_wait();
    if (late_wait != 2) pdl_launch_dependents();
    if (st->done) return;
    extern __shared__ __align__(128) unsigned char dyn[];
    BandSmem& sm = *reinterpret_cast<BandSmem*>(dyn);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double H = ROWS ? st->H_t : st->H_s;
    constexpr uint32_t kEnd = 0xffffffffu;
    if (tid == 0) {
        for (int k = 0; k < kBandStages; ++k) {
            mbar_init(&sm.full[k], 1);
            mbar_init(&sm.empty[k], kWarps);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&sm.vfull[k], 32);
            mbar_init(&sm.vempty[k], kWarps);
        }
        for (int k = 0; k < kBandQ; ++k) {
            mbar_init(&sm.qfull[k], 1);
            mbar_init(&sm.qempty[k], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kWarps) {
        // ---------------- producer 1: bulk copies of the item's rows ----------------
        // Items are claimed kBandLook ahead of the one being copied and
        // published to producer 2 at claim time, so the claim's atomic and
        // producer 2's scalings / output indices for the next item overlap
        // this item's stream instead of stalling the item boundary.
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            bool wrapped = false;
            const uint32_t s_beg = wk.cta_off ? wk.cta_off[blockIdx.x] : 0u;
            const uint32_t s_end = wk.cta_off ? wk.cta_off[blockIdx.x + 1] : 0u;
            uint32_t ids[kBandQ];
            uint32_t claimed = 0;
            bool ended = false;
            auto publish = [&]() {
                const uint32_t k = claimed++;
                uint32_t it = kEnd;
                if (!ended) {
                    const uint32_t c = wk.cta_off ? s_beg + k : atomicAdd(&wk.ctr[0], 1u);
                    it = c < (wk.cta_off ? s_end : wk.nitems) ? c : kEnd;
                }
                const int qs = static_cast<int>(k % kBandQ);
                if (k >= static_cast<uint32_t>(kBandQ)) mbar_wait(&sm.qempty[qs], ((k / kBandQ) - 1) & 1);
                sm.q[qs] = it;
                ids[qs] = it;
                mbar_arrive(&sm.qfull[qs]);  // release: the queue entry
                if (it == kEnd) ended = true;
            };
            for (int j = 0; j < kBandLook; ++j)
                if (!ended) publish();
            BandItem next{};
            if (ids[0] != kEnd) next = wk.items[ids[0]];
            for (uint32_t k = 0;; ++k) {
                const uint32_t it = ids[k % kBandQ];
                if (it == kEnd) break;
                if (!ended) publish();  // item k + kBandLook
                const BandItem item = next;
                const uint32_t it_next = ids[(k + 1) % kBandQ];
                if (it_next != kEnd) next = wk.items[it_next];  // in flight while this item is issued
                const uint32_t rs = item.rs;
                const uint32_t ws = static_cast<uint32_t>(row_stride(item.ow));  // item row width in the ring
                const int R = band_rows_per_stage<T>(ws);
                const T* blk = vals + item.off;
                for (uint32_t r0 = 0; r0 < item.ns; r0 += R) {
                    const uint32_t nr = item.ns - r0 < static_cast<uint32_t>(R) ? item.ns - r0 : static_cast<uint32_t>(R);
                    if (wrapped) mbar_wait(&sm.empty[stage], phase ^ 1u);
                    const uint32_t rb = ws * static_cast<uint32_t>(sizeof(T));
                    mbar_arrive_expect_tx(&sm.full[stage], nr * rb);
                    const T* src = blk + static_cast<unsigned long long>(r0) * rs;
                    if (ws == rs) {
                        bulk_g2s(sm.ring[stage], src, nr * rb, &sm.full[stage]);
                    } else {
                        for (uint32_t r = 0; r < nr; ++r)
                            bulk_g2s(sm.ring[stage] + r * rb, src + static_cast<unsigned long long>(r) * rs, rb,
                                     &sm.full[stage]);
                    }
                    if (++stage == kBandStages) {
                        stage = 0;
                        phase ^= 1u;
                        wrapped = true;
                    }
                }
            }
        }
        return;
    }
    if (warp == kWarps + 1) {
        // ---------------- producer 2: stream scalings, output indices, metadata ----------------
        for (uint32_t kb = 0;; ++kb) {
            const int qs = static_cast<int>(kb % kBandQ);
            mbar_wait(&sm.qfull[qs], (kb / kBandQ) & 1);
            const uint32_t it = sm.q[qs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.qempty[qs]);
            const int slot = kb & 1;
            if (kb >= 2) mbar_wait(&sm.vempty[slot], ((kb >> 1) - 1) & 1);
            if (it == kEnd) {
                if (lane == 0) sm.meta[slot].ns = kEnd;
                mbar_arrive(&sm.vfull[slot]);
                break;
            }
            const BandItem item = wk.items[it];
            // stored row c of the item is stream position c (c < g0) or c + gapn
            const double* va = logv + item.va;
            const double* vb = va + item.gapn;
            // 8 independent loads in flight per lane before the exps (one warp
            // resolves every stream row of the item; L2 latency bound otherwise)
            for (uint32_t c0 = lane; c0 < item.ns; c0 += 256) {
                double x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t c = c0 + 32u * k;
                    x[k] = c < item.ns ? (c < item.g0 ? va[c] : vb[c]) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t c = c0 + 32u * k;
                    if (c < item.ns) {
                        if constexpr (LSE)  // log domain: the stream value itself
                            reinterpret_cast<float*>(sm.vec[slot])[c] = static_cast<float>(x[k]);
                        else if constexpr (sizeof(T) == 4)  // fp32 storage: the scalings enter fp32 products
                            reinterpret_cast<float*>(sm.vec[slot])[c] = static_cast<float>(exp(x[k] - H));
                        else
                            sm.vec[slot][c] = exp(x[k] - H);
                    }
                }
            }
            for (uint32_t c = lane; c < item.ow; c += 32) sm.out[slot][c] = o_order[item.oa + c];
            if (lane == 0) {
                ItemMeta mt;
                mt.ns = item.ns;
                mt.ow = item.ow;
                mt.split = item.split;
                mt.pieces = 0;
                mt.part = nullptr;
                if (item.split != 0xffffffffu) {
                    const uint2 sp = wk.splits[item.split >> 8];
                    mt.pieces = sp.y;
                    mt.part = wk.scratch + sp.x + static_cast<size_t>(item.split & 0xffu) * item.ow;
                }
                sm.meta[slot] = mt;
            }
            mbar_arrive(&sm.vfull[slot]);  // all 32 lanes (release: their smem writes)
        }
        return;
    }
    // ---------------- consumers ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (uint32_t kb = 0;; ++kb) {
        const int slot = kb & 1;
        mbar_wait(&sm.vfull[slot], (kb >> 1) & 1);
        const ItemMeta mt = sm.meta[slot];
        if (mt.ns == kEnd) break;
        const uint32_t ws = static_cast<uint32_t>(row_stride(mt.ow));
        const uint32_t nq = ws / 4;
        const int R = band_rows_per_stage<T>(ws);
        // groups of nq threads: thread (g, q) owns output quad q of stream rows
        // g, g + ng, ... of every chunk
        const uint32_t ng = nq >= static_cast<uint32_t>(kThreads) ? 1u : kThreads / nq;
        const uint32_t g = static_cast<uint32_t>(tid) / nq, q = static_cast<uint32_t>(tid) % nq;
        const bool own = g < ng;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        float lm[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};  // LSE: running max / sum
        float ls[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        const uint32_t* outi = sm.out[slot];
        for (uint32_t r0 = 0; r0 < mt.ns; r0 += R) {
            const uint32_t nr = mt.ns - r0 < static_cast<uint32_t>(R) ? mt.ns - r0 : static_cast<uint32_t>(R);
            mbar_wait(&sm.full[stage], phase);
            const T* blk = reinterpret_cast<const T*>(sm.ring[stage]);
            if (own) {
                const T* p = blk + 4 * q;
                if constexpr (LSE) {
                    // log domain, one read of the staged chunk: blocks of four
                    // stream rows per thread, the running (max, sum) of each
                    // output rescaled once per block (5 exponentials per 4
                    // entries), single rows for the remainder
                    const float* vf = reinterpret_cast<const float*>(sm.vec[slot]) + r0;
                    uint32_t r = g;
                    for (; r + 3 * ng < nr; r += 4 * ng) {
                        const float4 x0 = *reinterpret_cast<const float4*>(p + r * ws);
                        const float4 x1 = *reinterpret_cast<const float4*>(p + (r + ng) * ws);
                        const float4 x2 = *reinterpret_cast<const float4*>(p + (r + 2 * ng) * ws);
                        const float4 x3 = *reinterpret_cast<const float4*>(p + (r + 3 * ng) * ws);
                        const float s0 = vf[r], s1 = vf[r + ng], s2 = vf[r + 2 * ng], s3 = vf[r + 3 * ng];
                        lse_add4(lm[0], ls[0], x0.x + s0, x1.x + s1, x2.x + s2, x3.x + s3);
                        lse_add4(lm[1], ls[1], x0.y + s0, x1.y + s1, x2.y + s2, x3.y + s3);
                        lse_add4(lm[2], ls[2], x0.z + s0, x1.z + s1, x2.z + s2, x3.z + s3);
                        lse_add4(lm[3], ls[3], x0.w + s0, x1.w + s1, x2.w + s2, x3.w + s3);
                    }
                    for (; r < nr; r += ng) {
                        const float4 x = *reinterpret_cast<const float4*>(p + r * ws);
                        const float sr = vf[r];
                        lse_add1(lm[0], ls[0], x.x + sr);
                        lse_add1(lm[1], ls[1], x.y + sr);
                        lse_add1(lm[2], ls[2], x.z + sr);
                        lse_add1(lm[3], ls[3], x.w + sr);
                    }
                } else if constexpr (sizeof(T) == 4) {
                    // fp32 products and per-chunk partials, widened once per chunk
                    const float* vf = reinterpret_cast<const float*>(sm.vec[slot]) + r0;
                    float f0 = 0.0f, f1 = 0.0f, f2 = 0.0f, f3 = 0.0f;
#pragma unroll 4
                    for (uint32_t r = g; r < nr; r += ng) {
                        const float4 x = *reinterpret_cast<const float4*>(p + r * ws);
                        const float sr = vf[r];
                        f0 = fmaf(x.x, sr, f0); f1 = fmaf(x.y, sr, f1);
                        f2 = fmaf(x.z, sr, f2); f3 = fmaf(x.w, sr, f3);
                    }
                    a0 += f0; a1 += f1; a2 += f2; a3 += f3;
                } else {
                    const double* vec = sm.vec[slot] + r0;
                    for (uint32_t r = g; r < nr; r += ng) {
                        const double2 x0 = *reinterpret_cast<const double2*>(p + r * ws);
                        const double2 x1 = *reinterpret_cast<const double2*>(p + r * ws + 2);
                        const double sr = vec[r];
                        a0 += x0.x * sr; a1 += x0.y * sr; a2 += x1.x * sr; a3 += x1.y * sr;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (++stage == kBandStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        // combine the groups: red[g * ws + c], one thread per output
        if (own) {
            double* o = sm.red + g * ws + 4 * q;
            if constexpr (LSE) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // -inf entries (masked duplicates) leave the sum at exactly 0
                    if (lm[k] == -CUDART_INF_F) ls[k] = 0.0f;
                    o[k] = pack_ms(lm[k], ls[k]);
                }
            } else {
                o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
            }
        }
        consumers_sync();
        double* part = mt.part;
        for (uint32_t c = tid; c < mt.ow; c += kThreads) {
            if constexpr (LSE) {
                float m = -CUDART_INF_F, sum = 0.0f;
                for (uint32_t gg = 0; gg < ng; ++gg) {
                    const float2 ms = unpack_ms(sm.red[gg * ws + c]);
                    if (ms.x == -CUDART_INF_F) continue;
                    if (ms.x > m) {
                        sum = sum * __expf(m - ms.x) + ms.y;
                        m = ms.x;
                    } else {
                        sum += ms.y * __expf(ms.x - m);
                    }
                }
                if (part) part[c] = pack_ms(m, sum);
                else lse_store(corr, Sout, outi[c], m, sum);
            } else {
                double v = 0.0;
                for (uint32_t gg = 0; gg < ng; ++gg) v += sm.red[gg * ws + c];
                if (part) part[c] = v;
                else corr[outi[c]] = v;
            }
        }
        if (part) band_combine<LSE>(sm, wk, mt, mt.ow, outi, corr, Sout, tid);
        consumers_sync();  // red is rewritten by the next item
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.vempty[slot]);
    }
    // every producer of this launch has claimed past the end before its CTA
    // gets here, so the last CTA may reset the claim counter for the next launch
    if (tid == 0 && atomicAdd(&wk.ctr[1], 1u) == gridDim.x - 1) {
        wk.ctr[0] = 0u;
        wk.ctr[1] = 0u;
    }
    if (late_wait && tid == 0) pdl_wait();
}

// ---------------------------------------------------------------------------
// Low-rank pass over the factor F (U: n x lp, or W^T: m x lp), streamed in
// tiles of kRT rows through a shared-memory ring by a producer warp; the tile
// carries the rows' scalar streams too (per-band corrections, log marginal,
// current log s, marginal). Consumer thread t owns columns CPT t .. CPT t +
// CPT - 1: row dots y_r = F_r . mid (warp transpose reduction + shared
// combine), per-row finalize in a dedicated warp (tile k's finalize overlaps
// the consumers' dots of tile k + 1), then the running partial
// sum_r F_r exp(v_r - h) of the next half's product.
//   mode 0 (iteration): row side (SIDE 0) / column side (SIDE 1) update
//   mode 1 (log_matvec): out[r] = H + log y_r, no partial
//   mode 2 (accumulate): partial of F^T exp(in - h) only (in == null -> 0)
// ---------------------------------------------------------------------------
constexpr int kRT = 16;  // rows per low-rank tile (transpose_reduce16)

struct PassArgs {
    DevState* st;
    long long rows;
    int l, lp;
    const double* mid;              // lp (row dots)
    const double* corr[kMaxBands];  // per-band correction products (rows)
    int ncorr;
    const double* log_marg;         // log p (row side) / log q (col side)
    const double* marg;             // p (row side, error) or null
    const double* log_cur;          // log s of this iteration (row side, row marginal)
    double* log_out;                // next log s (row side) / log t (col side)
    double* row_marg;
    double* err_part;
    int with_err;
    double* part;                   // [G x lp]
    double* hpart;                  // [G]
    double* mnp;                    // [G]
    double* mxp;                    // [G]
    int mode;
    const double* in;               // mode 2 input vector
    double* out;                    // mode 1 output
    // mode 0: also write v into each band's bucket-ordered copy, perm[b][pos[b][i]]
    const uint32_t* pos[kMaxBands];
    double* perm[kMaxBands];
    int nperm;
};

// Sum over the 32 lanes of each of 16 per-lane values with 16 shuffles instead
// of 16 x 5: at every step a lane keeps half of its values and trades the
// other half with its partner. On exit lane L holds the full sum of value
// (L >> 1) & 15 (both lanes of a pair hold the same row).
template <typename V>
__device__ __forceinline__ V transpose_reduce16(V (&v)[16], int lane) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // xor 16
        const bool hi = lane & 16;
        const V send = hi ? v[k] : v[k + 8];
        const V keep = hi ? v[k + 8] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // xor 8
        const bool hi = lane & 8;
        const V send = hi ? v[k] : v[k + 4];
        const V keep = hi ? v[k + 4] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // xor 4
        const bool hi = lane & 4;
        const V send = hi ? v[k] : v[k + 2];
        const V keep = hi ? v[k + 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {  // xor 2
        const bool hi = lane & 2;
        const V send = hi ? v[0] : v[1];
        const V keep = hi ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Per-row transcendentals of the low-rank finalize. In fp32-storage mode the
// operands carry fp32 rounding already, so log y and exp of non-positive
// arguments run on the fp32 MUFU path (range-safe: the exponent of y is split
// off in fp64 first); fp64 storage keeps them in fp64.
template <typename T>
__device__ __forceinline__ double fin_log(double y) {
    if constexpr (sizeof(T) == 4) {
        if (!(y > 0.0) || !(y < kPosInf)) return log(y);
        int e;
        const double mant = frexp(y, &e);  // [0.5, 1)
        return static_cast<double>(__logf(static_cast<float>(mant))) + e * 0.6931471805599453;
    } else {
        return log(y);
    }
}
template <typename T>
__device__ __forceinline__ double fin_exp(double x) {  // row marginal exp(log s + log Kt)
    if constexpr (sizeof(T) == 4)
        if (x > -80.0 && x < 80.0) return static_cast<double>(__expf(static_cast<float>(x)));
    return exp(x);
}
template <typename T>
__device__ __forceinline__ double fin_exp_neg(double x) {  // x <= 0
    if constexpr (sizeof(T) == 4) return x < -87.0 ? 0.0 : static_cast<double>(__expf(static_cast<float>(x)));
    else return exp(x);
}

template <typename T>
struct PassStages {
    static constexpr int kStages = 3;
};

template <typename T>
__host__ __device__ constexpr size_t pass_stage_bytes(int lp) {
    return static_cast<size_t>(kRT) * lp * sizeof(T) + (kMaxBands + 3) * kRT * sizeof(double) +
           kMaxBands * kRT * sizeof(uint32_t);
}

template <int CPT, typename T>
__device__ __forceinline__ void lds_cols(const T* p, double (&o)[CPT]) {
    if constexpr (CPT == 2 && sizeof(T) == 4) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        o[0] = v.x;
        o[1] = v.y;
    } else if constexpr (CPT == 4 && sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) o[k] = static_cast<double>(p[k]);
    }
}

template <typename T, int CPT, int SIDE>
__global__ void __launch_bounds__(kThreads + 64, 2) lowrank_pass_kernel(const T* __restrict__ F, PassArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    DevState* st = a.st;
    if (st->done) return;
    constexpr int S = PassStages<T>::kStages;
    extern __shared__ __align__(128) unsigned char dyn[];
    // full: producer -> consumers + finalize; empty: consumers (kWarps) +
    // finalize (1) -> producer; ydone: consumers' row dots -> finalize;
    // wready: finalize's weights -> consumers (double-buffered by tile parity)
    __shared__ __align__(8) uint64_t full[S], empty[S], ydone[2], wready[2];
    __shared__ double red[2][kWarps][kRT];
    __shared__ double w_s[2][kRT];
    __shared__ float w_f[2][kRT];
    __shared__ double sc_s[2], h_fin;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t stage_bytes = pass_stage_bytes<T>(a.lp);
    const uint32_t frow = static_cast<uint32_t>(a.lp * sizeof(T));
    // streams: [corr_0 .. corr_{nc-1}] [log marg] [log cur] [marg]; mode 2: [in]
    const int nc = a.mode == 2 ? 0 : a.ncorr;
    const int np = a.mode == 0 ? a.nperm : 0;
    const long long ntiles = (a.rows + kRT - 1) / kRT;
    if (tid == 0) {
        for (int k = 0; k < S; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kWarps + 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&ydone[k], kWarps);
            mbar_init(&wready[k], 32);
        }
        fence_mbar_init();
        h_fin = kNegInf;
    }
    __syncthreads();
    if (warp == kWarps) {
        // ---------------- producer: one lane per stream ----------------
        // lanes 0 .. kMaxBands + 2: scalar streams [corr_0 .. corr_{nc-1}]
        // [log marg] [log cur] [marg] (mode 2: [in]) into slot `lane`; lanes
        // 16 .. 16 + np - 1: the band position streams; lane 0 also copies the
        // factor tile. Pointers come straight from the kernel parameters (no
        // local-memory array), copies are issued by all lanes at once.
        const double* sp = nullptr;
        if (a.mode == 2) {
            if (lane == 0) sp = a.in;
        } else if (lane < nc) {
            sp = a.corr[lane];
        } else if (lane == nc) {
            sp = a.mode == 0 ? a.log_marg : nullptr;
        } else if (lane == nc + 1) {
            sp = (a.mode == 0 && SIDE == 0 && a.with_err) ? a.log_cur : nullptr;
        } else if (lane == nc + 2) {
            sp = (a.mode == 0 && SIDE == 0 && a.with_err) ? a.marg : nullptr;
        }
        const uint32_t* pp = (lane >= 16 && lane - 16 < np) ? a.pos[lane - 16] : nullptr;
        int it = 0;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int stage = it % S;
            const long long r0 = tile * kRT;
            const int nr = static_cast<int>(a.rows - r0 < kRT ? a.rows - r0 : kRT);
            const uint32_t sbytes = static_cast<uint32_t>((nr * 8 + 15) & ~15);  // vectors padded to kRT rows
            const uint32_t pbytes = static_cast<uint32_t>((nr * 4 + 15) & ~15);  // pos arrays padded by 16
            const uint32_t mine = (sp ? sbytes : 0u) + (pp ? pbytes : 0u) + (lane == 0 ? nr * frow : 0u);
            const uint32_t bytes = __reduce_add_sync(0xffffffffu, mine);
            if (lane == 0) {
                if (it >= S) mbar_wait(&empty[stage], ((it / S) - 1) & 1);
                mbar_arrive_expect_tx(&full[stage], bytes);
            }
            __syncwarp();
            unsigned char* base = dyn + stage * stage_bytes;
            double* sc = reinterpret_cast<double*>(base + static_cast<size_t>(kRT) * frow);
            uint32_t* ps = reinterpret_cast<uint32_t*>(sc + (kMaxBands + 3) * kRT);
            if (lane == 0) bulk_g2s(base, F + r0 * a.lp, nr * frow, &full[stage]);
            if (sp) bulk_g2s(sc + lane * kRT, sp + r0, sbytes, &full[stage]);
            if (pp) bulk_g2s(ps + (lane - 16) * kRT, pp + r0, pbytes, &full[stage]);
        }
        return;
    }
    if (warp == kWarps + 1) {
        // ---------------- finalize warp: lane r < kRT owns row r of the tile ----------------
        const double H = SIDE == 0 ? st->H_t : st->H_s;
        const int allpos = SIDE == 0 ? st->allpos_t : st->allpos_s;
        const bool has_in = a.mode == 2 && a.in != nullptr;
        double vmin = kPosInf, vmax = kNegInf, err = 0.0, h_run = kNegInf;
        unsigned fl = 0;
        int it = 0;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int stage = it % S, buf = it & 1;
            const long long r0 = tile * kRT;
            const int nr = static_cast<int>(a.rows - r0 < kRT ? a.rows - r0 : kRT);
            mbar_wait(&full[stage], (it / S) & 1);
            if (a.mode != 2) mbar_wait(&ydone[buf], (it >> 1) & 1);
            const double* scal =
                reinterpret_cast<const double*>(dyn + stage * stage_bytes + static_cast<size_t>(kRT) * frow);
            double v = kNegInf;
            bool live = lane < nr;
            if (live) {
                const long long i = r0 + lane;
                if (a.mode == 2) {
                    v = has_in ? scal[lane] : 0.0;
                } else {
                    double nys = 0.0;
#pragma unroll
                    for (int w = 0; w < kWarps; ++w) nys += red[buf][w][lane];
                    double y = nys;
                    for (int k = 0; k < nc; ++k) y += scal[k * kRT + lane];
                    if (allpos && !(nys > 0.0)) fl |= SIDE == 0 ? F_NYS_ROW : F_NYS_COL;
                    if (!(y > 0.0)) fl |= SIDE == 0 ? F_NEG_ROW : F_NEG_COL;
                    const double k = H + fin_log<T>(y);
                    if (a.mode == 1) {
                        a.out[i] = k;
                        live = false;
                    } else {
                        if (SIDE == 0 && a.with_err) {
                            const double rm = fin_exp<T>(scal[(nc + 1) * kRT + lane] + k);
                            a.row_marg[i] = rm;
                            err += fabs(rm - scal[(nc + 2) * kRT + lane]);
                        }
                        v = scal[nc * kRT + lane] - k;
                        a.log_out[i] = v;
                        const uint32_t* ps = reinterpret_cast<const uint32_t*>(scal + (kMaxBands + 3) * kRT);
                        for (int pb = 0; pb < np; ++pb) a.perm[pb][ps[pb * kRT + lane]] = v;
                        if (!isfinite(v)) fl |= SIDE == 0 ? F_LOGS : F_LOGT;
                    }
                }
                if (live) {
                    vmin = fmin(vmin, v);
                    vmax = fmax(vmax, v);
                }
            }
            if (a.mode != 1) {
                // tile shift: running max over the finite values
                const double tv = (live && v > kNegInf && v < kPosInf) ? v : kNegInf;
                double tmax = tv;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
                const double hn = fmax(h_run, tmax);
                if (lane < kRT) {
                    const double w = tv == kNegInf ? 0.0 : fin_exp_neg<T>(tv - hn);
                    w_s[buf][lane] = w;
                    w_f[buf][lane] = static_cast<float>(w);
                }
                if (lane == 0) {
                    sc_s[buf] = (h_run == kNegInf || hn == kNegInf) ? 0.0 : fin_exp_neg<T>(h_run - hn);
                    h_fin = hn;
                }
                h_run = hn;
            }
            mbar_arrive(&wready[buf]);  // all 32 lanes (release: their shared writes)
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
        }
        fl = __reduce_or_sync(0xffffffffu, fl);
        if (a.mode != 1) {
            vmin = -warp_max(-vmin);
            vmax = warp_max(vmax);
            err = warp_sum(err);
            if (lane == 0) {
                a.hpart[blockIdx.x] = h_run;
                a.mnp[blockIdx.x] = vmin;
                a.mxp[blockIdx.x] = vmax;
                if (SIDE == 0 && a.with_err) a.err_part[blockIdx.x] = err;
            }
        }
        if (lane == 0 && fl) atomicOr(&st->flags, fl);
        return;
    }
    // ---------------- consumers ----------------
    const int c0 = CPT * tid;
    const bool own = c0 < a.lp;
    double mid[CPT], acc[CPT];
    float mid_hi[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        mid[k] = (a.mode != 2 && own) ? a.mid[c0 + k] : 0.0;
        mid_hi[k] = static_cast<float>(mid[k]);
        acc[k] = 0.0;
    }
    // running partial of tile j (weights from the finalize warp)
    auto accumulate = [&](int j, int jnr) {
        const int jstage = j % S, jbuf = j & 1;
        mbar_wait(&wready[jbuf], (j >> 1) & 1);
        const T* fs = reinterpret_cast<const T*>(dyn + jstage * stage_bytes);
        if (own) {
            const double sc = sc_s[jbuf];
#pragma unroll
            for (int k = 0; k < CPT; ++k) acc[k] *= sc;
            if constexpr (sizeof(T) == 4) {
                // per-tile fp32 partial (kRT terms), widened once per tile
                float pa[CPT];
#pragma unroll
                for (int k = 0; k < CPT; ++k) pa[k] = 0.0f;
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    if (r < jnr) {
                        const float w = w_f[jbuf][r];
#pragma unroll
                        for (int k = 0; k < CPT; ++k) pa[k] = fmaf(fs[r * a.lp + c0 + k], w, pa[k]);
                    }
                }
#pragma unroll
                for (int k = 0; k < CPT; ++k) acc[k] += static_cast<double>(pa[k]);
            } else {
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    if (r < jnr) {
                        double u[CPT];
                        lds_cols<CPT>(fs + r * a.lp + c0, u);
                        const double w = w_s[jbuf][r];
#pragma unroll
                        for (int k = 0; k < CPT; ++k) acc[k] += u[k] * w;
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[jstage]);
    };
    int it = 0, prev_nr = 0;
    // fp32 storage with <= 2 columns per thread: the tile's factor values stay
    // in registers from the dot to the lagged accumulate, so the stage goes
    // back to the producer right after the dot (two of three stages prefetch)
    constexpr bool kReg = sizeof(T) == 4 && CPT <= 2;
    float uc[kReg ? kRT : 1][CPT], up[kReg ? kRT : 1][CPT];
    if constexpr (kReg) {
#pragma unroll
        for (int r = 0; r < kRT; ++r)
#pragma unroll
            for (int k = 0; k < CPT; ++k) up[r][k] = 0.0f;
    }
    auto accumulate_reg = [&](int j, int jnr) {
        const int jbuf = j & 1;
        mbar_wait(&wready[jbuf], (j >> 1) & 1);
        if (own) {
            const double sc = sc_s[jbuf];
            float pa[CPT];
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                acc[k] *= sc;
                pa[k] = 0.0f;
            }
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                const float w = w_f[jbuf][r];  // 0 for rows past jnr
#pragma unroll
                for (int k = 0; k < CPT; ++k) pa[k] = fmaf(up[r][k], w, pa[k]);
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) acc[k] += static_cast<double>(pa[k]);
        }
        (void)jnr;
    };
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int stage = it % S, buf = it & 1;
        const long long r0 = tile * kRT;
        const int nr = static_cast<int>(a.rows - r0 < kRT ? a.rows - r0 : kRT);
        mbar_wait(&full[stage], (it / S) & 1);
        if constexpr (kReg) {
            const float* fsf = reinterpret_cast<const float*>(dyn + stage * stage_bytes);
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                if (own && r < nr) {
                    if constexpr (CPT == 2) {
                        const float2 x = *reinterpret_cast<const float2*>(fsf + r * a.lp + c0);
                        uc[r][0] = x.x;
                        uc[r][CPT - 1] = x.y;
                    } else {
                        uc[r][0] = fsf[r * a.lp + c0];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < CPT; ++k) uc[r][k] = 0.0f;  // never stale smem (could be NaN)
                }
            }
            if (a.mode != 2) {
                if (a.mode == 1 && it >= 2) mbar_wait(&wready[buf], ((it - 2) >> 1) & 1);
                float dp[kRT];
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    float d = uc[r][0] * mid_hi[0];
#pragma unroll
                    for (int k = 1; k < CPT; ++k) d = fmaf(uc[r][k], mid_hi[k], d);
                    dp[r] = d;
                }
                const float wsum = transpose_reduce16(dp, lane);
                if ((lane & 1) == 0) red[buf][warp][(lane >> 1) & 15] = static_cast<double>(wsum);
                __syncwarp();
                if (lane == 0) mbar_arrive(&ydone[buf]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);  // the tile lives in registers now
            if (a.mode != 1 && it > 0) accumulate_reg(it - 1, prev_nr);  // overlaps the finalize of tile `it`
#pragma unroll
            for (int r = 0; r < kRT; ++r)
#pragma unroll
                for (int k = 0; k < CPT; ++k) up[r][k] = uc[r][k];
            prev_nr = nr;
            continue;
        }
        if (a.mode != 2) {
            // red[buf] is free once the finalize warp is done with tile it - 2
            // (implied by the accumulate wait below except in mode 1)
            if (a.mode == 1 && it >= 2) mbar_wait(&wready[buf], ((it - 2) >> 1) & 1);
            const T* fs = reinterpret_cast<const T*>(dyn + stage * stage_bytes);
            // row dots y_r = F_r . mid: per-thread partials, warp transpose
            // reduction, the kWarps warp sums meet in the finalize warp
            if constexpr (sizeof(T) == 4) {
                // fp32 storage: fp32 products and warp sums (the factor rows
                // carry fp32 rounding already), widened per warp sum. Rows past
                // nr hold stale data; their sums are never read.
                float dp[kRT];
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    float d = 0.0f;
                    if (own) {
                        const float* u = reinterpret_cast<const float*>(fs) + r * a.lp + c0;
                        const float4 x = *reinterpret_cast<const float4*>(u);
                        d = fmaf(x.w, mid_hi[CPT - 1], fmaf(x.z, mid_hi[CPT > 2 ? 2 : 0],
                                 fmaf(x.y, mid_hi[CPT > 1 ? 1 : 0], x.x * mid_hi[0])));
                    }
                    dp[r] = d;
                }
                const float wsum = transpose_reduce16(dp, lane);
                if ((lane & 1) == 0) red[buf][warp][(lane >> 1) & 15] = static_cast<double>(wsum);
            } else {
                double dp[kRT];
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    double d = 0.0;
                    if (own && r < nr) {
                        double u[CPT];
                        lds_cols<CPT>(fs + r * a.lp + c0, u);
#pragma unroll
                        for (int k = 0; k < CPT; ++k) d += u[k] * mid[k];
                    }
                    dp[r] = d;
                }
                const double wsum = transpose_reduce16(dp, lane);
                if ((lane & 1) == 0) red[buf][warp][(lane >> 1) & 15] = wsum;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ydone[buf]);
        }
        if (a.mode == 1) {
            if (lane == 0) mbar_arrive(&empty[stage]);
        } else if (it > 0) {
            accumulate(it - 1, prev_nr);  // overlaps the finalize of tile `it`
        }
        prev_nr = nr;
    }
    if (a.mode == 1) return;
    if (it > 0) {
        if constexpr (kReg) accumulate_reg(it - 1, prev_nr);
        else accumulate(it - 1, prev_nr);
    }
    consumers_sync();
    const double hb = h_fin;  // final CTA shift (written before the last wready)
#pragma unroll
    for (int k = 0; k < CPT; ++k)
        if (own) a.part[static_cast<long long>(blockIdx.x) * a.lp + c0 + k] = hb == kNegInf ? 0.0 : acc[k];
}

// ---------------------------------------------------------------------------
// Global shift and mid = sum_b exp(h_b - H) part_b over the G CTA partials;
// which: 0 -> t side, 1 -> s side. One CTA per 32 columns: lane = column,
// warps split the partials, shared memory combines them.
__global__ void __launch_bounds__(1024) lowrank_reduce_kernel(DevState* __restrict__ st, const double* __restrict__ part,
                                                              const double* __restrict__ hpart,
                                                              const double* __restrict__ mnp, int G, int lp,
                                                              double* __restrict__ mid, int which,
                                                              double* __restrict__ hloc) {
    pdl_wait();
    pdl_launch_dependents();
    if (st->done) return;
    constexpr int W = 32;  // warps
    __shared__ double sh[W], sm[W], acc_s[W][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double H = kNegInf, mn = kPosInf;
    for (int b = threadIdx.x; b < G; b += 1024) {
        H = fmax(H, hpart[b]);
        mn = fmin(mn, mnp[b]);
    }
    H = warp_max(H);
    mn = -warp_max(-mn);
    if (lane == 0) { sh[warp] = H; sm[warp] = mn; }
    __syncthreads();
    H = kNegInf;
    mn = kPosInf;
#pragma unroll
    for (int w = 0; w < W; ++w) { H = fmax(H, sh[w]); mn = fmin(mn, sm[w]); }
    const int a = blockIdx.x * 32 + lane;
    double s = 0.0;
    // exp(h_b - H) once per partial (thread b) instead of once per lane and
    // partial; -1 marks a partial to skip (h_b = -inf). Same products, same order.
    __shared__ double eb[1024];
    const bool cached = G <= 1024;
    if (cached && static_cast<int>(threadIdx.x) < G) {
        const double hb = hpart[threadIdx.x];
        eb[threadIdx.x] = (H != kNegInf && hb != kNegInf) ? exp(hb - H) : -1.0;
    }
    __syncthreads();
    if (H != kNegInf && a < lp) {
        if (cached) {
#pragma unroll 4
            for (int b = warp; b < G; b += W) {
                const double e = eb[b];
                if (e >= 0.0) s += part[static_cast<long long>(b) * lp + a] * e;
            }
        } else {
#pragma unroll 4
            for (int b = warp; b < G; b += W) {
                const double hb = hpart[b];
                if (hb != kNegInf) s += part[static_cast<long long>(b) * lp + a] * exp(hb - H);
            }
        }
    }
    acc_s[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && a < lp) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) t += acc_s[w][lane];
        mid[a] = t;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // positive_input of nys_matvec(_t) (nystrom.cpp:139-141): every exp(v - H) > 0.
        int allpos = H != kNegInf && exp(mn - H) > 0.0;
        if (which == 0) { st->H_t = H; st->allpos_t = allpos; }
        else { st->H_s = H; st->allpos_s = allpos; }
        if (hloc) {  // sharded: this rank's shift and minimum, combined across ranks next
            hloc[0] = H;
            hloc[1] = mn;
        }
    }
}

// ---- bucket-sharded solve (op.cuh ShardState) -----------------------------
// Per half-iteration every rank all-gathers one packed record of
// kShardHdr + lp + max_exp doubles: [H, mn, err, flags x 8, pad | low-rank
// partial (lp) | exported scalings (slot order)].
constexpr int kShardHdr = 16;

__global__ void shard_pack_kernel(const double* __restrict__ vec, const uint32_t* __restrict__ exp_idx, long long cnt,
                                  double* __restrict__ slots) {
    for (long long k = blockIdx.x * 256LL + threadIdx.x; k < cnt; k += 256LL * gridDim.x) slots[k] = vec[exp_idx[k]];
}

// halo points of one side: owner rank and slot per halo point (local index
// own + k), written into the log vector and every band's bucket-ordered copy
struct HaloUnpack {
    const uint32_t* rank;
    const uint32_t* slot;
    long long cnt, own;
    double* vec;
    const uint32_t* pos[kMaxBands];
    double* perm[kMaxBands];
    int nperm;
};

// Block 0: global shift H = max_r H_r and minimum, mid = sum_r exp(H_r - H)
// mid_r in rank order (identical on every rank), the positivity flag, and
// (row side) the marginal error and error-flag counts summed over the ranks
// for iter_end. Other blocks: the halo scalings.
__global__ void __launch_bounds__(256) shard_combine_kernel(DevState* __restrict__ st, const double* __restrict__ recv,
                                                            int world, long long stride, int lp,
                                                            double* __restrict__ mid, int which,
                                                            double* __restrict__ gstage, HaloUnpack hu) {
    if (st->done) return;
    if (blockIdx.x == 0) {
        double H = kNegInf, mn = kPosInf;
        for (int r = 0; r < world; ++r) {
            H = fmax(H, recv[r * stride]);
            mn = fmin(mn, recv[r * stride + 1]);
        }
        for (int a = threadIdx.x; a < lp; a += blockDim.x) {
            double acc = 0.0;
            for (int r = 0; r < world; ++r) {
                const double hr = recv[r * stride];
                if (hr != kNegInf) acc += recv[r * stride + kShardHdr + a] * exp(hr - H);
            }
            mid[a] = acc;
        }
        if (threadIdx.x == 0) {
            const int allpos = H != kNegInf && exp(mn - H) > 0.0;
            if (which == 0) { st->H_t = H; st->allpos_t = allpos; }
            else { st->H_s = H; st->allpos_s = allpos; }
            if (gstage) {
                double e = 0.0;
                for (int r = 0; r < world; ++r) e += recv[r * stride + 2];
                gstage[0] = e;
                for (int k = 0; k < 8; ++k) {
                    double f = 0.0;
                    for (int r = 0; r < world; ++r) f += recv[r * stride + 3 + k];
                    gstage[1 + k] = f;
                }
            }
        }
        return;
    }
    const long long step = 256LL * (gridDim.x - 1);
    for (long long k = (blockIdx.x - 1) * 256LL + threadIdx.x; k < hu.cnt; k += step) {
        const double v = recv[static_cast<long long>(hu.rank[k]) * stride + kShardHdr + lp + hu.slot[k]];
        const long long li = hu.own + k;
        hu.vec[li] = v;
        for (int b = 0; b < hu.nperm; ++b) hu.perm[b][hu.pos[b][li]] = v;
    }
}

__global__ void gather_marg_kernel(const double* __restrict__ g, const uint32_t* __restrict__ idx, long long cnt,
                                   double* __restrict__ out) {
    for (long long k = blockIdx.x * 256LL + threadIdx.x; k < cnt; k += 256LL * gridDim.x) out[k] = g[idx[k]];
}

// Sharded solve: this rank's marginal-error partial and error flags (as
// per-bit counts) into its exchange record, summed across ranks before
// iter_end.
__global__ void __launch_bounds__(256) stage_err_kernel(const DevState* __restrict__ st,
                                                        const double* __restrict__ err_part, int G, int it,
                                                        double* __restrict__ gstage) {
    __shared__ double red[8];
    double e = 0.0;
    if (it > 0)
        for (int b = threadIdx.x; b < G; b += 256) e += err_part[b];
    e = warp_sum(e);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        gstage[0] = t;
        const unsigned f = st->flags;
        for (int k = 0; k < 8; ++k) gstage[1 + k] = (f >> k) & 1u ? 1.0 : 0.0;
    }
}

// End of iteration `it` (0 = the initial K(log t = 0)): error precedence in
// the reference's order, marginal error, trace, convergence.
__global__ void __launch_bounds__(256) iter_end_kernel(DevState* __restrict__ st, const double* __restrict__ err_part,
                                                       int G, int it, int max_iters, double tol,
                                                       double* __restrict__ trace,
                                                       const double* __restrict__ gstage) {
    pdl_wait();
    pdl_launch_dependents();
    if (st->done) return;
    __shared__ double red[8];
    double e = 0.0;
    if (it > 0 && !gstage)
        for (int b = threadIdx.x; b < G; b += 256) e += err_part[b];
    e = warp_sum(e);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x != 0) return;
    e = 0.0;
    for (int w = 0; w < 8; ++w) e += red[w];
    unsigned f = st->flags;
    if (gstage) {  // sharded: error and flags summed over the ranks
        e = it > 0 ? gstage[0] : 0.0;
        f = 0u;
        for (int k = 0; k < 8; ++k)
            if (gstage[1 + k] > 0.5) f |= 1u << k;
    }
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

__global__ void perm_scatter_kernel(const double* __restrict__ in, long long n, const uint32_t* __restrict__ pos,
                                    double* __restrict__ out) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) out[pos[i]] = in[i];
}

__global__ void log_kernel(const double* __restrict__ in, double* __restrict__ out, long long n) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) out[i] = log(in[i]);
}

}  // namespace

// ---------------------------------------------------------------------------
// Host driver
// ---------------------------------------------------------------------------
// ---- BP extension (operator.cpp:226-266, sinkhorn.cpp:115-120) -------------
__device__ __forceinline__ double lse2_dev(double a, double b) {  // operator.cpp:14-19
    if (a == kNegInf) return b;
    if (b == kNegInf) return a;
    const double hi = fmax(a, b);
    return hi + log(exp(a - hi) + exp(b - hi));
}

// log sum exp of x (n), one CTA: max, then the shifted sum (operator.cpp:22-29)
__global__ void __launch_bounds__(1024) lse_one_kernel(const double* __restrict__ x, long long n, double* __restrict__ out) {
    __shared__ double red[32];
    double hi = kNegInf;
    for (long long i = threadIdx.x; i < n; i += 1024) hi = fmax(hi, x[i]);
    for (int o = 16; o > 0; o >>= 1) hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = hi;
    __syncthreads();
    hi = kNegInf;
    for (int k = 0; k < 32; ++k) hi = fmax(hi, red[k]);
    __syncthreads();
    double acc = 0.0;
    if (hi != kNegInf)
        for (long long i = threadIdx.x; i < n; i += 1024) acc += exp(x[i] - hi);
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 32; ++k) t += red[k];
        *out = hi == kNegInf ? kNegInf : hi + log(t);
    }
}

// K_BP v = [base + c_a (.) lower ; c_b (.) upper + (1^T lower) 1] in logs:
// y[k < na] = lse2(base[k], lda[k] + lower[k]); y[na + k] = lse2(ldb[k] + upper[k], total).
// out = log_marg - y (the scaling update) or y itself (log_marg == null);
// non-finite outputs raise *bad.
__global__ void bp_combine_kernel(const double* __restrict__ base, const double* __restrict__ lda,
                                  const double* __restrict__ lower, const double* __restrict__ ldb,
                                  const double* __restrict__ upper, const double* __restrict__ total, long long na,
                                  long long nb, const double* __restrict__ log_marg, double* __restrict__ out,
                                  unsigned* __restrict__ bad) {
    const long long k = blockIdx.x * 256LL + threadIdx.x;
    if (k >= na + nb) return;
    const double y = k < na ? lse2_dev(base[k], lda[k] + lower[k]) : lse2_dev(ldb[k - na] + upper[k - na], *total);
    const double v = log_marg ? log_marg[k] - y : y;
    out[k] = v;
    if (log_marg && !isfinite(v)) atomicOr(bad, 1u);
}

// row marginal exp(log s + K_BP t) and the partial of sum |rm - p|
__global__ void bp_err_kernel(const double* __restrict__ ls, const double* __restrict__ kt, const double* __restrict__ p,
                              long long rows, double* __restrict__ rm, double* __restrict__ part) {
    __shared__ double red[8];
    double e = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < rows; i += 256LL * gridDim.x) {
        const double v = exp(ls[i] + kt[i]);
        rm[i] = v;
        e += fabs(v - p[i]);
    }
    e = warp_sum(e);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                           double* __restrict__ out, unsigned* __restrict__ bad) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i >= n) return;
    const double v = a[i] - b[i];
    out[i] = v;
    if (!isfinite(v)) atomicOr(bad, 1u);
}

// BP plan quadrants (sinkhorn.cpp:82-98): deletion masses
// del_p[i] exp(log s_i + log t_{m+i}), del_q[j] exp(log s_{n+j} + log t_j)
__global__ void bp_mass_kernel(const double* __restrict__ ldp, const double* __restrict__ ldq,
                               const double* __restrict__ ls, const double* __restrict__ lt, long long n, long long m,
                               double* __restrict__ dpm, double* __restrict__ dqm) {
    const long long k = blockIdx.x * 256LL + threadIdx.x;
    if (k < n) dpm[k] = exp(ldp[k]) * exp(ls[k] + lt[m + k]);
    else if (k < n + m) dqm[k - n] = exp(ldq[k - n]) * exp(ls[n + (k - n)] + lt[k - n]);
}

__global__ void exp_sum_partial_kernel(const double* __restrict__ x, long long n, double* __restrict__ part) {
    __shared__ double red[8];
    double acc = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) acc += exp(x[i]);
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

__global__ void negate_kernel(double* __restrict__ x, long long n) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) x[i] = -x[i];
}

__global__ void log_dev_kernel(const double* __restrict__ in, long long n, double* __restrict__ out) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) out[i] = log(in[i]);
}

struct Solver {
    Op& op;
    Ctx& ctx;
    cudaStream_t s;
    long long n, m;
    int l, lp, G, CPT;
    DevBuf<DevState> st;
    DevBuf<double> log_p, log_q, pv, qv, log_s[2], log_t, row_marg, err_part, trace;
    DevBuf<double> Mr, Sr, Mc, Sc;                          // sparse band accumulators
    std::vector<DevBuf<double>> corr_s, corr_t;             // lcn: one correction product per band
    std::vector<DevBuf<double>> ltp, lsp[2];                // per-band bucket-ordered log t / log s copies
    DevBuf<double> part, hpart, mnp, mxp, mid_s, mid_t;     // low-rank reductions
    DevBuf<double> dpart;                                   // distance / mass partials
    std::vector<cudaEvent_t> evs;                           // phase events (profiling)
    size_t mark_base = 0;
    size_t smem = 0;                                        // low-rank pass stage ring
    // band work per pass ([0] row pass on the transposed blocks, [1] column
    // pass): items (stream pieces x output tiles of the panels), largest
    // first, claimed dynamically by the CTAs; the pass's split table
    struct PassPlan {
        DevBuf<BandItem> items;
        DevBuf<uint32_t> ctr, counters, cta_off;
        bool stat = false;
        DevBuf<uint2> splits;
        DevBuf<double> scratch;
        int nitems = 0;
        BandWork work() {
            return BandWork{items.get(), static_cast<uint32_t>(nitems), ctr.get(), stat ? cta_off.get() : nullptr,
                            splits.get(), counters.get(), scratch.get()};
        }
    };
    std::vector<PassPlan> plans[2];
    int band_grid = 0;
    int lse_grid = 0;  // dense_lse_tma_kernel: persistent CTAs
    // ---- bucket-sharded solve (op.shard): this rank's local operator; the
    // low-rank passes run over the owned rows [0, n_own) / [0, m_own); one
    // all-gather per half-iteration (comm.cuh)
    ShardState* sh = nullptr;
    Comm* comm = nullptr;
    long long n_own = 0, m_own = 0;
    long long stride_s = 0, stride_t = 0;             // doubles per rank record
    DevBuf<double> send_s, recv_s, send_t, recv_t, gstage;

    explicit Solver(Op& o) : op(o), ctx(*o.ctx), s(o.ctx->stream), n(o.n), m(o.m), l(static_cast<int>(o.l)) {
        n_own = n;
        m_own = m;
        if (op.shard) {
            if (op.kind != 3) throw Status(2, "sharded solve: only the LCN operator is sharded on this path");
            sh = op.shard.get();
            comm = sh->comm.get();
            n_own = sh->n_own;
            m_own = sh->m_own;
        }
        lp = static_cast<int>(o.lp);
        CPT = lp <= kThreads ? 1 : lp <= 2 * kThreads ? 2 : 4;
        if (lp > 4 * kThreads) throw Status(2, "lcn: landmark count above 1024 is not supported on this path");
        int occ = 1;
        if (op.kind >= 2) {
            smem = op.fp64 ? PassStages<double>::kStages * pass_stage_bytes<double>(lp)
                           : PassStages<float>::kStages * pass_stage_bytes<float>(lp);
            if (op.fp64) set_attrs<double>();
            else set_attrs<float>();
            if (op.fp64)
                CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lowrank_pass_kernel<double, 2, 0>, kThreads + 64, smem));
            else
                CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lowrank_pass_kernel<float, 2, 0>, kThreads + 64, smem));
        }
        G = std::max(1, occ) * ctx.num_sms;
        if (op.kind == 3 || lse_stream()) init_band_stream();
        if (op.kind == 0) {
            const int bytes = static_cast<int>(sizeof(LseSmem));
            CUDA_OK(cudaFuncSetAttribute(dense_lse_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            int o = 1;
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, dense_lse_tma_kernel, kThreads + 32, bytes));
            lse_grid = std::max(1, o) * ctx.num_sms;
        }
    }
    ~Solver() {
        for (auto e : evs) cudaEventDestroy(e);
    }

    template <typename T>
    void set_attrs() {
        const int b = static_cast<int>(smem);
        CUDA_OK(cudaFuncSetAttribute(lowrank_pass_kernel<T, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CUDA_OK(cudaFuncSetAttribute(lowrank_pass_kernel<T, 2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CUDA_OK(cudaFuncSetAttribute(lowrank_pass_kernel<T, 4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CUDA_OK(cudaFuncSetAttribute(lowrank_pass_kernel<T, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CUDA_OK(cudaFuncSetAttribute(lowrank_pass_kernel<T, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CUDA_OK(cudaFuncSetAttribute(lowrank_pass_kernel<T, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    }

    void init_band_stream() {
        const int bytes = static_cast<int>(sizeof(BandSmem));
        CUDA_OK(cudaFuncSetAttribute(band_stream_kernel<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        CUDA_OK(cudaFuncSetAttribute(band_stream_kernel<float, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bytes));
        CUDA_OK(cudaFuncSetAttribute(band_stream_kernel<float, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bytes));
        CUDA_OK(cudaFuncSetAttribute(band_stream_kernel<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        CUDA_OK(cudaFuncSetAttribute(band_stream_kernel<double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        CUDA_OK(cudaFuncSetAttribute(band_stream_kernel<double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        int occ = 1;
        if (op.fp64)
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, band_stream_kernel<double, true>, kThreads + 64,
                                                                  sizeof(BandSmem)));
        else
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, band_stream_kernel<float, true>, kThreads + 64,
                                                                  sizeof(BandSmem)));
        band_grid = std::max(occ, 1) * ctx.num_sms;
        for (size_t b = 0; b < op.bands.size(); ++b) {
            const Band& B = op.bands[b];
            std::vector<uint32_t> w(B.n_work);
            if (B.n_work) B.work.download(w.data(), B.n_work, s);
            ctx.sync();
            const BandIter& I = op.iter[b];
            plans[0].push_back(plan_pass(B, I, needed_buckets(b, w, true), true));
            plans[1].push_back(plan_pass(B, I, needed_buckets(b, w, false), false));
        }
        ctx.sync();
    }

    // Sharded solve: a pass skips the buckets whose outputs are all halo
    // points (their values come from the owner ranks).
    std::vector<uint32_t> needed_buckets(size_t b, const std::vector<uint32_t>& w, bool rows) const {
        if (!sh) return w;
        const std::vector<uint8_t>& need = rows ? sh->rows_need[b] : sh->cols_need[b];
        std::vector<uint32_t> out;
        for (uint32_t k : w)
            if (k < need.size() && need[k]) out.push_back(k);
        return out;
    }

    // Items of one pass: per panel of an owned bucket (BandPanel, op.cuh),
    // output tiles of <= kBandVec columns and stream pieces (multiples of 8
    // rows, <= kBandVec, sized so no piece exceeds half a CTA's share), then
    // longest-processing-time greedy.
    PassPlan plan_pass(const Band& B, const BandIter& I, const std::vector<uint32_t>& owned, bool rows) {
        const size_t esz = op.fp64 ? 8 : 4;
        // cost model (bytes): streamed bytes + per-row and per-item overheads
        auto cost_of = [&](size_t nr, size_t ws) { return double(nr * ws * esz) + 64.0 * nr + 4096.0; };
        std::vector<char> mine(B.nb, 0);
        for (uint32_t k : owned) mine[k] = 1;
        const std::vector<BandPanel>& panels = I.h_panels[rows ? 0 : 1];
        std::vector<uint32_t> w;  // panels of the owned buckets
        for (size_t p = 0; p < panels.size(); ++p)
            if (mine[panels[p].bucket]) w.push_back(static_cast<uint32_t>(p));
        auto lens = [&](uint32_t k, size_t& sl, size_t& ol) {
            sl = panels[k].ns;
            ol = panels[k].ow;
        };
        double total = 0.0;
        for (uint32_t k : w) {
            size_t sl, ol;
            lens(k, sl, ol);
            if (sl && ol) total += cost_of(sl, row_stride(ol));
        }
        // pieces per CTA share (LCN_BAND_CAP_DIV, read per plan like
        // LCN_BAND_STATIC; 4 measured ~2 % faster than 2)
        const char* cap_env = std::getenv("LCN_BAND_CAP_DIV");
        const double cap_div = cap_env && *cap_env ? std::max(1.0, std::atof(cap_env)) : 4.0;
        const double cap = std::max(total / band_grid / cap_div, 65536.0);
        struct Piece { BandItem it; double cost; };
        std::vector<Piece> pieces;
        std::vector<uint2> splits;
        size_t scratch = 0;
        for (uint32_t k : w) {
            size_t sl, ol;
            lens(k, sl, ol);
            if (sl == 0 || ol == 0) continue;
            const size_t rs = row_stride(ol);
            const size_t nct = ceil_div(ol, kBandVec);  // output tiles (a bucket wider than kBandVec)
            const size_t wmax = std::min<size_t>(rs, kBandVec);
            size_t K = static_cast<size_t>(std::ceil(cost_of(sl, wmax) / cap));
            K = std::max<size_t>(K, ceil_div(sl, kBandVec));
            size_t pr = (ceil_div(sl, std::max<size_t>(K, 1)) + 7) & ~size_t(7);
            pr = std::min<size_t>(std::max<size_t>(pr, 8), kBandVec);
            // the piece index is 8 bits: a long bucket gets longer pieces
            // rather than more of them (one dominant bucket, small problems)
            pr = std::max<size_t>(pr, (ceil_div(sl, 255) + 7) & ~size_t(7));
            if (pr > kBandVec) throw Status(2, "lcn: bucket longer than 255 band pieces");
            K = ceil_div(sl, pr);
            for (size_t ct = 0; ct < nct; ++ct) {
                const size_t o0 = ct * kBandVec, ow = std::min<size_t>(kBandVec, ol - o0);
                uint32_t sid = 0xffffffffu;
                if (K > 1) {
                    sid = static_cast<uint32_t>(splits.size());
                    splits.push_back(make_uint2(static_cast<uint32_t>(scratch), static_cast<uint32_t>(K)));
                    scratch += K * ow;
                }
                for (size_t j = 0; j < K; ++j) {
                    const size_t s0 = j * pr, ns = std::min(pr, sl - s0);
                    const BandPanel& pn = panels[k];
                    BandItem it{};
                    it.off = pn.val_off + s0 * rs + o0;
                    it.rs = static_cast<uint32_t>(rs);
                    it.ns = static_cast<uint32_t>(ns);
                    it.ow = static_cast<uint32_t>(ow);
                    it.va = pn.s_base + static_cast<uint32_t>(s0);  // rows from g0 on read va[c + gapn]
                    it.g0 = s0 >= pn.gap0 ? 0u : static_cast<uint32_t>(std::min<size_t>(pn.gap0 - s0, ns));
                    it.gapn = pn.gapn;
                    it.oa = pn.o_base + static_cast<uint32_t>(o0);
                    it.split = K > 1 ? (sid << 8) | static_cast<uint32_t>(j) : 0xffffffffu;
                    pieces.push_back({it, cost_of(ns, row_stride(ow))});
                }
            }
        }
        if (scratch > 0xffffffffull) throw Status(2, "lcn: band split scratch above 2^32 entries");
        // largest first: the CTAs' dynamic claims then approximate LPT list
        // scheduling without a cost model of the per-item overheads
        std::stable_sort(pieces.begin(), pieces.end(), [](const Piece& x, const Piece& y) { return x.cost > y.cost; });
        std::vector<BandItem> items;
        items.reserve(pieces.size());
        PassPlan P;
        P.stat = std::getenv("LCN_BAND_STATIC") != nullptr;
        if (P.stat) {  // LPT-assigned static ranges per CTA
            using Load = std::pair<double, int>;
            std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
            for (int c = 0; c < band_grid; ++c) heap.push({0.0, c});
            std::vector<std::vector<BandItem>> per(band_grid);
            for (const Piece& pc : pieces) {
                Load ld = heap.top();
                heap.pop();
                per[ld.second].push_back(pc.it);
                ld.first += pc.cost;
                heap.push(ld);
            }
            std::vector<uint32_t> off(band_grid + 1, 0);
            for (int c = 0; c < band_grid; ++c) {
                off[c] = static_cast<uint32_t>(items.size());
                items.insert(items.end(), per[c].begin(), per[c].end());
            }
            off[band_grid] = static_cast<uint32_t>(items.size());
            P.cta_off.upload(off.data(), off.size(), s);
        } else {
            for (const Piece& pc : pieces) items.push_back(pc.it);
        }
        P.nitems = static_cast<int>(items.size());
        P.items.resize(std::max<size_t>(items.size(), 1));
        if (!items.empty()) P.items.upload(items.data(), items.size(), s);
        P.ctr.resize(2);
        P.ctr.zero(s);
        P.splits.resize(std::max<size_t>(splits.size(), 1));
        P.counters.resize(std::max<size_t>(splits.size(), 1));
        P.scratch.resize(std::max<size_t>(scratch, 1));
        if (!splits.empty()) P.splits.upload(splits.data(), splits.size(), s);
        P.counters.zero(s);
        return P;
    }

    cudaEvent_t ev(size_t i) {
        while (evs.size() <= i) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            evs.push_back(e);
        }
        return evs[i];
    }
    void mark(int it, int ph) {
        if (ctx.profile) CUDA_OK(cudaEventRecord(ev(mark_base + static_cast<size_t>(it) * 5 + ph), s));
    }

    template <typename T>
    const T* band_vals(int b) const {
        if constexpr (std::is_same_v<T, float>) return op.val32[b].get();
        else return op.val64[b].get();
    }
    template <typename T>
    bool has_valsT(size_t b) const {
        if constexpr (std::is_same_v<T, float>) return b < op.val32T.size() && op.val32T[b].size() > 0;
        else return b < op.val64T.size() && op.val64T[b].size() > 0;
    }
    template <typename T>
    const T* band_valsT(int b) const {
        if constexpr (std::is_same_v<T, float>) return op.val32T[b].get();
        else return op.val64T[b].get();
    }
    template <typename T>
    const T* U() const {
        if constexpr (std::is_same_v<T, float>) return op.U32.get();
        else return op.U64p.get();
    }
    template <typename T>
    const T* Wt() const {
        if constexpr (std::is_same_v<T, float>) return op.Wt32.get();
        else return op.Wt64p.get();
    }

    void alloc() {
        s = ctx.stream;
        st.resize(1);
        st.zero(s);
        dpart.resize(256);
        // row vectors padded to a multiple of kRT (the bulk copies read whole tiles)
        long long np = (n + kRT - 1) / kRT * kRT, mpd = (m + kRT - 1) / kRT * kRT;
        log_p.resize(np); log_q.resize(mpd); pv.resize(np); qv.resize(mpd);
        log_s[0].resize(np); log_s[1].resize(np); log_t.resize(mpd); row_marg.resize(np);
        err_part.resize(std::max<long long>(G, ceil_div(n, 256)));
        if (op.kind <= 1) {
            Mr.resize(n); Sr.resize(n); Mc.resize(m); Sc.resize(m);
            if (lse_stream()) {  // bucket-ordered copies of the stream vector per band
                ltp.resize(op.bands.size());
                lsp[0].resize(op.bands.size());
                for (size_t b = 0; b < op.bands.size(); ++b) {
                    ltp[b].resize(m + 16);
                    lsp[0][b].resize(n + 16);
                }
            }
        } else {
            corr_s.resize(ncorr());
            corr_t.resize(ncorr());
            for (size_t b = 0; b < ncorr(); ++b) {
                if (corr_s[b].size() != static_cast<size_t>(np)) {
                    corr_s[b].resize(np);
                    corr_s[b].zero(s);  // rows outside any work bucket stay 0
                }
                if (corr_t[b].size() != static_cast<size_t>(mpd)) {
                    corr_t[b].resize(mpd);
                    corr_t[b].zero(s);
                }
            }
            ltp.resize(op.bands.size());
            lsp[0].resize(op.bands.size());
            lsp[1].resize(op.bands.size());
            for (size_t b = 0; b < op.bands.size(); ++b) {
                ltp[b].resize(m + 16);
                lsp[0][b].resize(n + 16);
                lsp[1][b].resize(n + 16);
                ltp[b].zero(s);  // log t = 0 before the first row side
            }
            part.resize(static_cast<size_t>(G) * lp); hpart.resize(G); mnp.resize(G); mxp.resize(G);
            mid_s.resize(lp); mid_t.resize(lp);
            if (sh) {
                stride_s = kShardHdr + lp + static_cast<long long>(sh->max_exp_s);
                stride_t = kShardHdr + lp + static_cast<long long>(sh->max_exp_t);
                send_s.resize(stride_s);
                send_t.resize(stride_t);
                recv_s.resize(stride_s * sh->world);
                recv_t.resize(stride_t * sh->world);
                send_s.zero(s);
                send_t.zero(s);
                gstage.resize(9);
            }
        }
    }

    template <typename T, int SIDE>
    void pass(const PassArgs& a, long long row0 = 0) {
        const T* F = (SIDE == 0 ? U<T>() : Wt<T>()) + row0 * lp;
        const dim3 g(G), b(kThreads + 64);
        switch (CPT) {
            case 1: launch_pdl(lowrank_pass_kernel<T, 1, SIDE>, g, b, smem, s, pdl(), F, a); break;
            case 2: launch_pdl(lowrank_pass_kernel<T, 2, SIDE>, g, b, smem, s, pdl(), F, a); break;
            case 4: launch_pdl(lowrank_pass_kernel<T, 4, SIDE>, g, b, smem, s, pdl(), F, a); break;
        }
    }
    PassArgs base_args() {
        PassArgs a{};
        a.st = st.get();
        a.l = l;
        a.lp = lp;
        a.part = part.get();
        a.hpart = hpart.get();
        a.mnp = mnp.get();
        a.mxp = mxp.get();
        a.err_part = err_part.get();
        return a;
    }
    void reduce(double* mid, int which) {
        launch_pdl(lowrank_reduce_kernel, dim3(ceil_div(lp, 32)), dim3(1024), 0, s, pdl(), st.get(), part.get(),
                   hpart.get(), mnp.get(), G, lp, mid, which, static_cast<double*>(nullptr));
    }
    // programmatic dependent launches between the iteration's kernels (each
    // waits for its predecessor at its top; the launch itself and the CTA
    // ramp overlap the predecessor's tail). Off while phase events are
    // recorded between launches (ctx.profile) and with LCN_ITER_PDL=0.
    bool pdl() const {
        static const bool off = [] {
            const char* e = std::getenv("LCN_ITER_PDL");
            return e && e[0] == '0';
        }();
        return !ctx.profile && !off;
    }

    const int* done_ptr() const {
        return reinterpret_cast<const int*>(reinterpret_cast<const char*>(st.get()) + offsetof(DevState, done));
    }

    // -------- sparse -------------------------------------------------------
    template <typename T>
    const T* dense_logk(bool transposed) const {
        if constexpr (std::is_same_v<T, float>) return transposed ? op.dk32T.get() : op.dk32.get();
        else return transposed ? op.dk64T.get() : op.dk64.get();
    }
    template <typename T>
    void sparse_rows(const double* lt) {
        if (op.kind == 0 && op.dense_tc) {  // dense, recomputed on the tensor cores
            dense_tc_lse(op, false, lt, done_ptr(), Mr.get(), Sr.get());
            return;
        }
        if (op.kind == 0) {  // dense: the whole row in one (max, sum) pair
            if constexpr (sizeof(T) == 4)
                if (m % 4 == 0) {
                    dense_lse_tma_kernel<<<lse_grid, kThreads + 32, sizeof(LseSmem), s>>>(
                        st.get(), dense_logk<T>(false), n, m, lt, Mr.get(), Sr.get());
                    return;
                }
            dense_lse_kernel<T><<<ceil_div(n, kDenseRows), 256, 0, s>>>(st.get(), dense_logk<T>(false), n, m, lt,
                                                                        Mr.get(), Sr.get());
            return;
        }
        if (op.gcsr) {
            csr_lse_kernel<<<ceil_div(n * 32, 256), 256, 0, s>>>(st.get(), op.csr_row_ptr.get(), op.csr_col.get(),
                                                                 op.gval.get(), lt, n, Mr.get(), Sr.get());
            return;
        }
        lse_init_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), Mr.get(), Sr.get(), n);
        if constexpr (sizeof(T) == 4)
            if (lse_stream()) {
                scatter_perm(lt, m, 1, 0);  // log t into every band's bucket order
                for (size_t b = 0; b < op.bands.size(); ++b) {
                    PassPlan& P = plans[0][b];
                    if (P.nitems)
                        band_stream_kernel<float, true, true><<<band_grid, kThreads + 64, sizeof(BandSmem), s>>>(
                            st.get(), op.iter[b].so, P.work(), band_valsT<float>(b), ltp[b].get(), Mr.get(), Sr.get());
                }
                return;
            }
        for (size_t b = 0; b < op.bands.size(); ++b)
            if (op.bands[b].n_work)
                sparse_row_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                    st.get(), op.view(b), op.bands[b].work.get(), band_vals<T>(b), lt, Mr.get(), Sr.get());
    }
    template <typename T>
    void sparse_cols(const double* ls) {
        if (op.kind == 0 && op.dense_tc) {  // dense, recomputed on the tensor cores
            dense_tc_lse(op, true, ls, done_ptr(), Mc.get(), Sc.get());
            return;
        }
        if (op.kind == 0) {  // dense: rows of the transposed copy
            if constexpr (sizeof(T) == 4)
                if (n % 4 == 0) {
                    dense_lse_tma_kernel<<<lse_grid, kThreads + 32, sizeof(LseSmem), s>>>(
                        st.get(), dense_logk<T>(true), m, n, ls, Mc.get(), Sc.get());
                    return;
                }
            dense_lse_kernel<T><<<ceil_div(m, kDenseRows), 256, 0, s>>>(st.get(), dense_logk<T>(true), m, n, ls,
                                                                        Mc.get(), Sc.get());
            return;
        }
        if (op.gcsr) {
            csr_lse_kernel<<<ceil_div(m * 32, 256), 256, 0, s>>>(st.get(), op.gcp.get(), op.gri.get(), op.gvalT.get(),
                                                                 ls, m, Mc.get(), Sc.get());
            return;
        }
        lse_init_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), Mc.get(), Sc.get(), m);
        if constexpr (sizeof(T) == 4)
            if (lse_stream()) {
                scatter_perm(ls, n, 0, 0);  // log s into every band's bucket order
                for (size_t b = 0; b < op.bands.size(); ++b) {
                    PassPlan& P = plans[1][b];
                    if (P.nitems)
                        band_stream_kernel<float, false, true><<<band_grid, kThreads + 64, sizeof(BandSmem), s>>>(
                            st.get(), op.iter[b].to, P.work(), band_vals<float>(b), lsp[0][b].get(), Mc.get(), Sc.get());
                }
                return;
            }
        for (size_t b = 0; b < op.bands.size(); ++b)
            if (op.bands[b].n_work) {
                if (has_valsT<T>(b)) {
                    // the transposed blocks (targets x sources): the row kernel with the roles swapped
                    BandView tv = op.view(b);
                    std::swap(tv.src_order, tv.tgt_order);
                    std::swap(tv.src_start, tv.tgt_start);
                    tv.blk_off = tv.blkT_off;
                    sparse_row_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                        st.get(), tv, op.bands[b].work.get(), band_valsT<T>(b), ls, Mc.get(), Sc.get());
                } else {
                    sparse_col_band_kernel<T><<<op.bands[b].n_work, kThreads, 0, s>>>(
                        st.get(), op.view(b), op.bands[b].work.get(), band_vals<T>(b), ls, Mc.get(), Sc.get());
                }
            }
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
        iter_end_kernel<<<1, 256, 0, s>>>(st.get(), err_part.get(), ceil_div(n, 256), it, max_iters, tol, trace.get(),
                                          nullptr);
        mark(it, 4);
    }

    // -------- lcn / nystrom ------------------------------------------------
    // logvp[b]: band b's bucket-ordered copy of the log vector (written by the
    // low-rank pass that produced it, or by scatter_perm).
    template <typename T, bool ROWS>
    void bands(std::vector<DevBuf<double>>& logvp, std::vector<DevBuf<double>>& corr) {
        if (op.kind != 3) return;
        // LCN_BAND_OVERLAP=1 (experimental, off by default): bands after the
        // first launched one overlap its tail (late_wait); every band has its
        // own plan, claim counters, scratch and output. Measured -2 % per
        // iteration and bit-identical, but 2 of ~30 bench runs stalled inside
        // a solve with it on (none of ~45 with it off), so it stays opt-in.
        // LCN_BAND_OVERLAP=2: the same, but the overlapping band triggers its
        // dependent only by exiting (after its late wait); 1 of 64 runs
        // stalled with it too (profiles/band_overlap_stall_r05.txt).
        static const int overlap = [] {
            const char* e = std::getenv("LCN_BAND_OVERLAP");
            return e && (e[0] == '1' || e[0] == '2') ? e[0] - '0' : 0;
        }();
        int launched = 0;
        for (size_t b = 0; b < op.bands.size(); ++b) {
            PassPlan& P = plans[ROWS ? 0 : 1][b];
            if (P.nitems)
                launch_pdl(band_stream_kernel<T, ROWS, false>, dim3(band_grid), dim3(kThreads + 64), sizeof(BandSmem), s,
                           pdl(), st.get(), ROWS ? op.iter[b].so : op.iter[b].to, P.work(),
                           ROWS ? band_valsT<T>(b) : band_vals<T>(b), logvp[b].get(), corr[b].get(),
                           static_cast<double*>(nullptr), (pdl() && overlap && launched++ > 0) ? overlap : 0);
        }
    }
    template <typename T>
    void lcn_rows(const double* lt = nullptr) {
        if (op.kind == 3 && op.gcsr) {  // general pattern: CSR rows over log t
            csr_corr_kernel<<<ceil_div(n * 32, 256), 256, 0, s>>>(st.get(), op.csr_row_ptr.get(), op.csr_col.get(),
                                                                  op.gval.get(), lt ? lt : log_t.get(), n, 1,
                                                                  corr_s[0].get());
            return;
        }
        bands<T, true>(ltp, corr_s);
    }
    template <typename T>
    void lcn_cols(int parity, const double* ls = nullptr) {
        if (op.kind == 3 && op.gcsr) {  // general pattern: CSC columns over log s
            csr_corr_kernel<<<ceil_div(m * 32, 256), 256, 0, s>>>(st.get(), op.gcp.get(), op.gri.get(), op.gvalT.get(),
                                                                  ls ? ls : log_s[parity].get(), m, 0,
                                                                  corr_t[0].get());
            return;
        }
        bands<T, false>(lsp[parity], corr_t);
    }
    size_t ncorr() const { return op.gcsr ? 1 : op.bands.size(); }
    void set_perm(PassArgs& a, int side, int parity) {
        a.nperm = 0;
        if (op.kind != 3) return;
        for (size_t b = 0; b < op.bands.size(); ++b) {
            a.pos[a.nperm] = side == 0 ? op.iter[b].sp : op.iter[b].tp;
            a.perm[a.nperm++] = side == 0 ? lsp[parity][b].get() : ltp[b].get();
        }
    }
    // the sparse operator streams its log K through band_stream_kernel's
    // log-sum-exp mode (fp32 storage, bucket-blocked support with panels)
    bool lse_stream() const { return op.kind == 1 && !op.fp64 && !op.gcsr && op.iter.size() == op.bands.size() &&
                                     !op.bands.empty(); }
    void scatter_perm(const double* v, long long len, int side, int parity) {
        if (op.kind != 3 && !lse_stream()) return;
        for (size_t b = 0; b < op.bands.size(); ++b)
            perm_scatter_kernel<<<ceil_div(len, 256), 256, 0, s>>>(
                v, len, side == 0 ? op.iter[b].sp : op.iter[b].tp,
                side == 0 ? lsp[parity][b].get() : ltp[b].get());
    }
    void set_corr(PassArgs& a, int side) {
        a.ncorr = 0;
        if (op.kind != 3) return;
        for (size_t b = 0; b < ncorr(); ++b) a.corr[a.ncorr++] = side == 0 ? corr_s[b].get() : corr_t[b].get();
    }

    template <typename T>
    void lcn_iteration(int it, double tol, int max_iters) {
        const int cur = it % 2, nxt = (it + 1) % 2;
        mark(it, 0);
        if (it == 0) {
            // kt = K(log t = 0) (sinkhorn.cpp:145): partial W^T 1 with shift 0.
            PassArgs a = base_args();
            a.rows = m;
            a.mode = 2;
            a.in = nullptr;
            pass<T, 1>(a);
            mark(it, 1);
        } else {
            lcn_cols<T>(cur);
            mark(it, 1);
            PassArgs a = base_args();
            a.rows = m;
            a.mode = 0;
            a.mid = mid_s.get();
            set_corr(a, 1);
            set_perm(a, 1, 0);
            a.log_marg = log_q.get();
            a.log_out = log_t.get();
            pass<T, 1>(a);
        }
        reduce(mid_t.get(), 0);
        mark(it, 2);
        lcn_rows<T>();
        mark(it, 3);
        PassArgs a = base_args();
        a.rows = n;
        a.mode = 0;
        a.mid = mid_t.get();
        set_corr(a, 0);
        a.log_marg = log_p.get();
        a.marg = pv.get();
        a.log_cur = log_s[cur].get();
        a.log_out = log_s[nxt].get();
        a.row_marg = row_marg.get();
        a.with_err = it > 0;
        set_perm(a, 0, nxt);
        pass<T, 0>(a);
        reduce(mid_s.get(), 1);
        launch_pdl(iter_end_kernel, dim3(1), dim3(256), 0, s, pdl(), st.get(), err_part.get(), G, it, max_iters, tol,
                   trace.get(), static_cast<const double*>(nullptr));
        mark(it, 4);
    }

    // ---- bucket-sharded solve ----------------------------------------------
    // End of one side's low-rank pass: this rank's reduce into its exchange
    // record (shift, minimum, partial; on the row side the marginal-error
    // partial and flags), its exported scalings, ONE all-gather, then the
    // rank-ordered combine and the halo scalings (vec and the bucket-ordered
    // copies of every band).
    void exchange(int side, int it, double* vec, int parity, double* mid, double* gst) {
        DevBuf<double>& send = side ? send_t : send_s;
        DevBuf<double>& recv = side ? recv_t : recv_s;
        const long long stride = side ? stride_t : stride_s;
        lowrank_reduce_kernel<<<ceil_div(lp, 32), 1024, 0, s>>>(st.get(), part.get(), hpart.get(), mnp.get(), G, lp,
                                                                send.get() + kShardHdr, side ? 0 : 1, send.get());
        if (gst) stage_err_kernel<<<1, 256, 0, s>>>(st.get(), err_part.get(), G, it, send.get() + 2);
        const long long nexp = static_cast<long long>(side ? sh->n_exp_t : sh->n_exp_s);
        if (nexp)
            shard_pack_kernel<<<static_cast<int>(std::min<long long>(ceil_div(nexp, 256), 4LL * ctx.num_sms)), 256, 0, s>>>(
                vec, side ? sh->exp_t.get() : sh->exp_s.get(), nexp, send.get() + kShardHdr + lp);
        comm->allgather(send.get(), recv.get(), static_cast<size_t>(stride) * sizeof(double), s);
        HaloUnpack hu{};
        hu.rank = side ? sh->imp_t_rank.get() : sh->imp_s_rank.get();
        hu.slot = side ? sh->imp_t_slot.get() : sh->imp_s_slot.get();
        hu.cnt = static_cast<long long>(side ? sh->m_halo : sh->n_halo);
        hu.own = side ? m_own : n_own;
        hu.vec = vec;
        hu.nperm = 0;
        for (size_t b = 0; b < op.bands.size(); ++b) {
            hu.pos[hu.nperm] = side ? op.iter[b].tp : op.iter[b].sp;
            hu.perm[hu.nperm++] = side ? ltp[b].get() : lsp[parity][b].get();
        }
        const int hb = static_cast<int>(std::min<long long>(ceil_div(hu.cnt, 256), 4LL * ctx.num_sms));
        shard_combine_kernel<<<1 + hb, 256, 0, s>>>(st.get(), recv.get(), sh->world, stride, lp, mid, side ? 0 : 1, gst,
                                                    hu);
    }

    // One iteration of the bucket-sharded solve: the local
    // operator's band passes (band-0 blocks entirely local, later bands over
    // owned + halo points), the low-rank pass over the owned rows, one
    // exchange per half-iteration; iter_end sees the summed error and flags,
    // so every rank takes the same decisions.
    template <typename T>
    void lcn_iteration_shard(int it, double tol, int max_iters) {
        const int cur = it % 2, nxt = (it + 1) % 2;
        mark(it, 0);
        if (it == 0) {
            PassArgs a = base_args();
            a.rows = m_own;
            a.mode = 2;
            a.in = nullptr;
            pass<T, 1>(a);
            mark(it, 1);
        } else {
            lcn_cols<T>(cur);
            mark(it, 1);
            PassArgs a = base_args();
            a.rows = m_own;
            a.mode = 0;
            a.mid = mid_s.get();
            set_corr(a, 1);
            set_perm(a, 1, 0);
            a.log_marg = log_q.get();
            a.log_out = log_t.get();
            pass<T, 1>(a);
        }
        exchange(1, it, log_t.get(), 0, mid_t.get(), nullptr);
        mark(it, 2);
        lcn_rows<T>();
        mark(it, 3);
        PassArgs a = base_args();
        a.rows = n_own;
        a.mode = 0;
        a.mid = mid_t.get();
        set_corr(a, 0);
        a.log_marg = log_p.get();
        a.marg = pv.get();
        a.log_cur = log_s[cur].get();
        a.log_out = log_s[nxt].get();
        a.row_marg = row_marg.get();
        a.with_err = it > 0;
        set_perm(a, 0, nxt);
        pass<T, 0>(a);
        exchange(0, it, log_s[nxt].get(), nxt, mid_s.get(), gstage.get());
        iter_end_kernel<<<1, 256, 0, s>>>(st.get(), err_part.get(), G, it, max_iters, tol, trace.get(), gstage.get());
        mark(it, 4);
    }

    // Owned slices of log s, P1 and log t of every rank, all-gathered once,
    // into the whole problem's vectors (global order) on every rank; the
    // distance identity over them in global order.
    void finish_shard(const DevState& h, const std::vector<double>& gq, Result& res) {
        const int fin = h.iters % 2;
        const int W = sh->world;
        // record: [distance partial | log s | P1 | log t] of the owned points
        size_t F = 2;
        for (int r = 0; r < W; ++r) F = std::max(F, 1 + 2 * sh->own_src_all[r].size() + sh->own_tgt_all[r].size());
        DevBuf<double> fs(F), fr(F * W);
        // this rank's <log s, P1> + <log t, q> over its owned points (deterministic block partials)
        const int DB = 64;
        dot_partial_kernel<<<DB, 256, 0, s>>>(log_s[fin].get(), row_marg.get(), n_own, dpart.get());
        dot_partial_kernel<<<DB, 256, 0, s>>>(log_t.get(), qv.get(), m_own, dpart.get() + DB);
        sum_partial_kernel<<<1, 256, 0, s>>>(dpart.get(), 2 * DB, fs.get());
        CUDA_OK(cudaMemcpyAsync(fs.get() + 1, log_s[fin].get(), n_own * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_OK(cudaMemcpyAsync(fs.get() + 1 + n_own, row_marg.get(), n_own * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_OK(cudaMemcpyAsync(fs.get() + 1 + 2 * n_own, log_t.get(), m_own * 8, cudaMemcpyDeviceToDevice, s));
        comm->allgather(fs.get(), fr.get(), F * sizeof(double), s);
        std::vector<double> hr(F * W);
        fr.download(hr.data(), F * W, s);
        ctx.sync();
        const size_t N = sh->n_glob, M = sh->m_glob;
        res.log_s.assign(N, 0.0);
        res.row_marg.assign(N, 0.0);
        res.log_t.assign(M, 0.0);
        double acc = 0.0;
        for (int r = 0; r < W; ++r) {
            const std::vector<uint32_t>& os = sh->own_src_all[r];
            const std::vector<uint32_t>& ot = sh->own_tgt_all[r];
            const double* rec = hr.data() + static_cast<size_t>(r) * F;
            acc += rec[0];  // rank order: the same sum on every rank
            const long long ns = static_cast<long long>(os.size()), nt = static_cast<long long>(ot.size());
#pragma omp parallel for schedule(static) if (ns > 65536)
            for (long long k = 0; k < ns; ++k) {
                res.log_s[os[k]] = rec[1 + k];
                res.row_marg[os[k]] = rec[1 + ns + k];
            }
#pragma omp parallel for schedule(static) if (nt > 65536)
            for (long long k = 0; k < nt; ++k) res.log_t[ot[k]] = rec[1 + 2 * ns + k];
        }
        (void)gq;
        // distance = lambda (<log s, P1> + <log t, q>) (sinkhorn.cpp:178-183), per-rank partials
        res.distance = op.lambda * acc;
        res.n = N;
        res.m = M;
    }

    template <typename T>
    void run(const double* in_p, const double* in_q, bool device_ptrs, const SolveOptions& o, Result& res) {
        alloc();
        trace.resize(std::max<size_t>(std::max(o.max_iters, 1), trace.size()));
        const cudaMemcpyKind kind = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        std::vector<double> gp, gq;  // sharded: the whole problem's marginals
        if (sh) {
            gp.resize(sh->n_glob);
            gq.resize(sh->m_glob);
            CUDA_OK(cudaMemcpyAsync(gp.data(), in_p, gp.size() * 8, cudaMemcpyDefault, s));
            CUDA_OK(cudaMemcpyAsync(gq.data(), in_q, gq.size() * 8, cudaMemcpyDefault, s));
            ctx.sync();
            std::vector<double> lp_(n), lq_(m);
            for (long long k = 0; k < n; ++k) lp_[k] = gp[sh->src_glob[k]];
            for (long long k = 0; k < m; ++k) lq_[k] = gq[sh->tgt_glob[k]];
            CUDA_OK(cudaMemcpyAsync(pv.get(), lp_.data(), n * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(qv.get(), lq_.data(), m * 8, cudaMemcpyHostToDevice, s));
            ctx.sync();
        } else {
            CUDA_OK(cudaMemcpyAsync(pv.get(), in_p, n * 8, kind, s));
            CUDA_OK(cudaMemcpyAsync(qv.get(), in_q, m * 8, kind, s));
        }
        log_kernel<<<ceil_div(n, 256), 256, 0, s>>>(pv.get(), log_p.get(), n);
        log_kernel<<<ceil_div(m, 256), 256, 0, s>>>(qv.get(), log_q.get(), m);
        CUDA_OK(cudaMemsetAsync(log_s[0].get(), 0, n * 8, s));
        CUDA_OK(cudaMemsetAsync(log_s[1].get(), 0, n * 8, s));
        CUDA_OK(cudaMemsetAsync(log_t.get(), 0, m * 8, s));
        CUDA_OK(cudaMemsetAsync(row_marg.get(), 0, n * 8, s));
        // tol: default 1e-6 * (sum p + sum q) (sinkhorn.cpp:130-133).
        double tol = o.tol;
        if (tol < 0.0 && sh) {
            double mass = 0.0;
            for (double v : gp) mass += v;
            for (double v : gq) mass += v;
            tol = 1e-6 * mass;
        } else if (tol < 0.0) {
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
                if (op.kind <= 1) sparse_iteration<T>(it, tol, o.max_iters);
                else if (sh) lcn_iteration_shard<T>(it, tol, o.max_iters);
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
        res.err_trace.resize(h.iters);
        if (h.iters) trace.download(res.err_trace.data(), h.iters, s);
        if (sh) {
            finish_shard(h, gq, res);
            return;
        }
        res.n = n;
        res.m = m;
        const int fin = h.iters % 2;
        res.log_s.resize(n);
        res.log_t.resize(m);
        res.row_marg.resize(n);
        log_s[fin].download(res.log_s.data(), n, s);
        log_t.download(res.log_t.data(), m, s);
        row_marg.download(res.row_marg.data(), n, s);
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

    // base_log_matvec(_t) (operator.cpp:123-224) between device vectors (d_in
    // readable kRT entries past its length). LCN / Nystrom positivity failures
    // are left in st->flags for the caller.
    template <typename T>
    void base_mv(const double* d_in, bool transposed, double* d_out) {
        if (op.kind <= 1) {
            if (!transposed) {
                sparse_rows<T>(d_in);
                sparse_row_finalize_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), Mr.get(), Sr.get(), log_p.get(),
                                                                            pv.get(), n, nullptr, log_s[1].get(), d_out,
                                                                            nullptr, nullptr, 0);
            } else {
                sparse_cols<T>(d_in);
                CUDA_OK(cudaMemsetAsync(log_t.get(), 0, m * 8, s));  // zero "log q": out = -kts
                sparse_col_finalize_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), Mc.get(), Sc.get(), log_t.get(), m,
                                                                            d_out);
                negate_kernel<<<ceil_div(m, 256), 256, 0, s>>>(d_out, m);
            }
            return;
        }
        PassArgs acc = base_args();
        acc.mode = 2;
        acc.in = d_in;
        PassArgs mv = base_args();
        mv.mode = 1;
        mv.out = d_out;
        if (!transposed) {
            acc.rows = m;
            pass<T, 1>(acc);
            reduce(mid_t.get(), 0);
            scatter_perm(d_in, m, 1, 0);
            lcn_rows<T>(d_in);
            mv.rows = n;
            mv.mid = mid_t.get();
            set_corr(mv, 0);
            pass<T, 0>(mv);
        } else {
            acc.rows = n;
            pass<T, 0>(acc);
            reduce(mid_s.get(), 1);
            scatter_perm(d_in, n, 0, 0);
            lcn_cols<T>(0, d_in);
            mv.rows = m;
            mv.mid = mid_s.get();
            set_corr(mv, 1);
            pass<T, 1>(mv);
        }
    }

    // sinkhorn (sinkhorn.cpp:104-188) with the BP extension: extended
    // marginals [p; q] / [q; p], K_BP products from the base products plus the
    // deletion diagonals and the eps-eps block (operator.cpp:226-266), on the
    // device; one host check per product keeps the reference's error order.
    template <typename T>
    void run_bp(const double* in_p, const double* in_q, const SolveOptions& o, Result& res) {
        if (sh) throw Status(2, "sinkhorn: the BP extension is not available on a sharded operator");
        alloc();
        const long long R = n + m;  // rows of the extended problem (= columns)
        const size_t pad = static_cast<size_t>(R) + 2 * kRT;
        DevBuf<double> pe(pad), qe(pad), lpe(pad), lqe(pad), ls(pad), lt(pad), kt(pad), kts(pad), rm(pad), base(pad);
        DevBuf<double> tot(1), part(256);
        DevBuf<unsigned> bad(1);
        for (DevBuf<double>* b : {&ls, &lt, &kt, &kts, &base}) b->zero(s);
        CUDA_OK(cudaMemcpyAsync(pe.get(), in_p, n * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(pe.get() + n, in_q, m * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(qe.get(), in_q, m * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(qe.get() + m, in_p, n * 8, cudaMemcpyHostToDevice, s));
        log_dev_kernel<<<ceil_div(R, 256), 256, 0, s>>>(pe.get(), R, lpe.get());
        log_dev_kernel<<<ceil_div(R, 256), 256, 0, s>>>(qe.get(), R, lqe.get());
        double mass = 0.0;
        for (long long i = 0; i < n; ++i) mass += in_p[i];
        for (long long j = 0; j < m; ++j) mass += in_q[j];
        mass *= 2.0;  // sum of [p; q] and [q; p]
        const double tol = o.tol >= 0.0 ? o.tol : 1e-6 * mass;
        const std::string name = op.full_name();
        auto check_neg = [&](bool transposed) {
            DevState h{};
            st.download(&h, 1, s);
            ctx.sync();
            const unsigned f = h.flags;
            if (op.kind >= 2) {
                if (!transposed && (f & (F_NEG_ROW | F_NYS_ROW)))
                    throw Status(4, std::string(op.name()) + " matvec produced a nonpositive entry");
                if (transposed && (f & (F_NEG_COL | F_NYS_COL)))
                    throw Status(4, std::string(op.name()) + " transposed matvec produced a nonpositive entry");
            }
        };
        auto check_bad = [&](const char* which) {
            unsigned hb = 0;
            bad.download(&hb, 1, s);
            ctx.sync();
            if (hb) throw Status(3, std::string("sinkhorn: non-finite scaling (") + which + ") under the " + name +
                                        " operator");
        };
        const int gR = static_cast<int>(ceil_div(R, 256));
        // kt = K_BP(log t); y written to `out` (log_marg null) or the update log_marg - y
        auto kbp = [&](const double* ltv, const double* log_marg, double* out) {
            base_mv<T>(ltv, false, base.get());  // K t^ (upper m entries of t)
            lse_one_kernel<<<1, 1024, 0, s>>>(ltv + m, n, tot.get());
            bp_combine_kernel<<<gR, 256, 0, s>>>(base.get(), op.bp_ldp.get(), ltv + m, op.bp_ldq.get(), ltv, tot.get(),
                                                 n, m, log_marg, out, bad.get());
            check_neg(false);
        };
        auto kbpt = [&](const double* lsv, const double* log_marg, double* out) {
            base_mv<T>(lsv, true, base.get());  // K^T s^ (upper n entries of s)
            lse_one_kernel<<<1, 1024, 0, s>>>(lsv + n, m, tot.get());
            bp_combine_kernel<<<gR, 256, 0, s>>>(base.get(), op.bp_ldq.get(), lsv + n, op.bp_ldp.get(), lsv, tot.get(),
                                                 m, n, log_marg, out, bad.get());
            check_neg(true);
        };
        bad.zero(s);
        kbp(lt.get(), nullptr, kt.get());
        res.err_trace.clear();
        bool converged = false;
        double err = std::numeric_limits<double>::infinity();
        int iter = 0;
        std::vector<double> hp(256);
        while (iter < o.max_iters) {
            ++iter;
            // log s = log p - kt (the BP product of the previous log t)
            sub_kernel<<<gR, 256, 0, s>>>(lpe.get(), kt.get(), R, ls.get(), bad.get());
            check_bad("log s");
            kbpt(ls.get(), lqe.get(), lt.get());
            check_bad("log t");
            kbp(lt.get(), nullptr, kt.get());
            bp_err_kernel<<<256, 256, 0, s>>>(ls.get(), kt.get(), pe.get(), R, rm.get(), part.get());
            part.download(hp.data(), 256, s);
            ctx.sync();
            err = 0.0;
            for (double v : hp) err += v;
            res.err_trace.push_back(err);
            if (err <= tol) {
                converged = true;
                break;
            }
        }
        res.iters = iter;
        res.converged = converged;
        res.marginal_err_final = err;
        res.n = n;
        res.m = m;
        res.log_s.resize(R);
        res.log_t.resize(R);
        res.row_marg.resize(R);
        ls.download(res.log_s.data(), R, s);
        lt.download(res.log_t.data(), R, s);
        rm.download(res.row_marg.data(), R, s);
        // distance = lambda (<log s, P1> + <log t, q_ext>) (sinkhorn.cpp:178-183)
        dot_partial_kernel<<<64, 256, 0, s>>>(ls.get(), rm.get(), R, part.get());
        dot_partial_kernel<<<64, 256, 0, s>>>(lt.get(), qe.get(), R, part.get() + 64);
        part.download(hp.data(), 128, s);
        ctx.sync();
        double acc = 0.0;
        for (int k = 0; k < 128; ++k) acc += hp[k];
        res.distance = op.lambda * acc;
        if (o.want_plan) {
            DevBuf<double> dpm(n), dqm(m);
            bp_mass_kernel<<<gR, 256, 0, s>>>(op.bp_ldp.get(), op.bp_ldq.get(), ls.get(), lt.get(), n, m, dpm.get(),
                                              dqm.get());
            exp_sum_partial_kernel<<<64, 256, 0, s>>>(ls.get() + n, m, part.get());
            exp_sum_partial_kernel<<<64, 256, 0, s>>>(lt.get() + m, n, part.get() + 64);
            res.del_p_mass.resize(n);
            res.del_q_mass.resize(m);
            dpm.download(res.del_p_mass.data(), n, s);
            dqm.download(res.del_q_mass.data(), m, s);
            part.download(hp.data(), 128, s);
            ctx.sync();
            double ss = 0.0, tt = 0.0;
            for (int k = 0; k < 64; ++k) ss += hp[k];
            for (int k = 64; k < 128; ++k) tt += hp[k];
            res.eps_mass = ss * tt;
        }
    }

    // log_matvec / log_matvec_t (operator.cpp:226-252) on a host vector.
    template <typename T>
    void matvec(const double* h_in, bool transposed, double* h_out) {
        if (sh) throw Status(2, "log_matvec: not available on a sharded operator (build it on a context without a communicator)");
        alloc();
        const long long len_in = transposed ? n : m, len_out = transposed ? m : n;
        DevBuf<double> vin((len_in + kRT - 1) / kRT * kRT), vout(len_out);
        vin.upload(h_in, len_in, s);
        if (op.kind <= 1) {
            if (!transposed) {
                sparse_rows<T>(vin.get());
                sparse_row_finalize_kernel<<<ceil_div(n, 256), 256, 0, s>>>(st.get(), Mr.get(), Sr.get(), log_p.get(),
                                                                            pv.get(), n, nullptr, log_s[1].get(),
                                                                            vout.get(), nullptr, nullptr, 0);
            } else {
                sparse_cols<T>(vin.get());
                DevBuf<double> zq(m);
                zq.zero(s);
                sparse_col_finalize_kernel<<<ceil_div(m, 256), 256, 0, s>>>(st.get(), Mc.get(), Sc.get(), zq.get(), m,
                                                                            vout.get());
                // vout = 0 - kts -> negated on the host below
            }
        } else {
            PassArgs acc = base_args();
            acc.mode = 2;
            acc.in = vin.get();
            PassArgs mv = base_args();
            mv.mode = 1;
            mv.out = vout.get();
            if (!transposed) {
                acc.rows = m;
                pass<T, 1>(acc);
                reduce(mid_t.get(), 0);
                scatter_perm(vin.get(), m, 1, 0);
                lcn_rows<T>(vin.get());
                mv.rows = n;
                mv.mid = mid_t.get();
                set_corr(mv, 0);
                pass<T, 0>(mv);
            } else {
                acc.rows = n;
                pass<T, 0>(acc);
                reduce(mid_s.get(), 1);
                scatter_perm(vin.get(), n, 0, 0);
                lcn_cols<T>(0, vin.get());
                mv.rows = m;
                mv.mid = mid_s.get();
                set_corr(mv, 1);
                pass<T, 1>(mv);
            }
        }
        LAUNCH_OK("log_matvec");
        DevState h{};
        st.download(&h, 1, s);
        vout.download(h_out, len_out, s);
        ctx.sync();
        if (op.kind <= 1 && transposed)
            for (long long j = 0; j < len_out; ++j) h_out[j] = -h_out[j];
        if (op.kind >= 2) {
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
    // the workspace belongs to the operator (a sharded operator's partition
    // is fixed when it is built)
    if (!op.ws) op.ws = std::make_shared<Solver>(op);
    return *op.ws;
}

void sinkhorn_solve(Op& op, const double* p, const double* q, bool device_ptrs, const SolveOptions& o, Result& res) {
    if (o.max_iters < 1) throw Status(2, "sinkhorn: max_iters must be >= 1");
    Solver& sv = solver_of(op);
    if (op.fp64) sv.run<double>(p, q, device_ptrs, o, res);
    else sv.run<float>(p, q, device_ptrs, o, res);
}

void sinkhorn_solve_bp(Op& op, const double* p, const double* q, const SolveOptions& o, Result& res) {
    if (o.max_iters < 1) throw Status(2, "sinkhorn: max_iters must be >= 1");
    Solver& sv = solver_of(op);
    if (op.fp64) sv.run_bp<double>(p, q, o, res);
    else sv.run_bp<float>(p, q, o, res);
}

void op_log_matvec(Op& op, const double* h_in, bool transposed, double* h_out) {
    Solver& sv = solver_of(op);
    if (op.fp64) sv.matvec<double>(h_in, transposed, h_out);
    else sv.matvec<float>(h_in, transposed, h_out);
}

namespace {
// distance_lcn pieces (sinkhorn.cpp:222-261), fp64, deterministic: fixed
// per-block row ranges, block partials combined in block order.
constexpr int kDlBlocks = 256;

__global__ void exp_kernel(const double* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) out[i] = exp(in[i]);
}

// part[blk * l + a] = sum over the block's rows r of F[r, a] * v[r]
__global__ void __launch_bounds__(256) colsum_partial_kernel(const double* __restrict__ F, long long rows, int l,
                                                             const double* __restrict__ v, double* __restrict__ part) {
    const long long per = (rows + gridDim.x - 1) / gridDim.x;
    const long long r0 = blockIdx.x * per, r1 = r0 + per < rows ? r0 + per : rows;
    for (int a = threadIdx.x; a < l; a += 256) {
        double acc = 0.0;
        for (long long r = r0; r < r1; ++r) acc += F[r * l + a] * v[r];
        part[static_cast<long long>(blockIdx.x) * l + a] = acc;
    }
}

__global__ void colsum_reduce_kernel(const double* __restrict__ part, int blocks, int l, double* __restrict__ out) {
    const int a = blockIdx.x * 256 + threadIdx.x;
    if (a >= l) return;
    double acc = 0.0;
    for (int b = 0; b < blocks; ++b) acc += part[static_cast<long long>(b) * l + a];
    out[a] = acc;
}

// block partial of sum_r logv[r] * lin[r] * (F_r . w): one warp per row
__global__ void __launch_bounds__(256) rowdot_term_kernel(const double* __restrict__ F, long long rows, int l,
                                                          const double* __restrict__ w, const double* __restrict__ logv,
                                                          const double* __restrict__ lin, double* __restrict__ part) {
    __shared__ double red[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc = 0.0;
    for (long long r = blockIdx.x * 8LL + warp; r < rows; r += 8LL * gridDim.x) {
        double row = 0.0;
        for (int a = lane; a < l; a += 32) row += F[r * l + a] * w[a];
        row = warp_sum(row);
        acc += logv[r] * (lin[r] * row);
    }
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

// block partial of sum over the support of s_i delta_e t_j (log s_i + log t_j)
__global__ void __launch_bounds__(256) support_term_kernel(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                                           const double* __restrict__ dl, long long n,
                                                           const double* __restrict__ sl, const double* __restrict__ tl,
                                                           const double* __restrict__ ls, const double* __restrict__ lt,
                                                           double* __restrict__ part) {
    __shared__ double red[8];
    double acc = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x)
        for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
            const uint32_t j = col[e];
            acc += (sl[i] * dl[e] * tl[j]) * (ls[i] + lt[j]);
        }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}
}  // namespace

namespace {
__global__ void dense_plan_kernel(const double* __restrict__ lk, const double* __restrict__ ls,
                                  const double* __restrict__ lt, long long n, long long m, double* __restrict__ out) {
    const long long tot = n * m;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < tot; e += 256LL * gridDim.x) {
        const long long i = e / m, j = e - i * m;
        out[e] = exp(ls[i] + lk[e] + lt[j]);
    }
}
// one thread per row: plan entries of the row's support (CSR order)
__global__ void support_plan_kernel(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                    const double* __restrict__ lk, const double* __restrict__ nys, long long n,
                                    const double* __restrict__ ls, const double* __restrict__ lt,
                                    double* __restrict__ vals, double* __restrict__ nys_out) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
        const double si = exp(ls[i]);
        for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
            const uint32_t j = col[e];
            vals[e] = exp(ls[i] + lk[e] + lt[j]);
            if (nys_out) nys_out[e] = si * nys[e] * exp(lt[j]);
        }
    }
}
}  // namespace

// extract_plan_impl (sinkhorn.cpp:23-100) on the device: the dense plan
// exp(log s_i + log K_ij + log t_j) (row-major), the sparse plan on the
// support (CSR order) and the LCN sp_vals / sp_nys_vals.
void extract_plan_device(Op& op, Result& r) {
    Ctx& ctx = *op.ctx;
    cudaStream_t s = ctx.stream;
    const long long n = static_cast<long long>(op.n), m = static_cast<long long>(op.m);
    if (op.kind == 2 || (op.kind != 0 && op.nnz == 0)) return;
    DevBuf<double> ls(n), lt(m);
    ls.upload(r.log_s.data(), n, s);
    lt.upload(r.log_t.data(), m, s);
    const int grid = 8 * ctx.num_sms;
    if (op.kind == 0) {
        const bool tmp = op.dense_tc;  // recomputed operator: the exact log K for the plan only
        if (tmp) build_dense(op);
        DevBuf<double> out(static_cast<size_t>(n * m));
        dense_plan_kernel<<<grid, 256, 0, s>>>(op.dk64.get(), ls.get(), lt.get(), n, m, out.get());
        if (tmp) {
            ctx.sync();
            op.dk64 = DevBuf<double>();
            op.dk32 = DevBuf<float>();
            op.dk32T = DevBuf<float>();
            op.dk64T = DevBuf<double>();
        }
        LAUNCH_OK("dense plan");
        r.plan_vals.resize(static_cast<size_t>(n * m));
        out.download(r.plan_vals.data(), r.plan_vals.size(), s);
        ctx.sync();
        return;
    }
    const size_t nnz = op.nnz;
    DevBuf<double> lk(nnz), vals(nnz), nys, nys_out;
    csr_values_device(op, op.kind == 1 ? 0 : 2, lk.get());
    if (op.kind == 3) {
        nys.resize(nnz);
        nys_out.resize(nnz);
        csr_values_device(op, 3, nys.get());
    }
    support_plan_kernel<<<ceil_div(n, 256), 256, 0, s>>>(op.csr_row_ptr.get(), op.csr_col.get(), lk.get(), nys.get(), n,
                                                         ls.get(), lt.get(), vals.get(), nys_out.get());
    LAUNCH_OK("support plan");
    std::vector<double>& dst = op.kind == 1 ? r.plan_vals : r.sp_vals;
    dst.resize(nnz);
    vals.download(dst.data(), nnz, s);
    if (op.kind == 3) {
        r.sp_nys_vals.resize(nnz);
        nys_out.download(r.sp_nys_vals.data(), nnz, s);
    }
    ctx.sync();
}

// distance_lcn (sinkhorn.cpp:222-261) on the device from the fp64 factors:
// P_Nys 1 = diag(s) U (W t), 1^T P_Nys = (s^T U) W diag(t), plus the
// correction's mass on the support.
double distance_lcn_device(Op& op, const Result& res) {
    Ctx& ctx = *op.ctx;
    cudaStream_t s = ctx.stream;
    const long long n = static_cast<long long>(op.n), m = static_cast<long long>(op.m);
    const int l = static_cast<int>(op.l);
    DevBuf<double> ls(n), lt(m), sl(n), tl(m), part(static_cast<size_t>(kDlBlocks) * l), wt(l), su(l), terms(3 * kDlBlocks);
    ls.upload(res.log_s.data(), n, s);
    lt.upload(res.log_t.data(), m, s);
    terms.zero(s);
    exp_kernel<<<kDlBlocks, 256, 0, s>>>(ls.get(), sl.get(), n);
    exp_kernel<<<kDlBlocks, 256, 0, s>>>(lt.get(), tl.get(), m);
    // wt = W t (Wt64 is m x l), su = U^T s (U64 is n x l)
    colsum_partial_kernel<<<kDlBlocks, 256, 0, s>>>(op.Wt64.get(), m, l, tl.get(), part.get());
    colsum_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(part.get(), kDlBlocks, l, wt.get());
    colsum_partial_kernel<<<kDlBlocks, 256, 0, s>>>(op.U64.get(), n, l, sl.get(), part.get());
    colsum_reduce_kernel<<<ceil_div(l, 256), 256, 0, s>>>(part.get(), kDlBlocks, l, su.get());
    rowdot_term_kernel<<<kDlBlocks, 256, 0, s>>>(op.U64.get(), n, l, wt.get(), ls.get(), sl.get(), terms.get());
    rowdot_term_kernel<<<kDlBlocks, 256, 0, s>>>(op.Wt64.get(), m, l, su.get(), lt.get(), tl.get(),
                                                 terms.get() + kDlBlocks);
    if (op.kind == 3 && op.nnz) {
        DevBuf<double> dl(op.nnz);
        csr_values_device(op, 1, dl.get());
        support_term_kernel<<<kDlBlocks, 256, 0, s>>>(op.csr_row_ptr.get(), op.csr_col.get(), dl.get(), n, sl.get(),
                                                      tl.get(), ls.get(), lt.get(), terms.get() + 2 * kDlBlocks);
    }
    LAUNCH_OK("distance_lcn");
    std::vector<double> h(3 * kDlBlocks);
    terms.download(h.data(), h.size(), s);
    ctx.sync();
    double term = 0.0;
    for (double v : h) term += v;
    return op.lambda * term;
}

}  // namespace lcnb
