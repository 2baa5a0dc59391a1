// Bit-exact k-means on the device: k-means++ seeding, nearest-centroid
// assignment and Lloyd updates reproducing /root/reference/proj/src/kmeans.cpp
// bit for bit:
//   * every squared distance is the sequential fp64 fold of kmeans.cpp:12-19,
//     evaluated with explicitly rounded ops (no FMA contraction);
//   * argmin ties go to the lowest centroid index (strict < over c = 0..k-1,
//     kmeans.cpp:76-82);
//   * the k-means++ running total and the target scan are the serial left
//     folds of kmeans.cpp:36-40 / 51-58, reproduced exactly by the binade
//     fold below (fl(s + x) = s + u * RN(x / u) while s stays in one binade);
//   * centroid sums are per-(cluster, dim) folds in increasing point index
//     (kmeans.cpp:106-114), then ctr = sum * (1/count) (kmeans.cpp:115-121);
//   * empty clusters are re-seeded in increasing cluster order to the first
//     farthest point among clusters of size > 1 (kmeans.cpp:122-139).
#include <cub/cub.cuh>
#include <cublas_v2.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "async.cuh"
#include "ctx.cuh"
#include "kmeans.cuh"
#include "kmeans_tc.cuh"
#include "op.cuh"
#include "tiles.cuh"

namespace lcnb {

// ---- cp.async (LDGSTS) helpers: global -> shared without a register round
// trip, so a warp can put many loads in flight before it waits once.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte elements");
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(sizeof(T))
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NG>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NG) : "memory"); }

// ---- assign_nearest (kmeans.cpp:67-85) -------------------------------------
// rows != null: evaluate only the points rows[0 .. N) (the filter's
// ambiguous list) and write out[rows[i]].
template <typename T>
__global__ void __launch_bounds__(256) assign_exact_kernel(const T* __restrict__ X, long long N, int d,
                                                           const double* __restrict__ Cm, int k,
                                                           uint32_t* __restrict__ out, double* __restrict__ best_out,
                                                           const uint32_t* __restrict__ rows,
                                                           float* __restrict__ ub = nullptr,
                                                           float* __restrict__ lb = nullptr,
                                                           double* __restrict__ part = nullptr, int cper = 0) {
    __shared__ double As[KC][TP + 1];
    __shared__ double Bs[KC][TC + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const long long p0 = static_cast<long long>(blockIdx.x) * TP;
    double best[4], sec[4];  // sec: second smallest fold (Lloyd's lower bound)
    int arg[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { best[i] = sec[i] = kPosInf; arg[i] = 0; }
    // part: this CTA scans the centroids [y cper, (y + 1) cper) only and
    // writes (best, second, index) for assign_exact_merge_kernel
    const int cb = part ? static_cast<int>(blockIdx.y) * cper : 0;
    const int ce = part ? min(k, cb + cper) : k;
    for (int c0 = cb; c0 < ce; c0 += TC) {
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        for (int k0 = 0; k0 < d; k0 += KC) {
            load_slab<T>(As, X, rows, p0, N, d, k0);
            load_slab<double>(Bs, Cm, nullptr, c0, k, d, k0);
            __syncthreads();
            tile_fold<0>(As, Bs, ty, tx, acc);
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int c = c0 + tx + 16 * j;
            if (c < ce)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (acc[i][j] < best[i]) { sec[i] = best[i]; best[i] = acc[i][j]; arg[i] = c; }
                    else if (acc[i][j] < sec[i]) sec[i] = acc[i][j];
                }
        }
    }
    // (value, index) lexicographic min over the 16 threads sharing a point;
    // the second smallest value of the multiset alongside.
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double b = best[i], s2 = sec[i];
        int a = arg[i];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            double ob = __shfl_xor_sync(0xffffffffu, b, o);
            double os = __shfl_xor_sync(0xffffffffu, s2, o);
            int oa = __shfl_xor_sync(0xffffffffu, a, o);
            s2 = fmin(fmin(s2, os), fmax(b, ob));
            if (ob < b || (ob == b && oa < a)) { b = ob; a = oa; }
        }
        long long p = p0 + ty + 16 * i;
        if (part) {
            if (tx == 0 && p < N) {
                double* pr = part + (static_cast<long long>(blockIdx.y) * N + p) * 3;
                pr[0] = b;
                pr[1] = s2;
                pr[2] = static_cast<double>(a);
            }
            continue;
        }
        if (tx == 0 && p < N) {
            const long long q = rows ? rows[p] : p;
            out[q] = static_cast<uint32_t>(a);
            if (best_out) best_out[q] = b;
            if (ub) {  // folds are within 1e-12 (relative) of the true squares
                ub[q] = __double2float_ru(__dsqrt_ru(b * (1.0 + 1e-12)));
                lb[q] = __double2float_rd(__dsqrt_rd(s2 * (1.0 - 1e-12)));
            }
        }
    }
}

// Merge of the centroid groups of assign_exact_kernel: groups in increasing
// centroid order, (value, index) lexicographic minimum (the lowest index on
// ties, as the sequential scan), the second smallest value alongside.
__global__ void assign_exact_merge_kernel(const double* __restrict__ part, int groups, long long N,
                                          const uint32_t* __restrict__ rows, uint32_t* __restrict__ out,
                                          double* __restrict__ best_out, float* __restrict__ ub,
                                          float* __restrict__ lb) {
    const long long p = blockIdx.x * 256LL + threadIdx.x;
    if (p >= N) return;
    double b = kPosInf, s2 = kPosInf;
    int a = 0;
    for (int g = 0; g < groups; ++g) {
        const double* pr = part + (static_cast<long long>(g) * N + p) * 3;
        const double ob = pr[0], os = pr[1];
        const int oa = static_cast<int>(pr[2]);
        s2 = fmin(fmin(s2, os), fmax(b, ob));
        if (ob < b || (ob == b && oa < a)) { b = ob; a = oa; }
    }
    const long long q = rows ? rows[p] : p;
    out[q] = static_cast<uint32_t>(a);
    if (best_out) best_out[q] = b;
    if (ub) {
        ub[q] = __double2float_ru(__dsqrt_ru(b * (1.0 + 1e-12)));
        lb[q] = __double2float_rd(__dsqrt_rd(s2 * (1.0 - 1e-12)));
    }
}

// Exact scan of n listed points (rows) or of all points: point tiles x
// centroid groups so a short ambiguous list still fills the GPU.
template <typename T>
void assign_exact_launch(Ctx& ctx, const T* X, long long n, int d, const double* C, int k, uint32_t* out,
                         double* best_out, const uint32_t* rows, float* ub, float* lb) {
    if (n <= 0) return;
    cudaStream_t s = ctx.stream;
    const long long ptiles = ceil_div(n, TP);
    const int ctiles = static_cast<int>(ceil_div(k, TC));
    const int want = static_cast<int>(std::min<long long>(ctiles, ceil_div(4LL * ctx.num_sms, ptiles)));
    if (want <= 1) {
        assign_exact_kernel<T><<<static_cast<unsigned>(ptiles), 256, 0, s>>>(X, n, d, C, k, out, best_out, rows, ub, lb);
        LAUNCH_OK("assign_exact_kernel");
        return;
    }
    const int cper = static_cast<int>(ceil_div(ctiles, want)) * TC;
    const int groups = static_cast<int>(ceil_div(k, cper));
    DevBuf<double> part(static_cast<size_t>(groups) * n * 3);
    assign_exact_kernel<T><<<dim3(static_cast<unsigned>(ptiles), groups), 256, 0, s>>>(
        X, n, d, C, k, out, best_out, rows, ub, lb, part.get(), cper);
    assign_exact_merge_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, s>>>(part.get(), groups, n, rows, out,
                                                                                     best_out, ub, lb);
    LAUNCH_OK("assign_exact_kernel (centroid groups)");
}

// ---- k-means++ (kmeans.cpp:23-65) ------------------------------------------
constexpr int kFoldChunk = 2048;  // fold chunk (see the chunk-parallel exact fold below)
// Several k-means++ sequences over the same points are seeded together (the
// LSH bands and the landmarks of one build): every step kernel runs one grid
// row per sequence (y = blockIdx.y), its arrays at base + y * stride, and a
// sequence whose k is reached sits the remaining steps out.
constexpr int kMaxSeq = 4;
struct PPB {
    long long sN;  // per-point arrays
    int sC;        // per-chunk arrays
    int sK;        // per-seed arrays (max k)
    int k[kMaxSeq];
};
// dist2[i] = min(dist2[i], sqdist(x_i, x_last)), strict < as kmeans.cpp:38.
// Pruning (exactness-preserving): near[i] is the seed whose fold gave
// dist2[i]; with dc[j] = |x_{seed j} - x_last| (fp64, |rel err| < 1e-13), the
// triangle inequality |x_i - x_last| >= dc[near] - |x_i - x_near| shows that
// dc[near] >= 2 sqrt(dist2[i]) (with margins) makes the new fold >= dist2[i],
// so the point cannot update and is skipped. The remaining points of a block
// are compacted and folded exactly (one thread per point, slabs staged).
// Pruning pass: one thread per point; the points that can still update are
// appended to `list` (warp-aggregated; the order is irrelevant: every point
// is updated independently).
constexpr int kPruneThreads = 512;
__global__ void __launch_bounds__(kPruneThreads, 4) pp_prune_kernel(long long N, int t, const double* __restrict__ dist2,
                                                       const uint32_t* __restrict__ near,
                                                       const double* __restrict__ dc, uint32_t* __restrict__ list,
                                                       unsigned* __restrict__ count, double* __restrict__ csum,
                                                       unsigned* __restrict__ surv_count, double* __restrict__ bsum,
                                                       PPB pb) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (t + 1 >= pb.k[y]) return;
    dist2 += y * pb.sN;
    near += y * pb.sN;
    dc += y * pb.sK;
    list += y * pb.sN;
    count += y;
    csum += y * pb.sC;
    bsum += y * pb.sC;
    if (surv_count) surv_count += y;
    if (surv_count && blockIdx.x == 0 && threadIdx.x == 0) *surv_count = 0u;  // this step's filter survivors
    // one block per fold chunk (kFoldChunk points, kPP per thread, strided
    // for coalescing; 512 threads x 4 points keep the registers low enough
    // for 4 blocks per SM): one list-append atomic per chunk, and the
    // chunk's dist2 sum (a tree; the exact pass corrects it by its updates)
    constexpr int kPP = kFoldChunk / kPruneThreads;
    constexpr int kW = kPruneThreads / 32;
    __shared__ unsigned wcnt[kW], wbase[kW], bbase;
    __shared__ double wsum[kW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long base = static_cast<long long>(blockIdx.x) * kFoldChunk + threadIdx.x;
    unsigned m[kPP];
    double bs = 0.0;
    unsigned wc = 0;
    // all loads first (memory-level parallelism), then the gathers, then the tests
    double D[kPP], C[kPP];
    uint32_t nr[kPP];
#pragma unroll
    for (int j = 0; j < kPP; ++j) {
        const long long p = base + j * kPruneThreads;
        D[j] = p < N ? dist2[p] : 0.0;
        nr[j] = p < N && t > 0 ? near[p] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kPP; ++j) C[j] = t > 0 ? dc[nr[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < kPP; ++j) {
        const long long p = base + j * kPruneThreads;
        bool need = p < N;
        bs += D[j];
        // squared form of dc(near) (1 - 1e-12) >= 2 sqrt(D) (1 + 1e-9), with
        // wider margins (the fp64 products round within 2^-52)
        if (need && t > 0 && D[j] < kPosInf && C[j] * C[j] * (1.0 - 1e-11) >= 4.0 * D[j] * (1.0 + 1e-8)) need = false;
        m[j] = __ballot_sync(0xffffffffu, need);
        wc += __popc(m[j]);
    }
    bs = warp_sum(bs);
    if (lane == 0) {
        wcnt[warp] = wc;
        wsum[warp] = bs;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        double cs = 0.0;
        for (int w = 0; w < kW; ++w) {
            wbase[w] = tot;
            tot += wcnt[w];
            cs += wsum[w];
        }
        bbase = tot ? atomicAdd(count, tot) : 0u;
        csum[blockIdx.x] = cs;
        bsum[blockIdx.x] = cs;  // the pre-update sum (pp_pick_kernel's error bound)
    }
    __syncthreads();
    unsigned off = bbase + wbase[warp];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kPP; ++j) {
        if ((m[j] >> lane) & 1) list[off + __popc(m[j] & lt)] = static_cast<uint32_t>(base + j * kPruneThreads);
        off += __popc(m[j]);
    }
}

// Exact pass over the listed points: each warp stages 32 listed rows in
// shared memory with coalesced loads (row stride d + 1: conflict-free), then
// lane j folds row j sequentially in fp64 (kmeans.cpp:12-19) and applies the
// strict-< update (kmeans.cpp:38).
template <typename T>
__global__ void __launch_bounds__(128) pp_exact_kernel(const T* __restrict__ X, int d,
                                                       const uint32_t* __restrict__ chosen, int t,
                                                       double* __restrict__ dist2, uint32_t* __restrict__ near,
                                                       const uint32_t* __restrict__ list,
                                                       const unsigned* __restrict__ count,
                                                       double* __restrict__ csum, int cshift, PPB pb) {
    const int y = blockIdx.y;  // the center load below runs before the wait (see pp_filter_i8_kernel)
    if (t + 1 >= pb.k[y]) {
        pdl_wait();
        pdl_launch_dependents();
        return;
    }
    chosen += y * pb.sK;
    dist2 += y * pb.sN;
    near += y * pb.sN;
    list += y * pb.sN;
    count += y;
    csum += y * pb.sC;
    extern __shared__ __align__(16) unsigned char dyn[];
    double* cs = reinterpret_cast<double*>(dyn);  // the new seed, fp64
    T* rows = reinterpret_cast<T*>(cs + d);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T* buf = rows + static_cast<size_t>(warp) * 32 * (d + 1);
    const long long last = chosen[t];
    for (int k = threadIdx.x; k < d; k += blockDim.x) cs[k] = static_cast<double>(X[last * d + k]);
    __syncthreads();
    pdl_wait();  // the filter's survivor list
    pdl_launch_dependents();
    const unsigned cnt = *count;
    for (unsigned b0 = (blockIdx.x * nw + warp) * 32u; b0 < cnt; b0 += gridDim.x * nw * 32u) {
        const unsigned nb = cnt - b0 < 32u ? cnt - b0 : 32u;
        const uint32_t mine = lane < static_cast<int>(nb) ? list[b0 + lane] : 0u;
        for (unsigned j = 0; j < nb; ++j) {
            const long long row = __shfl_sync(0xffffffffu, mine, j);
            for (int k = lane; k < d; k += 32) cp_async_elem(&buf[j * (d + 1) + k], X + row * d + k);
        }
        cp_async_commit();
        cp_async_wait<0>();  // one memory latency per 32 rows
        __syncwarp();
        if (lane < static_cast<int>(nb)) {
            const T* r = buf + lane * (d + 1);
            double acc = 0.0;
            for (int k = 0; k < d; ++k) {
                const double df = xsub(static_cast<double>(r[k]), cs[k]);
                acc = xadd(acc, xmul(df, df));
            }
            const double old = dist2[mine];
            if (acc < old) {
                dist2[mine] = acc;
                near[mine] = static_cast<uint32_t>(t);
                if (old < kPosInf) atomicAdd(&csum[mine >> cshift], acc - old);
            }
        }
        __syncwarp();
    }
}

// ---- fp16 pre-filter of the exact pass --------------------------------------
// Most listed points cannot update (the triangle bound is weak in high
// dimensions), yet proving it exactly costs a 4d-byte row read and a d-step
// fp64 fold. An fp16 copy x^ = s h (s a power of two per row, |h| <= 1) with
// a rigorous eps_x >= ||x - x^||_2 decides most of them from 2d bytes:
//   ||x - c|| >= ||x^ - c32|| - eps_x - eps_c        (norm triangle inequality)
// with c32 the fp32 center (eps_c >= ||c - c32||) and ||x^ - c32||^2 from an
// fp32 sum whose relative error is below (dp + 4) 2^-23. When the square of
// that lower bound, less 1e-12 relative (the fp64 fold's own error is below
// (d + 2) 2^-53), is >= dist2[i], the exact fold cannot be < dist2[i]
// (kmeans.cpp:38 updates on strict <), so the point is skipped; every other
// point gets the exact fold.
constexpr int kFiltMaxQ = 4;  // 8-byte chunks per lane: rows of up to 512 halves
#ifdef LCN_WALK_PROFILE
__device__ unsigned long long g_filt_surv;
#endif

template <typename T>
__global__ void __launch_bounds__(256) pp_half_prep_kernel(const T* __restrict__ X, long long N, int d, int dp,
                                                           __half* __restrict__ Xh, float2* __restrict__ se) {
    const long long row = blockIdx.x * 8LL + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= N) return;
    const T* x = X + row * d;
    double m = 0.0;
    for (int k = lane; k < d; k += 32) m = fmax(m, fabs(static_cast<double>(x[k])));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    int e = 0;
    frexp(m, &e);  // m < 2^e
    const bool ok = m == 0.0 || (m < 1e30 && m > 1e-30);
    const double sc = ldexp(1.0, e), inv = ldexp(1.0, -e);
    double err2 = 0.0;
    for (int k = lane; k < dp; k += 32) {
        const double v = k < d ? static_cast<double>(x[k]) : 0.0;
        const __half h = __float2half_rn(static_cast<float>(v * inv));
        Xh[row * dp + k] = h;
        const double df = v - static_cast<double>(__half2float(h)) * sc;
        err2 += df * df;
    }
    err2 = warp_sum(err2);
    if (lane == 0)
        se[row] = make_float2(static_cast<float>(sc), ok ? __double2float_ru(sqrt(err2) * (1.0 + 1e-12) + 1e-300)
                                                         : kPosInf);
}

// int8 filter copy: per row a power-of-two scale s with max |x| / s <= 127,
// q_k = rint(x_k / s) (q s exact in fp32), and eps = |x - q s| in fp64,
// rounded up: half the bytes of the fp16 copy per listed point for the
// filter pass, whose rigorous bound absorbs the coarser grid.
template <typename T>
__global__ void __launch_bounds__(256) pp_i8_prep_kernel(const T* __restrict__ X, long long N, int d, int dp,
                                                         int8_t* __restrict__ Xq, float2* __restrict__ se,
                                                         int* __restrict__ qn) {
    const long long row = blockIdx.x * 8LL + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= N) return;
    const T* x = X + row * d;
    double m = 0.0;
    for (int k = lane; k < d; k += 32) m = fmax(m, fabs(static_cast<double>(x[k])));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const bool ok = m == 0.0 || (m < 1e30 && m > 1e-30);
    int e = 0;
    frexp(m / 127.0, &e);  // m / 127 < 2^e
    const double sc = ok && m > 0.0 ? ldexp(1.0, e) : 1.0, inv = 1.0 / sc;
    double err2 = 0.0;
    int q2 = 0;
    for (int k = lane; k < dp; k += 32) {
        const double v = k < d ? static_cast<double>(x[k]) : 0.0;
        double qv = ok ? rint(v * inv) : 0.0;
        qv = fmin(fmax(qv, -127.0), 127.0);
        Xq[row * dp + k] = static_cast<int8_t>(qv);
        const double df = v - qv * sc;
        err2 += df * df;
        q2 += static_cast<int>(qv) * static_cast<int>(qv);
    }
    err2 = warp_sum(err2);
    q2 = warp_sum(q2);
    if (lane == 0) {
        se[row] = make_float2(static_cast<float>(sc), ok ? __double2float_ru(sqrt(err2) * (1.0 + 1e-12) + 1e-300)
                                                         : kPosInf);
        if (qn) qn[row] = q2;  // |q|^2, exact (<= 512 * 127^2)
    }
}

// 32 values per lane -> lane l gets the warp sum of value l (31 shuffles)
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const bool hi = lane & w;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const float send = hi ? v[i] : v[i + w];
            const float keep = hi ? v[i + w] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
    }
    return v[0];
}

// Filter only (the default): the same bound as pp_filter_exact_kernel, but
// the survivors are appended to `surv` and folded by pp_exact_kernel in a
// second launch with 32 lanes per warp. Folding them inside the filter kept
// 8 lanes busy for a 128-step dependent fp64 chain between two batches of
// row loads, so the filter pass streamed at < 3 TB/s. Here a warp issues
// all 32 rows' loads of a batch before it computes, and the next batch's
// list entries, scales and dist2 are loaded before the current batch is
// reduced.
template <typename T, typename QT, int NQ>
__global__ void __launch_bounds__(128) pp_filter_kernel(const T* __restrict__ X, const QT* __restrict__ Xh,
                                                        const float2* __restrict__ se, int d, int dp,
                                                        const uint32_t* __restrict__ chosen, int t,
                                                        const double* __restrict__ dist2,
                                                        const uint32_t* __restrict__ list,
                                                        const unsigned* __restrict__ count,
                                                        uint32_t* __restrict__ surv, unsigned* __restrict__ surv_count,
                                                        PPB pb) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (t + 1 >= pb.k[y]) return;
    chosen += y * pb.sK;
    dist2 += y * pb.sN;
    list += y * pb.sN;
    count += y;
    surv += y * pb.sN;
    surv_count += y;
    __shared__ float c32[NQ * 128];
    __shared__ double eps_part[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long last = chosen[t];
    double e2 = 0.0;
    for (int k = threadIdx.x; k < NQ * 128; k += blockDim.x) {
        const double v = k < d ? static_cast<double>(X[last * d + k]) : 0.0;
        const float f = static_cast<float>(v);
        c32[k] = f;
        const double df = v - static_cast<double>(f);
        e2 += df * df;
    }
    e2 = warp_sum(e2);
    if (lane == 0) eps_part[warp] = e2;
    __syncthreads();
    double ec2 = 0.0;
    for (int w = 0; w < nw; ++w) ec2 += eps_part[w];
    const double ec = sqrt(ec2) * (1.0 + 1e-12) + 1e-300;
    const double gam = 1.0 - (dp + 4) * 1.1920928955078125e-07;  // (dp + 4) 2^-23
    float4 cq[NQ];
    bool qin[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int ch = lane + 32 * q;
        qin[q] = ch * 4 < dp;
        cq[q] = qin[q] ? make_float4(c32[4 * ch], c32[4 * ch + 1], c32[4 * ch + 2], c32[4 * ch + 3])
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const unsigned cnt = *count;
    const unsigned stride = gridDim.x * nw * 32u;
    unsigned b0 = (blockIdx.x * nw + warp) * 32u;
    // batch b0's list entry, scale and dist2 (prefetched one batch ahead)
    uint32_t mine = 0;
    float2 my_se = make_float2(0.f, 0.f);
    double my_d2 = 0.0;
    if (b0 < cnt && lane < static_cast<int>(min(32u, cnt - b0))) {
        mine = list[b0 + lane];
        my_se = se[mine];
        my_d2 = dist2[mine];
    }
    for (; b0 < cnt; b0 += stride) {
        const unsigned nb = cnt - b0 < 32u ? cnt - b0 : 32u;
        // rows past the batch read row 0 (harmless; their lanes are ignored)
        // rows in groups of RB: at most 32 8-byte loads in flight per lane
        // (the register budget), issued before the group is reduced
        using Raw = typename std::conditional<sizeof(QT) == 2, uint2, int>::type;
        constexpr int RB = NQ == 1 ? 32 : 8;
        float part[32];
        // the next batch's list entries (independent of this batch's rows)
        const unsigned b1 = b0 + stride;
        uint32_t nmine = 0;
        float2 nse = make_float2(0.f, 0.f);
        double nd2 = 0.0;
#pragma unroll
        for (int g = 0; g < 32; g += RB) {
            Raw raw[RB][NQ];
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                const long long row = __shfl_sync(0xffffffffu, mine, g + j);
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (qin[q]) raw[j][q] = __ldcs(reinterpret_cast<const Raw*>(Xh + row * dp + 4 * (lane + 32 * q)));
            }
            if (g == 0 && b1 < cnt && lane < static_cast<int>(min(32u, cnt - b1))) {
                nmine = list[b1 + lane];
                nse = se[nmine];
                nd2 = dist2[nmine];
            }
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                const float sj = __shfl_sync(0xffffffffu, my_se.x, g + j);
                float acc = 0.f;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    if (!qin[q]) continue;
                    float2 a, b;
                    if constexpr (sizeof(QT) == 2) {
                        a = __half22float2(*reinterpret_cast<const __half2*>(&raw[j][q].x));
                        b = __half22float2(*reinterpret_cast<const __half2*>(&raw[j][q].y));
                    } else {
                        const char4 c4 = *reinterpret_cast<const char4*>(&raw[j][q]);
                        a = make_float2(static_cast<float>(c4.x), static_cast<float>(c4.y));
                        b = make_float2(static_cast<float>(c4.z), static_cast<float>(c4.w));
                    }
                    const float d0 = fmaf(a.x, sj, -cq[q].x), d1 = fmaf(a.y, sj, -cq[q].y);
                    const float d2 = fmaf(b.x, sj, -cq[q].z), d3 = fmaf(b.y, sj, -cq[q].w);
                    acc = fmaf(d0, d0, acc);
                    acc = fmaf(d1, d1, acc);
                    acc = fmaf(d2, d2, acc);
                    acc = fmaf(d3, d3, acc);
                }
                part[g + j] = acc;
            }
        }
        const float A = transpose_reduce32(part, lane);
        bool need = false;
        if (lane < static_cast<int>(nb)) {
            const double lo = sqrt(static_cast<double>(A) * gam) - static_cast<double>(my_se.y) - ec;
            need = !(lo > 0.0 && lo * lo * (1.0 - 1e-12) >= my_d2);
        }
        const unsigned sv = __ballot_sync(0xffffffffu, need);
        if (sv) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(surv_count, static_cast<unsigned>(__popc(sv)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (need) surv[base + __popc(sv & ((1u << lane) - 1u))] = mine;
        }
        mine = nmine;
        my_se = nse;
        my_d2 = nd2;
    }
}

// Integer filter over int8 rows (the default filter). The new center is
// quantised per step to int16 with a power-of-two scale s_c (c^ = s_c q_c,
// eps_c >= |c - c^|), so the squared distance of the two quantised points,
//   |x^ - c^|^2 = s_x^2 |q_x|^2 - 2 s_x s_c (q_x . q_c) + s_c^2 |q_c|^2,
// needs only the integer dot q_x . q_c: two dp2a per lane and row (int16 x
// int8, exact int32) instead of four int8 -> fp32 conversions and eight
// FMAs (the conversions made the early, all-candidate steps issue-bound:
// ncu, 50 % SM throughput at 2.4 TB/s). |q_x|^2 comes from the prep pass.
// The three terms are exact in fp64 and the two adds err by < 2^-52 of
// their magnitudes; then, as before, |x - c| >= |x^ - c^| - eps_x - eps_c.
template <int NQ>
__device__ __forceinline__ int dp2a_row(const int (&raw)[NQ], const int (&qlo)[NQ], const int (&qhi)[NQ]) {
    int acc = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        acc = __dp2a_lo(qlo[q], raw[q], acc);
        acc = __dp2a_hi(qhi[q], raw[q], acc);
    }
    return acc;
}

template <typename T, int NQ>
__global__ void __launch_bounds__(128) pp_filter_i8_kernel(const T* __restrict__ X, const int8_t* __restrict__ Xq,
                                                           const float2* __restrict__ se, const int* __restrict__ qn,
                                                           int d, int dp, const uint32_t* __restrict__ chosen, int t,
                                                           const double* __restrict__ dist2,
                                                           const uint32_t* __restrict__ list,
                                                           const unsigned* __restrict__ count,
                                                           uint32_t* __restrict__ surv,
                                                           unsigned* __restrict__ surv_count, PPB pb) {
    // the center's quantisation needs only chosen[t] (the previous step's
    // pick, complete before the prune kernel passed its wait) and X: it runs
    // before this grid waits for the prune kernel
    const int y = blockIdx.y;
    if (t + 1 >= pb.k[y]) {
        pdl_wait();
        pdl_launch_dependents();
        return;
    }
    chosen += y * pb.sK;
    dist2 += y * pb.sN;
    list += y * pb.sN;
    count += y;
    surv += y * pb.sN;
    surv_count += y;
    __shared__ short qc[NQ * 128];
    __shared__ double wred[4][2];
    __shared__ double cmax_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long last = chosen[t];
    // scale of the center: a power of two with max |c| / s_c <= 32767
    double m = 0.0;
    for (int k = threadIdx.x; k < d; k += blockDim.x) m = fmax(m, fabs(static_cast<double>(X[last * d + k])));
    m = warp_max(m);
    if (lane == 0) wred[warp][0] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int w = 0; w < nw; ++w) mm = fmax(mm, wred[w][0]);
        cmax_s = mm;
    }
    __syncthreads();
    const double cmax = cmax_s;
    int e = 0;
    frexp(cmax / 32767.0, &e);  // cmax / 32767 < 2^e
    const bool cok = cmax < 1e30 && (cmax == 0.0 || cmax > 1e-30);
    const double sc = cok && cmax > 0.0 ? ldexp(1.0, e) : 1.0, inv = 1.0 / sc;
    double e2 = 0.0, n2 = 0.0;
    for (int k = threadIdx.x; k < NQ * 128; k += blockDim.x) {
        const double v = k < d ? static_cast<double>(X[last * d + k]) : 0.0;
        double qv = cok ? rint(v * inv) : 0.0;
        qv = fmin(fmax(qv, -32767.0), 32767.0);
        qc[k] = static_cast<short>(qv);
        const double df = v - qv * sc;
        e2 += df * df;
        n2 += qv * qv;  // exact: integers < 2^53
    }
    e2 = warp_sum(e2);
    n2 = warp_sum(n2);
    __syncthreads();  // wred reuse
    if (lane == 0) {
        wred[warp][0] = e2;
        wred[warp][1] = n2;
    }
    __syncthreads();
    double ec2 = 0.0, ncq = 0.0;
    for (int w = 0; w < nw; ++w) {
        ec2 += wred[w][0];
        ncq += wred[w][1];
    }
    const double ec = cok ? sqrt(ec2) * (1.0 + 1e-12) + 1e-300 : kPosInf;
    const double sc2n = sc * sc * ncq;
    int qlo[NQ], qhi[NQ];
    bool qin[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int ch = lane + 32 * q;
        qin[q] = ch * 4 < dp;
        const int k = qin[q] ? 4 * ch : 0;
        qlo[q] = qin[q] ? (static_cast<unsigned short>(qc[k]) | (static_cast<int>(qc[k + 1]) << 16)) : 0;
        qhi[q] = qin[q] ? (static_cast<unsigned short>(qc[k + 2]) | (static_cast<int>(qc[k + 3]) << 16)) : 0;
    }
    pdl_wait();  // the prune kernel's candidate list
    pdl_launch_dependents();
    const unsigned cnt = *count;
    const unsigned stride = gridDim.x * nw * 32u;
    unsigned b0 = (blockIdx.x * nw + warp) * 32u;
    uint32_t mine = 0;
    float2 my_se = make_float2(0.f, 0.f);
    double my_d2 = 0.0;
    int my_qn = 0;
    if (b0 < cnt && lane < static_cast<int>(min(32u, cnt - b0))) {
        mine = list[b0 + lane];
        my_se = se[mine];
        my_d2 = dist2[mine];
        my_qn = qn[mine];
    }
    const unsigned lt = (1u << lane) - 1u;
    for (; b0 < cnt; b0 += stride) {
        const unsigned nb = cnt - b0 < 32u ? cnt - b0 : 32u;
        constexpr int RB = NQ == 1 ? 32 : 16;
        int part[32];
        const unsigned b1 = b0 + stride;
        uint32_t nmine = 0;
        float2 nse = make_float2(0.f, 0.f);
        double nd2 = 0.0;
        int nqn = 0;
#pragma unroll
        for (int g = 0; g < 32; g += RB) {
            int raw[RB][NQ];
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                // rows past the batch read row 0 (harmless; their lanes are ignored)
                const long long row = __shfl_sync(0xffffffffu, mine, g + j);
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    raw[j][q] = qin[q] ? __ldcs(reinterpret_cast<const int*>(Xq + row * dp + 4 * (lane + 32 * q))) : 0;
            }
            if (g == 0 && b1 < cnt && lane < static_cast<int>(min(32u, cnt - b1))) {
                nmine = list[b1 + lane];
                nse = se[nmine];
                nd2 = dist2[nmine];
                nqn = qn[nmine];
            }
#pragma unroll
            for (int j = 0; j < RB; ++j) part[g + j] = dp2a_row<NQ>(raw[j], qlo, qhi);
        }
        // lane l gets the dot of row l (exact integer sums)
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
            const bool hi = lane & w;
#pragma unroll
            for (int i = 0; i < w; ++i) {
                const int send = hi ? part[i] : part[i + w];
                const int keep = hi ? part[i + w] : part[i];
                part[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
            }
        }
        bool need = false;
        if (lane < static_cast<int>(nb)) {
            const double sx = static_cast<double>(my_se.x);
            const double t1 = sx * sx * static_cast<double>(my_qn);
            const double t2 = 2.0 * sx * sc * static_cast<double>(part[0]);
            const double a2 = (t1 - t2) + sc2n;
            const double a2lo = a2 - 4.440892098500626e-16 * (t1 + fabs(t2) + sc2n);  // 2^-51
            const double lo = sqrt(fmax(a2lo, 0.0)) * (1.0 - 2.220446049250313e-16) - static_cast<double>(my_se.y) - ec;
            need = !(lo > 0.0 && lo * lo * (1.0 - 1e-12) >= my_d2);
        }
        const unsigned sv = __ballot_sync(0xffffffffu, need);
        if (sv) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(surv_count, static_cast<unsigned>(__popc(sv)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (need) surv[base + __popc(sv & lt)] = mine;
        }
        mine = nmine;
        my_se = nse;
        my_d2 = nd2;
        my_qn = nqn;
    }
}

// dc[j] = |x_{chosen[j]} - x_{chosen[t]}| for j < t (fp64, one warp per j)
template <typename T>
__global__ void __launch_bounds__(256) seed_dist_kernel(const T* __restrict__ X, int d,
                                                        const uint32_t* __restrict__ chosen, int t,
                                                        double* __restrict__ dc, unsigned* __restrict__ surv_count,
                                                        PPB pb) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (t + 1 >= pb.k[y]) return;
    chosen += y * pb.sK;
    dc += y * pb.sK;
    if (surv_count && blockIdx.x == 0 && threadIdx.x == 0) surv_count[y] = 0u;  // this step's filter survivors
    const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (j >= t) return;
    const long long a = chosen[j], b = chosen[t];
    double s2 = 0.0;
    for (int k = lane; k < d; k += 32) {
        const double df = static_cast<double>(X[a * d + k]) - static_cast<double>(X[b * d + k]);
        s2 += df * df;
    }
    s2 = warp_sum(s2);
    if (lane == 0) dc[j] = sqrt(s2);
}

// Exact emulation of the sequential fp64 fold s_{i+1} = fl(s_i + x_i)
// (kmeans.cpp:36-40, 51-58). While s is a normal number in the binade
// [2^e, 2^(e+1)) its grid is u = 2^(e-52) and fl(s + x) = s + u * RN(x/u)
// (x >= 0), RN ties to even on the running significand (ParInc below); runs
// of elements are composed exactly in int64. An element leaves the fast path
// when x/u is huge or the running sum would reach 2^(e+1); it is added with a
// real fp64 add and the binade is recomputed. With search, the fold also
// returns the first index whose running sum is >= target and whose element is
// > 0 (kmeans.cpp:51-58).
constexpr double kMinNormal = 2.2250738585072014e-308;
constexpr long long kTwo53 = 1LL << 53;
constexpr long long kTwo52 = 1LL << 52;

// IEEE-754 bit access for positive normal doubles (exact, no libm calls):
// binade exponent, 53-bit integer significand, and the inverse.
__device__ __forceinline__ int dbl_exp(double s) {
    return static_cast<int>((__double_as_longlong(s) >> 52) & 0x7ff) - 1023;
}
__device__ __forceinline__ long long dbl_sig(double s) {
    return (__double_as_longlong(s) & (kTwo52 - 1)) | kTwo52;
}
__device__ __forceinline__ double dbl_make(long long sig, int e) {  // sig in [2^52, 2^53)
    return __longlong_as_double((static_cast<long long>(e + 1023) << 52) | (sig - kTwo52));
}
// x * 2^(52 - e), correctly rounded like scalbn (a product with an exact
// power of two); scalbn itself when the power is not representable
__device__ __forceinline__ double scale_to_grid(double x, int e) {
    const int k = 52 - e;
    if (k <= 1023 && k >= -1022) return x * __longlong_as_double(static_cast<long long>(k + 1023) << 52);
    return scalbn(x, k);
}

// Effect of a run of additions on the integer significand S (grid u of one
// binade): an element x = u (K + f) adds K, or K + 1 when f > 1/2; an exact
// tie f = 1/2 rounds to even, adding K + ((S + K) & 1). So a run maps S to
// S + inc[S & 1]; runs compose associatively:
//   (f then g).inc[p] = f.inc[p] + g.inc[(p + f.inc[p]) & 1].
struct ParInc {
    long long i0, i1;
};
// Increments saturate at 2^61: a run that large has left its binade anyway
// (only runs below 2^53 are used), and int64 cannot overflow.
constexpr long long kIncSat = 1LL << 61;
__device__ __forceinline__ ParInc par_compose(ParInc f, ParInc g) {
    const long long a = f.i0 + ((f.i0 & 1) ? g.i1 : g.i0);
    const long long b = f.i1 + (((1 + f.i1) & 1) ? g.i1 : g.i0);
    return {a < kIncSat ? a : kIncSat, b < kIncSat ? b : kIncSat};
}
// element x scaled to the grid (q = x / u, 0 <= q < 2^53)
__device__ __forceinline__ ParInc par_element(double q) {
    const double K = floor(q), f = q - K;
    const long long k = static_cast<long long>(K);
    if (f == 0.5) return {k + (k & 1), k + ((k + 1) & 1)};
    const long long r = k + (f > 0.5 ? 1 : 0);
    return {r, r};
}
__device__ __forceinline__ ParInc par_shfl_up(ParInc v, int o) {
    return {__shfl_up_sync(0xffffffffu, v.i0, o), __shfl_up_sync(0xffffffffu, v.i1, o)};
}
// inclusive warp scan of ParInc in lane order (identity {0, 0})
__device__ __forceinline__ ParInc par_scan(ParInc v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const ParInc t = par_shfl_up(v, o);
        if (lane >= o) v = par_compose(t, v);
    }
    return v;
}

// Conversion-free par_element: for 0 <= q < 2^52, q + 2^52 rounds q to the
// nearest integer with ties to even (the grid of [2^52, 2^53) is 1), and the
// bits of that sum minus the bits of 2^52 are the integer itself. A tie
// (|q - RNE(q)| == 1/2, exact by Sterbenz) gives the other neighbour for the
// odd parity. q in [2^52, 2^53) is already an integer. Same values as
// par_element.
constexpr double kTwo52d = 4503599627370496.0;
__device__ __forceinline__ ParInc par_element_fast(double q) {
    const bool hiq = q >= kTwo52d;
    const double t = hiq ? q : q + kTwo52d;
    const long long r = __double_as_longlong(t) - 0x4330000000000000LL + (hiq ? kTwo52 : 0);
    const double diff = hiq ? 0.0 : q - (t - kTwo52d);
    const long long r1 = fabs(diff) == 0.5 ? r + (diff > 0.0 ? 1 : -1) : r;
    return {r, r1};
}
// Composition without saturation, for operands whose components are at most
// 2^53 each and at most 2^10 of them (no int64 overflow); stored plans are
// clamped to 2^53 (a clamped run leaves its binade anyway).
__device__ __forceinline__ ParInc par_compose_ns(ParInc f, ParInc g) {
    return {f.i0 + ((f.i0 & 1) ? g.i1 : g.i0), f.i1 + ((f.i1 & 1) ? g.i0 : g.i1)};
}
__device__ __forceinline__ ParInc par_scan_ns(ParInc v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const ParInc t = par_shfl_up(v, o);
        if (lane >= o) v = par_compose_ns(t, v);
    }
    return v;
}
__device__ __forceinline__ longlong2 par_clamp(ParInc v) {
    return make_longlong2(min(v.i0, kTwo53), min(v.i1, kTwo53));
}

// ---- chunk-parallel exact fold ----------------------------------------------
// The fold over N values is cut into chunks of kFoldChunk. Most chunks lie
// inside one binade of the running sum, where the fold's result depends only
// on that binade: S_end = S_start + u_e * sum_j RN(x_j / u_e). So
//   A) approximate chunk sums (any order; accumulated by the prune pass,
//      corrected by the exact pass)                  -> predicted start A_c
//   B) predicted binade e_c of each chunk (dirty if the interval
//      [A_c (1-1e-9), A_{c+1} (1+1e-9)] straddles a power of two)
//   C) the chunk's parity function R_c(e_c) = {inc[0], inc[1]} in parallel
//      (ties included), dirty only on huge x; B and C in fold_round
//   D) one warp walks the chunks in order with the exact running sum: runs
//      of clean chunks whose actual binade matches e_c advance by a
//      parity-scan of their R_c, any other chunk by warp_fold_chunk
//      (segment tables, literal folds where the binade changes).
// The prediction only decides which path a chunk takes; the walk re-checks
// the actual binade, so the result is exact regardless.

__global__ void fold_chunk_sum_kernel(const double* __restrict__ x, long long N, double* __restrict__ csum,
                                      double* __restrict__ bsum, int hs, PPB pb) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (hs >= pb.k[y]) return;
    x += y * pb.sN;
    csum += y * pb.sC;
    bsum += y * pb.sC;
    __shared__ double red[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long b0 = static_cast<long long>(blockIdx.x) * kFoldChunk + warp * 256;
    double s = 0.0;
    for (int j = 0; j < 8; ++j) {
        const long long i = b0 + lane + 32 * j;
        s += i < N ? x[i] : 0.0;
    }
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        csum[blockIdx.x] = t;
        bsum[blockIdx.x] = t;
    }
}

// C) per chunk: its parity function for the predicted binade (clean chunks)
// and, per segment of kSegLen elements, a predicted base binade eb_s (from
// the approximate running sum at the segment's start and end) with the
// segment's parity functions for binades eb_s and eb_s + 1. The walk skips
// whole segments with them and folds literally only the segments in which
// the running sum changes binade; the first such segment (predicted) is
// recorded so the walk can prefetch it. Segments get their own base binade
// so that even the first chunk, where the sum climbs many binades from zero,
// is mostly skipped.
constexpr int kSegLen = 64;
constexpr int kSegs = kFoldChunk / kSegLen;
static_assert(kSegs == 32, "one segment table entry per lane and binade");
constexpr int kRoundPer = kFoldChunk / 256;          // contiguous elements per thread
constexpr int kLanesPerSeg = kSegLen / kRoundPer;    // lanes per segment
static_assert(kLanesPerSeg == 8, "segmented scans below are width 8");
constexpr int kNoBinade = -100000;

__device__ __forceinline__ ParInc par_scan8(ParInc v, int lane) {  // inclusive, within 8-lane groups
#pragma unroll
    for (int o = 1; o < kLanesPerSeg; o <<= 1) {
        const ParInc t = par_shfl_up(v, o);
        if ((lane & (kLanesPerSeg - 1)) >= o) v = par_compose_ns(t, v);
    }
    return v;
}

// predicted binade of a fold interval [lo, hi] (approximate sums widened by
// 1e-9): its binade when it has one, the lower one when it straddles one
// power of two, none otherwise
__device__ __forceinline__ void predict_binade(double a, double b, int& e_one, int& e_base) {
    const double lo = a * (1.0 - 1e-9), hi = b * (1.0 + 1e-9);
    e_one = e_base = kNoBinade;
    if (lo >= kMinNormal && hi < kPosInf) {
        const int el = ilogb(lo), eh = ilogb(hi);
        if (el == eh) e_one = el;
        if (eh - el <= 1) e_base = el;
    }
}

// One chunk of fold_round_kernel (cb = the chunk).
__device__ __forceinline__ void fold_round_chunk(const int cb, const double* __restrict__ x, long long N,
                                                 const double* __restrict__ csum, int* __restrict__ ebin,
                                                 longlong2* __restrict__ R, longlong2* __restrict__ Rseg,
                                                 int* __restrict__ Eseg, int* __restrict__ spred,
                                                 unsigned* __restrict__ smask, double* __restrict__ s0end) {
    __shared__ ParInc stot[kSegs];
    __shared__ double ssum[kSegs];
    __shared__ double red[8];
    __shared__ int sbase[kSegs];
    __shared__ int all_one, e_chunk;
    __shared__ __align__(16) double c0buf[kFoldChunk];  // chunk 0, folded literally by block 0
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / kLanesPerSeg;
    const int si = warp * (32 / kLanesPerSeg) + g;
    const long long b = static_cast<long long>(cb) * kFoldChunk + threadIdx.x * kRoundPer;
    double xv[kRoundPer];
    double xsum = 0.0;
#pragma unroll
    for (int j = 0; j < kRoundPer; ++j) {
        xv[j] = b + j < N ? x[b + j] : 0.0;
        xsum += xv[j];
    }
    // approximate start of this chunk: the earlier chunks' approximate sums
    double a = 0.0;
    for (int c = threadIdx.x; c < static_cast<int>(cb); c += 256) a += csum[c];
    a = warp_sum(a);
    if (lane == 0) red[warp] = a;
#pragma unroll
    for (int o = 1; o < kLanesPerSeg; o <<= 1) xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
    if ((lane & (kLanesPerSeg - 1)) == 0) ssum[si] = xsum;
    if (cb == 0)
#pragma unroll
        for (int j = 0; j < kRoundPer; ++j) c0buf[threadIdx.x * kRoundPer + j] = xv[j];
    __syncthreads();
    if (warp == 0) {  // approximate segment starts -> per-segment binades
        double a0 = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) a0 += red[w];
        const double v = ssum[lane];
        double incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double tt = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += tt;
        }
        int e_one, e_base, ec_one, ec_base;
        predict_binade(a0 + (incl - v), a0 + incl, e_one, e_base);
        predict_binade(a0, a0 + __shfl_sync(0xffffffffu, incl, 31), ec_one, ec_base);
        sbase[lane] = e_base;
        Eseg[static_cast<long long>(cb) * kSegs + lane] = e_base;
        const unsigned straddle = __ballot_sync(0xffffffffu, e_one == kNoBinade);
        const unsigned one = __ballot_sync(0xffffffffu, e_one == ec_one && ec_one != kNoBinade);
        if (lane == 0) {
            all_one = one == 0xffffffffu;
            e_chunk = ec_one;
            ebin[cb] = ec_one;
            spred[cb] = straddle ? __ffs(straddle) - 1 : 0;
            smask[cb] = straddle;
        }
    }
    __syncthreads();
    const int eb = sbase[si];
    ParInc acc0{0, 0}, acc1{0, 0};
    bool bad0 = eb == kNoBinade, bad1 = eb == kNoBinade;
    if (eb != kNoBinade) {
        // grid scalings 2^(52-eb), 2^(51-eb) as exact power-of-two products
        // when representable (scale_to_grid's fast path), else scalbn per
        // element. Each map is at most 2^53 (q < 2^53), so 8 of them compose
        // without saturation.
        const int k0 = 52 - eb;
        const bool fast = k0 <= 1023 && k0 - 1 >= -1022;
        const double f0 = fast ? __longlong_as_double(static_cast<long long>(k0 + 1023) << 52) : 0.0;
        const double f1 = fast ? __longlong_as_double(static_cast<long long>(k0 + 1022) << 52) : 0.0;
        // one binade at a time (register pressure: 4 blocks per SM)
        auto maps = [&](double f, int e, bool& bad) {
            ParInc p[kRoundPer];
#pragma unroll
            for (int j = 0; j < kRoundPer; ++j) {
                const double q = fast ? xv[j] * f : scale_to_grid(xv[j], e);
                const bool in = b + j < N;
                bad |= in && !(q < 9007199254740992.0);
                p[j] = in && q < 9007199254740992.0 ? par_element_fast(q) : ParInc{0, 0};
            }
            return par_compose_ns(par_compose_ns(par_compose_ns(p[0], p[1]), par_compose_ns(p[2], p[3])),
                                  par_compose_ns(par_compose_ns(p[4], p[5]), par_compose_ns(p[6], p[7])));
        };
        acc0 = maps(f0, eb, bad0);
        acc1 = maps(f1, eb + 1, bad1);
    }
    static_assert(kRoundPer == 8, "tree composition above");
    const unsigned gmask = 0xffu << (g * kLanesPerSeg);
    const bool sbad0 = (__ballot_sync(0xffffffffu, bad0) & gmask) != 0;
    const bool sbad1 = (__ballot_sync(0xffffffffu, bad1) & gmask) != 0;
    acc0 = par_scan8(acc0, lane);
    acc1 = par_scan8(acc1, lane);
    longlong2* seg = Rseg + static_cast<long long>(cb) * (2 * kSegs);
    if ((lane & (kLanesPerSeg - 1)) == kLanesPerSeg - 1) {
        seg[si] = sbad0 ? make_longlong2(-1, -1) : par_clamp(acc0);
        seg[kSegs + si] = sbad1 ? make_longlong2(-1, -1) : par_clamp(acc1);
        const longlong2 cl = par_clamp(acc0);
        stot[si] = sbad0 ? ParInc{-1, -1} : ParInc{cl.x, cl.y};
    }
    __syncthreads();
    if (warp == 0) {
        // clean chunk: every segment predicted inside the chunk's binade; its
        // map is the composition of the segment maps (lane = segment)
        const bool ok = all_one && __ballot_sync(0xffffffffu, stot[lane].i0 < 0) == 0;
        const ParInc sl = stot[lane];
        const ParInc tot = par_scan_ns(sl.i0 < 0 ? ParInc{0, 0} : sl, lane);
        if (lane == 31) R[cb] = ok ? par_clamp(tot) : make_longlong2(-1, -1);
        if (cb == 0) {
            // chunk 0 starts the fold at 0, where the sum climbs binade after
            // binade: fold it literally here, in parallel with the other chunks
            const double2* c2 = reinterpret_cast<const double2*>(c0buf);
            const int cnt0 = static_cast<int>(min(N, static_cast<long long>(kFoldChunk)));
            double S = 0.0;
#pragma unroll 8
            for (int i = 0; i < cnt0 / 2; ++i) {
                const double2 w = c2[i];
                S = xadd(S, w.x);
                S = xadd(S, w.y);
            }
            if (cnt0 & 1) S = xadd(S, c0buf[cnt0 - 1]);
            if (lane == 0) *s0end = S;
        }
    }
    (void)e_chunk;
}

// Persistent over the chunks (grid-stride): a certified step (skip) costs
// only the resident CTAs' exit, not a 977-CTA launch.
__global__ void __launch_bounds__(256, 4) fold_round_kernel(const double* __restrict__ x, long long N,
                                                            const double* __restrict__ csum, int* __restrict__ ebin,
                                                         longlong2* __restrict__ R, longlong2* __restrict__ Rseg,
                                                         int* __restrict__ Eseg, int* __restrict__ spred,
                                                         unsigned* __restrict__ smask, double* __restrict__ s0end,
                                                         const int* __restrict__ skip, int hs, PPB pb, int nch) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (hs >= pb.k[y]) return;
    if (skip && skip[y]) return;  // pp_pick_kernel certified this step's pick
    x += y * pb.sN;
    csum += y * pb.sC;
    ebin += y * pb.sC;
    R += y * pb.sC;
    Rseg += static_cast<long long>(y) * pb.sC * 2 * kSegs;
    Eseg += static_cast<long long>(y) * pb.sC * kSegs;
    spred += y * pb.sC;
    smask += y * pb.sC;
    s0end += y;
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
        fold_round_chunk(c, x, N, csum, ebin, R, Rseg, Eseg, spred, smask, s0end);
        __syncthreads();  // the chunk's shared tables are reused by the next
    }
}

// ---- literal fold of one segment -------------------------------------------
// A segment in which the running sum changes binade, meets a huge element or
// (search) reaches the target is folded literally: s = fl(s + x_i) in index
// order, the reference's own loop. The warp stages the segment in shared
// memory and every lane runs the same add chain on broadcast loads, so no
// result needs broadcasting back. The walk is one warp: its cost is latency
// chains, and a dependent fp64 add (8 cycles) over one short segment beats
// any further parity round; the parity tables skip the segments without
// events.
constexpr int kPerLane = kSegLen / 32;
constexpr int kGrp = 8;  // search granularity
constexpr int kWalkThreads = 256;
constexpr int kMaxPre = 48;  // dirty chunks whose tables and segment are prefetched

struct SegFold {
    double s;
    long long pick;  // >= 0: search hit (global index)
};

// Development timing of the walk (build with EXTRA=-DLCN_WALK_PROFILE; the
// host prints cycles per launch when LCN_WALK_STATS is set).
#ifdef LCN_WALK_PROFILE
__device__ unsigned long long g_wt[16];
__host__ void* g_wt_ptr() {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_wt);
    return p;
}
#define WALK_T(v) const long long v = clock64()
#define WALK_ADD(i, val) if ((threadIdx.x & 31) == 0) atomicAdd(&g_wt[i], static_cast<unsigned long long>(val))
#else
#define WALK_T(v)
#define WALK_ADD(i, val)
#endif

// zero-padded: adding +0 leaves a positive sum unchanged
__device__ __noinline__ double warp_add_segment(const double* __restrict__ buf, double S) {
    const double2* b2 = reinterpret_cast<const double2*>(buf);
#pragma unroll
    for (int i = 0; i < kSegLen / 2; ++i) {
        const double2 w = b2[i];
        S = xadd(S, w.x);
        S = xadd(S, w.y);
    }
    return S;
}
// The sum is monotone: the target is reached inside a group iff the group's
// end reaches it.
__device__ __noinline__ SegFold warp_search_segment(const double* __restrict__ buf, long long g0, double S,
                                                    double target) {
#pragma unroll
    for (int g = 0; g < kSegLen / kGrp; ++g) {
        double s2 = S;
#pragma unroll
        for (int j = 0; j < kGrp; ++j) s2 = xadd(s2, buf[g * kGrp + j]);
        if (s2 >= target) {
#pragma unroll 1
            for (int j = 0; j < kGrp; ++j) {
                const double wj = buf[g * kGrp + j];
                S = xadd(S, wj);
                if (S >= target && wj > 0.0) return {S, g0 + g * kGrp + j};
            }
        }
        S = s2;
    }
    return {S, -1};
}

// Exact fold of chunk c from the running sum S (one warp). Runs of segments
// whose parity tables match S's binade advance by one scan; the segment in
// which the sum leaves the binade (or reaches the target) is folded
// literally. tabs: the chunk's 2 x kSegs tables (shared memory when
// prefetched); pre: segment sp's values when prefetched; smask: segments
// predicted to change binade (loaded while the previous one is folded).
__device__ __noinline__ SegFold warp_fold_chunk(const double* __restrict__ x, double* __restrict__ buf, long long N,
                                                int c, int sp, unsigned smask, const longlong2* __restrict__ tabs,
                                                const int* __restrict__ ebs, const double* __restrict__ pre, double S,
                                                bool search, double target) {
    const int lane = threadIdx.x & 31;
    const long long base = static_cast<long long>(c) * kFoldChunk;
    const int cnt = static_cast<int>(min(N - base, static_cast<long long>(kFoldChunk)));
    const int nseg = (cnt + kSegLen - 1) / kSegLen;
    auto load = [&](int sg, double (&v)[kPerLane]) {
        const int i0 = sg * kSegLen + lane * kPerLane;
#pragma unroll
        for (int j = 0; j < kPerLane; ++j) v[j] = i0 + j < cnt ? x[base + i0 + j] : 0.0;
    };
    // lane l: segment l's tables and base binade
    const longlong2 tab0 = tabs[lane], tab1 = tabs[kSegs + lane];
    const int eb_l = ebs[lane];
    double cur[kPerLane];
    int cur_sg = min(sp, nseg - 1);
    if (pre) {
#pragma unroll
        for (int j = 0; j < kPerLane; ++j) cur[j] = pre[lane * kPerLane + j];
    } else {
        load(cur_sg, cur);
    }
    int sg = 0;
#pragma unroll 1
    while (sg < nseg) {
        if (S >= kMinNormal && S < kPosInf) {
            const int eS = dbl_exp(S);
            const long long Si = dbl_sig(S);
            // this lane's segment map for the binade eS, if its tables have it
            const int jl = eS - eb_l;
            const longlong2 own = (eb_l == kNoBinade || (jl != 0 && jl != 1)) ? make_longlong2(-1, -1)
                                  : (jl ? tab1 : tab0);
            const int src = min(sg + lane, kSegs - 1);
            const long long t0 = __shfl_sync(0xffffffffu, own.x, src);
            const long long t1 = __shfl_sync(0xffffffffu, own.y, src);
            const bool in = sg + lane < nseg;
            const ParInc r{in ? t0 : 0, in ? t1 : 0};
            const unsigned inval = __ballot_sync(0xffffffffu, in && t0 < 0);
            int fb = inval ? __ffs(inval) - 1 : nseg - sg;
            if (fb > 0) {
                const ParInc pf = par_scan_ns(lane < fb ? r : ParInc{0, 0}, lane);
                const long long P = (Si & 1) ? pf.i1 : pf.i0;
                bool ev = lane < fb && Si + P >= kTwo53;
                if (search && lane < fb && !ev && dbl_make(Si + P, eS) >= target) ev = true;
                const unsigned evm = __ballot_sync(0xffffffffu, ev);
                if (evm) fb = min(fb, __ffs(evm) - 1);
                if (fb > 0) {
                    S = dbl_make(Si + __shfl_sync(0xffffffffu, P, fb - 1), eS);
                    sg += fb;
                    if (sg >= nseg) break;
                }
            }
        }
        if (cur_sg != sg) {
            load(sg, cur);
            cur_sg = sg;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kPerLane; ++j) buf[lane * kPerLane + j] = cur[j];
        __syncwarp();
        if (sg + 1 < nseg && ((smask >> (sg + 1)) & 1)) {  // predicted fold: load it during this one
            load(sg + 1, cur);
            cur_sg = sg + 1;
        }
        WALK_T(ts0);
        if (search) {
            const SegFold r = warp_search_segment(buf, base + static_cast<long long>(sg) * kSegLen, S, target);
            if (r.pick >= 0) return r;
            S = r.s;
        } else {
            S = warp_add_segment(buf, S);
        }
        WALK_T(ts1);
        WALK_ADD(6, ts1 - ts0);
        WALK_ADD(7, 1);
        ++sg;
    }
    return {S, -1};
}

// D) walk + draw + pick for k-means++ step t (kmeans.cpp:35-62). raw[] holds
// the caller's engine draws in order; a step with total <= 0 consumes none
// (kmeans.cpp:42-47). Warp 0 walks the chunks in order; the other warps help
// stage the chunk plans and find the target chunk.
__global__ void __launch_bounds__(kWalkThreads) pp_walk_pick_kernel(
    double* __restrict__ dist2, unsigned char* __restrict__ used, long long N, int nch, const int* __restrict__ ebin,
    const int* __restrict__ spred, const longlong2* __restrict__ R, const longlong2* __restrict__ Rseg,
    const int* __restrict__ Eseg, const unsigned* __restrict__ smask, const double* __restrict__ s0end,
    double* __restrict__ csum, unsigned* __restrict__ cand_count, double* __restrict__ sstart, const unsigned long long* __restrict__ raw, int n_raw, int* __restrict__ draw_counter,
    uint32_t* __restrict__ chosen, int t, int staged, const int* __restrict__ skip, PPB pb) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (t >= pb.k[y]) return;
    if (skip && skip[y]) return;  // pp_pick_kernel certified this step's pick
    dist2 += y * pb.sN;
    used += y * pb.sN;
    ebin += y * pb.sC;
    spred += y * pb.sC;
    R += y * pb.sC;
    Rseg += static_cast<long long>(y) * pb.sC * 2 * kSegs;
    Eseg += static_cast<long long>(y) * pb.sC * kSegs;
    smask += y * pb.sC;
    s0end += y;
    csum += y * pb.sC;
    cand_count += y;
    sstart += y * (pb.sC + 1);
    raw += y * pb.sK;
    n_raw = pb.k[y] - 1;
    draw_counter += y;
    chosen += y * pb.sK;
    __shared__ int flag_min;
    __shared__ double total;
    __shared__ __align__(16) double segbuf[kSegLen];
    __shared__ int wcount[kWalkThreads / 32];
    __shared__ int pre_list[kMaxPre];
    extern __shared__ __align__(16) unsigned char wdyn[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WALK_T(T0);
    // the next step's prune appends to the candidate list from zero
    if (threadIdx.x == 0) *cand_count = 0u;
    // chunk plans and the running-sum table in shared memory when they fit:
    // one memory latency for all plans instead of one per 32-chunk group;
    // then the segment tables and the predicted crossing segment of every
    // chunk the walk will fold (R < 0), so those folds start without a
    // memory round trip
    int* slot = nullptr;
    longlong2* pre_tab = nullptr;
    double* pre_seg = nullptr;
    int* pre_eb = nullptr;
    if (staged) {
        pre_tab = reinterpret_cast<longlong2*>(wdyn);
        pre_seg = reinterpret_cast<double*>(pre_tab + kMaxPre * 2 * kSegs);
        pre_eb = reinterpret_cast<int*>(pre_seg + kMaxPre * kSegLen);
        longlong2* Rs = reinterpret_cast<longlong2*>(pre_eb + kMaxPre * kSegs);
        double* ss = reinterpret_cast<double*>(Rs + nch);
        int* es = reinterpret_cast<int*>(ss + nch + 1);
        int* ps = es + nch;
        slot = ps + nch;
        unsigned* ms = reinterpret_cast<unsigned*>(slot + nch);
        // contiguous chunk ranges per thread, so slots follow chunk order
        const int per = (nch + kWalkThreads - 1) / kWalkThreads;
        const int c0 = min(nch, static_cast<int>(threadIdx.x) * per), c1 = min(nch, c0 + per);
        int nd = 0;
        for (int c = c0; c < c1; ++c) {
            const longlong2 r = R[c];
            Rs[c] = r;
            es[c] = ebin[c];
            ps[c] = spred[c];
            ms[c] = smask[c];
            nd += r.x < 0 && c > 0;
        }
        int incl = nd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wcount[warp] = incl;
        __syncthreads();
        int off = incl - nd;
        for (int w = 0; w < warp; ++w) off += wcount[w];
        for (int c = c0; c < c1; ++c) {
            int sl = -1;
            if (Rs[c].x < 0 && c > 0) {
                if (off < kMaxPre) {
                    sl = off;
                    pre_list[off] = c;
                }
                ++off;
            }
            slot[c] = sl;
        }
        __syncthreads();
        int ndirty = 0;
        for (int w = 0; w < kWalkThreads / 32; ++w) ndirty += wcount[w];
        ndirty = min(ndirty, kMaxPre);
        for (int e = threadIdx.x; e < ndirty * 2 * kSegs; e += kWalkThreads) {
            const int sl = e / (2 * kSegs), k = e % (2 * kSegs);
            pre_tab[e] = Rseg[static_cast<long long>(pre_list[sl]) * (2 * kSegs) + k];
        }
        for (int e = threadIdx.x; e < ndirty * kSegs; e += kWalkThreads) {
            const int sl = e / kSegs, k = e % kSegs;
            pre_eb[e] = Eseg[static_cast<long long>(pre_list[sl]) * kSegs + k];
        }
        for (int e = threadIdx.x; e < ndirty * kSegLen; e += kWalkThreads) {
            const int sl = e / kSegLen, k = e % kSegLen;
            const int c = pre_list[sl];
            const long long i = static_cast<long long>(c) * kFoldChunk + static_cast<long long>(ps[c]) * kSegLen + k;
            pre_seg[e] = i < N ? dist2[i] : 0.0;
        }
        __syncthreads();
        R = Rs;
        ebin = es;
        spred = ps;
        smask = ms;
        sstart = ss;
    }
    WALK_T(T1);
    if (threadIdx.x < 32) {
        // chunk 0 was folded literally by fold_round
        double S = *s0end;
        if (lane == 0) sstart[0] = 0.0;
        // kCPL x 32 chunks per step: a run of clean chunks in the running
        // sum's binade advances by one exact parity scan of their R_c; each
        // lane composes its kCPL chunks, then steps through them for their
        // exact starts (sstart) and the first chunk whose end leaves the
        // binade
        constexpr int kCPL = 4;
        for (int cb = 1; cb < nch; cb += 32 * kCPL) {
            ParInc rj[kCPL];
            int ej[kCPL];
#pragma unroll
            for (int j = 0; j < kCPL; ++j) {
                const int c = cb + kCPL * lane + j;
                const longlong2 r2 = c < nch ? R[c] : make_longlong2(-1, -1);
                rj[j] = ParInc{r2.x, r2.y};
                ej[j] = c < nch ? ebin[c] : 0;
            }
            const int cnt = min(32 * kCPL, nch - cb);
            int k = 0;
#pragma unroll 1
            while (k < cnt) {
                const bool normal = S >= kMinNormal && S < kPosInf;
                const int eS = normal ? dbl_exp(S) : -100001;
                const long long Si = normal ? dbl_sig(S) : 0;
                int lbad = 1 << 30;
#pragma unroll
                for (int j = 0; j < kCPL; ++j) {
                    const int idx = kCPL * lane + j;
                    const bool in = idx >= k && idx < cnt;
                    const bool ok = normal && ej[j] == eS && rj[j].i0 >= 0;
                    if (in && !ok && lbad == (1 << 30)) lbad = idx;
                }
                int fb = min(static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(lbad))), cnt);
                if (fb > k) {
                    ParInc f{0, 0};
#pragma unroll
                    for (int j = 0; j < kCPL; ++j) {
                        const int idx = kCPL * lane + j;
                        if (idx >= k && idx < fb) f = par_compose_ns(f, rj[j]);
                    }
                    const ParInc inc = par_scan_ns(f, lane);
                    const ParInc up = par_shfl_up(inc, 1);
                    long long cur = Si + (lane ? ((Si & 1) ? up.i1 : up.i0) : 0);
                    int lcross = 1 << 30;
#pragma unroll
                    for (int j = 0; j < kCPL; ++j) {
                        const int idx = kCPL * lane + j;
                        if (idx >= k && idx < fb && lcross == (1 << 30)) {
                            sstart[cb + idx] = dbl_make(cur, eS);
                            const long long nx = cur + ((cur & 1) ? rj[j].i1 : rj[j].i0);
                            if (nx >= kTwo53) lcross = idx;  // this chunk leaves the binade
                            else cur = nx;
                        }
                    }
                    // a chunk whose end leaves the binade is folded segment-wise
                    fb = min(fb, static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(lcross))));
                    if (fb > k) S = dbl_make(__shfl_sync(0xffffffffu, cur, (fb - 1) / kCPL), eS);
                }
                if (fb < cnt) {
                    const int c = cb + fb;
                    if (lane == 0) sstart[c] = S;
                    WALK_T(ta);
                    const int sl = slot ? slot[c] : -1;
                    S = sl >= 0 ? warp_fold_chunk(dist2, segbuf, N, c, spred[c], smask[c], pre_tab + sl * 2 * kSegs,
                                                  pre_eb + sl * kSegs, pre_seg + sl * kSegLen, S, false, 0.0).s
                                : warp_fold_chunk(dist2, segbuf, N, c, spred[c], smask[c],
                                                  Rseg + static_cast<long long>(c) * 2 * kSegs,
                                                  Eseg + static_cast<long long>(c) * kSegs, nullptr, S, false, 0.0).s;
                    WALK_T(tb);
                    WALK_ADD(c == 0 ? 8 : 2, tb - ta);
                    WALK_ADD(3, 1);
                    k = fb + 1;
                } else {
                    k = cnt;
                }
            }
        }
        if (lane == 0) {
            sstart[nch] = S;
            total = S;
        }
    }
    WALK_T(T2);
    __syncthreads();
    const double S = total;
    long long pick;
    if (S <= 0.0) {
        pick = N;  // all remaining points coincide with a centroid: first unused
        for (long long base = 0; base < N; base += 32) {
            bool free_ = base + lane < N && used[base + lane] == 0;
            unsigned m = __ballot_sync(0xffffffffu, free_);
            if (m) { pick = base + __ffs(m) - 1; break; }
        }
    } else {
        const int di = *draw_counter;
        const unsigned long long u = di < n_raw ? raw[di] : 0ull;
        // generate_canonical<double,53>(mt19937_64): double(u) / 2^64, clamped
        // below 1 (libstdc++ random.tcc); uniform_real(0,total) = c*total + 0.
        double c = __ull2double_rn(u) * 5.421010862427522e-20;  // exact: * 2^-64
        if (c >= 1.0) c = 0.99999999999999989;                 // nextafter(1, 0)
        const double target = xadd(xmul(c, xsub(S, 0.0)), 0.0);
        // first chunk whose running sum reaches the target (the sum is
        // monotone): every thread tests its chunks, block-wide minimum
        if (threadIdx.x == 0) flag_min = nch;
        __syncthreads();
        for (int cc = threadIdx.x; cc < nch; cc += kWalkThreads)
            if (sstart[cc + 1] >= target) {
                atomicMin(&flag_min, cc);
                break;
            }
        __syncthreads();
        const int cstar = flag_min;
        pick = -1;
        if (threadIdx.x < 32) {
            // the running sum reaches the target inside chunk cstar (an element
            // that raises it is > 0); later chunks only as a guard
            double sc = cstar < nch ? sstart[cstar] : 0.0;
            for (int cc = cstar; cc < nch && pick < 0; ++cc) {
                const SegFold sr = warp_fold_chunk(dist2, segbuf, N, cc, 0, 0u, Rseg + static_cast<long long>(cc) * 2 * kSegs,
                                                   Eseg + static_cast<long long>(cc) * kSegs, nullptr, sc, true, target);
                pick = sr.pick;
                sc = sr.s;
            }
            if (pick < 0) pick = N - 1;
        }
        if (threadIdx.x == 0) *draw_counter = di + 1;
    }
    if (threadIdx.x == 0) {
        WALK_T(T3);
        WALK_ADD(0, T1 - T0);
        WALK_ADD(1, T2 - T1);
        WALK_ADD(4, T3 - T2);
        WALK_ADD(5, 1);
        chosen[t] = static_cast<uint32_t>(pick);
        if (pick < N) {
            dist2[pick] = 0.0;
            used[pick] = 1;
        }
    }
}

// ---- certified pick (kmeans.cpp:49-58) without the exact fold ---------------
// The running sum of the reference is only consumed through two comparisons:
// target = c * total (uniform_real(0, total)) and the first i with
// acc_i >= target. So the pick is decided by any approximation Q_i of the
// prefix sums whose distance to the fold acc_i is bounded by a known W:
//   * the fold over non-negative values: |acc_i - P_i| <= gamma_N T
//     (P the real prefix, gamma_k = k u / (1 - k u), u = 2^-53);
//   * Q from the chunk sums csum: the prune pass writes each chunk's sum as a
//     tree (height <= 16, also kept in bsum), the exact pass adds each
//     update's fl(new - old) atomically: at most 2048 adds per chunk, each
//     rounding within u of the chunk's pre-update sum, so the chunk sum is
//     within (2 * 2048 + 20) u bsum_c of the real one; the scans here add
//     a tree of height < 64 + nch / 1024.
// Hence |acc_i - Q_i| <= W = 2 (N + nch + 128) u T + 8400 u sum(bsum)
// (twice the bounds), the reference's target lies in c T +- (W + slop), and
// an index i with
//   Q_i - W' >= mid + W'   and   Q_{i-1} + W' < mid - W'
// (W' = W + 16 u T covers the fl products and differences here) IS the
// reference's pick: acc is monotone, and acc_{i-1} < target <= acc_i forces
// dist2[i] > 0 (the second half of kmeans.cpp:53). Such an i exists unless
// the target falls within ~4 W of a prefix boundary (probability ~4 N W / T,
// ~3e-3 per step at N = 2e6); those steps, the total <= 0 branch and
// non-finite sums set skip = 0 and the exact fold + walk run as before.
// One CTA: scan of the chunk sums, target chunk, that chunk's 2048 values.
constexpr int kPickThreads = 1024;
__global__ void __launch_bounds__(kPickThreads) pp_pick_kernel(
    double* __restrict__ dist2, unsigned char* __restrict__ used, long long N, int nch,
    double* __restrict__ csum, double* __restrict__ bsum, double* __restrict__ qbuf,
    int* __restrict__ skip, unsigned* __restrict__ cand_count, const unsigned long long* __restrict__ raw, int n_raw,
    int* __restrict__ draw_counter, uint32_t* __restrict__ chosen, int t, unsigned* __restrict__ n_fallback,
    double slack, const unsigned* __restrict__ surv_count, unsigned long long* __restrict__ stats, int qsmem,
    PPB pb) {
    pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.y;
    if (t >= pb.k[y]) return;
    dist2 += y * pb.sN;
    used += y * pb.sN;
    csum += y * pb.sC;
    bsum += y * pb.sC;
    qbuf += y * pb.sC;
    skip += y;
    cand_count += y;
    raw += y * pb.sK;
    n_raw = pb.k[y] - 1;
    draw_counter += y;
    chosen += y * pb.sK;
    n_fallback += y;
    if (surv_count) surv_count += y;
    if (stats) stats += 2 * y;
    if (stats && threadIdx.x == 0) {  // candidates and exact folds of this step (LCN_TIMING)
        stats[0] += *cand_count;
        stats[1] += surv_count ? *surv_count : 0u;
    }
    __shared__ double red[kPickThreads / 32], bred[kPickThreads / 32];
    __shared__ double carry_s, bs_s;
    extern __shared__ __align__(16) unsigned char pdyn[];
    if (qsmem) qbuf = reinterpret_cast<double*>(pdyn);  // the chunk prefix sums stay on chip
    __shared__ int cstar_s, istar_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr double u = 1.1102230246251565e-16;  // 2^-53
    if (threadIdx.x == 0) {
        carry_s = 0.0;
        bs_s = 0.0;
        cstar_s = nch;
        istar_s = kFoldChunk;
    }
    __syncthreads();
    // inclusive scan of the chunk sums (qbuf[c] = Q at the end of chunk c)
    // and the sum of the pre-update sums
    for (int c0 = 0; c0 < nch; c0 += kPickThreads) {
        const int c = c0 + threadIdx.x;
        const double v = c < nch ? csum[c] : 0.0;
        const double bv = warp_sum(c < nch ? bsum[c] : 0.0);
        double incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double tt = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += tt;
        }
        if (lane == 31) red[warp] = incl;
        if (lane == 0) bred[warp] = bv;
        __syncthreads();
        double off = carry_s;
        for (int w = 0; w < warp; ++w) off += red[w];
        if (c < nch) qbuf[c] = off + incl;
        __syncthreads();
        if (threadIdx.x == kPickThreads - 1) carry_s = off + incl;
        if (threadIdx.x == 0) {
            double bb = bs_s;
            for (int w = 0; w < kPickThreads / 32; ++w) bb += bred[w];
            bs_s = bb;
        }
        __syncthreads();
    }
    const double T = carry_s, BS = bs_s;
    const int di = *draw_counter;
    const double W = (2.0 * static_cast<double>(N + nch + 128) * u * T + 8400.0 * u * BS) * slack + 16.0 * u * T;
    if (!(T > 0.0) || !(T < kPosInf) || !(BS < kPosInf) || di >= n_raw || !(W < 1e-3 * T)) {
        if (threadIdx.x == 0) {
            *skip = 0;
            atomicAdd(n_fallback, 1u);
        }
        return;
    }
    double c = __ull2double_rn(raw[di]) * 5.421010862427522e-20;  // as pp_walk_pick_kernel
    if (c >= 1.0) c = 0.99999999999999989;
    const double mid = c * T, tlo = mid - W, thi = mid + W;
    for (int cc = threadIdx.x; cc < nch; cc += kPickThreads)
        if (qbuf[cc] >= mid) {
            atomicMin(&cstar_s, cc);
            break;
        }
    __syncthreads();
    const int cs = min(cstar_s, nch - 1);
    const double A = cs > 0 ? qbuf[cs - 1] : 0.0;
    // the chunk's prefix: kPer contiguous values per thread, then warp / block
    constexpr int kPer = kFoldChunk / kPickThreads;
    const long long b = static_cast<long long>(cs) * kFoldChunk + threadIdx.x * kPer;
    double xv[kPer];
    double run = 0.0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        xv[j] = b + j < N ? dist2[b + j] : 0.0;
        run += xv[j];
    }
    double incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double tt = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += tt;
    }
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    // exclusive prefix by a shuffle (a summation tree, unlike incl - run)
    double q = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) q = 0.0;
    for (int w = 0; w < warp; ++w) q += red[w];
    q += A;  // Q just before this thread's first value
    double qprev = q;
    int hit = -1;
    double qhit = 0.0, qhprev = 0.0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const double qn = qprev + xv[j];
        if (hit < 0 && b + j < N && qn >= mid) {
            hit = threadIdx.x * kPer + j;
            qhit = qn;
            qhprev = qprev;
        }
        qprev = qn;
    }
    if (hit >= 0) atomicMin(&istar_s, hit);
    __syncthreads();
    if (hit >= 0 && hit == istar_s) {
        const long long pick = static_cast<long long>(cs) * kFoldChunk + hit;
        const bool ok = tlo > 0.0 && qhit - W >= thi && qhprev + W < tlo;
        if (ok) {
            chosen[t] = static_cast<uint32_t>(pick);
            dist2[pick] = 0.0;
            used[pick] = 1;
            *draw_counter = di + 1;
            *cand_count = 0u;
        } else {
            atomicAdd(n_fallback, 1u);
        }
        *skip = ok ? 1 : 0;
    } else if (threadIdx.x == 0 && istar_s == kFoldChunk) {
        *skip = 0;  // not in the predicted chunk: the exact walk decides
        atomicAdd(n_fallback, 1u);
    }
}

__global__ void fill_kernel(double* p, long long n, double v) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) p[i] = v;
}

template <typename T>
void kmeans_pp_batch(Ctx& ctx, const T* X, long long N, int d, const std::vector<PPSeq>& seqs) {
    cudaStream_t s = ctx.stream;
    const int S = static_cast<int>(seqs.size());
    if (S < 1) return;
    if (S > kMaxSeq) {  // in groups of kMaxSeq
        for (int g = 0; g < S; g += kMaxSeq)
            kmeans_pp_batch<T>(ctx, X, N, d,
                               std::vector<PPSeq>(seqs.begin() + g, seqs.begin() + std::min(S, g + kMaxSeq)));
        return;
    }
    int KM = 1;
    for (const auto& q : seqs) KM = std::max(KM, q.k);
    const int nch = ceil_div(N, kFoldChunk);
    PPB pb{};
    pb.sN = N;
    pb.sC = nch;
    pb.sK = KM;
    for (int y = 0; y < kMaxSeq; ++y) pb.k[y] = y < S ? seqs[y].k : 0;
    const size_t SN = static_cast<size_t>(S) * N, SC = static_cast<size_t>(S) * nch, SK = static_cast<size_t>(S) * KM;
    DevBuf<double> dist2(SN), csum(SC), bsum(SC), qbuf(SC), sstart(static_cast<size_t>(S) * (nch + 1));
    DevBuf<int> ebin(SC), spred(SC), Eseg(SC * kSegs);
    DevBuf<unsigned> smask(SC);
    DevBuf<double> s0end(S);
    DevBuf<longlong2> R(SC), Rseg(SC * 2 * kSegs);
    DevBuf<unsigned char> used(SN);
    // walk: chunk plans + running-sum table staged in shared memory if they fit
    size_t walk_smem = static_cast<size_t>(nch) * (sizeof(longlong2) + sizeof(double) + 4 * sizeof(int)) + sizeof(double) +
                       static_cast<size_t>(kMaxPre) * (2 * kSegs * sizeof(longlong2) + kSegLen * sizeof(double) +
                                                       kSegs * sizeof(int));
    // staged walk (its plans in 200 KB of shared memory) only on request:
    // with the certified pick the walk runs on ~0.4 % of the steps, and a
    // launch that needs a whole SM's shared memory just to exit costs more
    // (LCN_PP_WALK_STAGED=1, or always without the certified pick)
    const char* wsenv = std::getenv("LCN_PP_WALK_STAGED");
    const char* wenv0 = std::getenv("LCN_PP_EXACT_WALK");
    const bool want_staged = (wsenv && wsenv[0] == '1') || (wenv0 && wenv0[0] == '1');
    int walk_staged = want_staged && walk_smem <= 200 * 1024;
    if (walk_staged)
        allow_max_dyn_smem(pp_walk_pick_kernel);
    else
        walk_smem = 0;
    DevBuf<uint32_t> near(SN), list(SN), chosen(SK);
    DevBuf<unsigned> cnt(S);
    DevBuf<double> dc(SK);
    // exact-pass geometry: warps per CTA so one CTA's row buffers stay <= 96 KB
    int ex_warps = 4;
    while (ex_warps > 1 && static_cast<size_t>(ex_warps) * 32 * (d + 1) * sizeof(T) > 96 * 1024) ex_warps >>= 1;
    const size_t ex_smem = static_cast<size_t>(d) * 8 + static_cast<size_t>(ex_warps) * 32 * (d + 1) * sizeof(T);
    if (ex_smem > 200 * 1024) throw Status(2, "k-means++: dimension too large for the exact seeding pass");
    allow_max_dyn_smem(pp_exact_kernel<T>);
    int ex_occ = 1;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ex_occ, pp_exact_kernel<T>, ex_warps * 32, ex_smem));
    // one CTA per SM and sequence: a step has a few thousand survivors (early
    // steps loop); more CTAs only cost launch and smem reconfiguration
    const int ex_grid = ctx.num_sms;
    (void)ex_occ;
    // filter copy of the points (shared by the sequences): int8 rows with a
    // power-of-two scale per row (default: the integer filter) or fp16 rows
    // (LCN_PP_FILTER=f16: tighter bound, twice the bytes); rows up to 512
    // values, else (or LCN_PP_NOFILTER) every candidate is folded exactly
    const char* fenv = std::getenv("LCN_PP_FILTER");
    const bool i8 = !(fenv && std::string(fenv) == "f16");
    const int qsz = i8 ? 1 : 2;
    const int dp = i8 ? (d + 15) / 16 * 16 : (d + 7) / 8 * 8;
    const bool filt = dp <= kFiltMaxQ * 128 && std::getenv("LCN_PP_NOFILTER") == nullptr;
    DevBuf<unsigned char> Xq(filt ? static_cast<size_t>(N) * dp * qsz : 1);
    DevBuf<float2> se(filt ? static_cast<size_t>(N) : 1);
    DevBuf<int> qn(filt && i8 ? static_cast<size_t>(N) : 1);
    const int nq = (dp / 4 + 31) / 32;
    using FsH = void (*)(const T*, const __half*, const float2*, int, int, const uint32_t*, int, const double*,
                         const uint32_t*, const unsigned*, uint32_t*, unsigned*, PPB);
    const FsH fs_h = nq == 1 ? pp_filter_kernel<T, __half, 1>
                   : nq == 2 ? pp_filter_kernel<T, __half, 2>
                   : nq == 3 ? pp_filter_kernel<T, __half, 3>
                             : pp_filter_kernel<T, __half, 4>;
    using FiQ = void (*)(const T*, const int8_t*, const float2*, const int*, int, int, const uint32_t*, int,
                         const double*, const uint32_t*, const unsigned*, uint32_t*, unsigned*, PPB);
    const FiQ fi_q = nq == 1 ? pp_filter_i8_kernel<T, 1>
                   : nq == 2 ? pp_filter_i8_kernel<T, 2>
                   : nq == 3 ? pp_filter_i8_kernel<T, 3>
                             : pp_filter_i8_kernel<T, 4>;
    int f_grid = ctx.num_sms;
    if (filt) {
        int occ = 1;
        if (i8)
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fi_q, 128, 0));
        else
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fs_h, 128, 0));
        f_grid = std::max(1, occ) * ctx.num_sms;
        if (i8)
            pp_i8_prep_kernel<T><<<ceil_div(N, 8), 256, 0, s>>>(X, N, d, dp, reinterpret_cast<int8_t*>(Xq.get()),
                                                               se.get(), qn.get());
        else
            pp_half_prep_kernel<T><<<ceil_div(N, 8), 256, 0, s>>>(X, N, d, dp, reinterpret_cast<__half*>(Xq.get()),
                                                                 se.get());
        LAUNCH_OK("kmeans++ filter copy");
    }
    DevBuf<uint32_t> surv(filt ? SN : 1);
    DevBuf<unsigned> scnt(S);
    // the callers' engine draws, one row of KM per sequence
    std::vector<unsigned long long> hraw(SK, 0ull);
    for (int y = 0; y < S; ++y)
        std::copy(seqs[y].raw.begin(), seqs[y].raw.begin() + std::min<size_t>(seqs[y].raw.size(), KM), hraw.begin() + y * KM);
    DevBuf<unsigned long long> d_raw(SK);
    d_raw.upload(hraw.data(), SK, s);
    DevBuf<int> counter(S);
    // certified pick first (pp_pick_kernel); the exact fold + walk only
    // when it cannot decide. LCN_PP_EXACT_WALK=1 always runs the exact walk.
    const char* wenv = std::getenv("LCN_PP_EXACT_WALK");
    const bool fast = !(wenv && wenv[0] == '1');
    const char* senv = std::getenv("LCN_PP_CERT_SLACK");  // test hook: widen the certificate (more fallbacks)
    const double slack = senv ? std::max(1.0, std::atof(senv)) : 1.0;
    const size_t pk_smem = static_cast<size_t>(nch) * 8 <= 160 * 1024 ? static_cast<size_t>(nch) * 8 : 0;
    if (pk_smem > 48 * 1024) allow_max_dyn_smem(pp_pick_kernel);
    DevBuf<int> skip(S);
    DevBuf<unsigned> nfall(S);
    const bool timing = std::getenv("LCN_TIMING") != nullptr;
    DevBuf<unsigned long long> pstats(2 * S);
    pstats.zero(s);
    skip.zero(s);
    nfall.zero(s);
    used.zero(s);
    near.zero(s);
    counter.zero(s);
    csum.zero(s);
    cnt.zero(s);
    scnt.zero(s);
    fill_kernel<<<ceil_div(static_cast<long long>(SN), 256), 256, 0, s>>>(dist2.get(), static_cast<long long>(SN),
                                                                          kPosInf);
    {
        std::vector<uint32_t> h0(SK, 0u);
        for (int y = 0; y < S; ++y) h0[static_cast<size_t>(y) * KM] = static_cast<uint32_t>(seqs[y].first);
        chosen.upload(h0.data(), SK, s);
        const unsigned char one = 1;
        for (int y = 0; y < S; ++y)
            CUDA_OK(cudaMemcpyAsync(used.get() + static_cast<size_t>(y) * N + seqs[y].first, &one, 1,
                                    cudaMemcpyHostToDevice, s));
        ctx.sync();  // the host staging above goes out of scope
    }
    // the step chain with programmatic dependent launches (LCN_PP_PDL=0: plain)
    const char* penv = std::getenv("LCN_PP_PDL");
    const bool pdl = !(penv && penv[0] == '0');
    const dim3 b256(256), b128(128);
    const unsigned Sy = static_cast<unsigned>(S);
    const int fr_grid = std::min(nch, 4 * ctx.num_sms);
    for (int t = 1; t < KM; ++t) {
        if (t > 1)
            launch_pdl(seed_dist_kernel<T>, dim3(ceil_div(t - 1, 8), Sy), b256, 0, s, pdl, X, d, chosen.get(), t - 1,
                       dc.get(), scnt.get(), pb);
        launch_pdl(pp_prune_kernel, dim3(nch, Sy), dim3(kPruneThreads), 0, s, pdl, N, t - 1, dist2.get(), near.get(), dc.get(),
                   list.get(), cnt.get(), csum.get(), scnt.get(), bsum.get(), pb);
        if (filt) {
            if (i8)
                launch_pdl(fi_q, dim3(f_grid, Sy), b128, 0, s, pdl, X, reinterpret_cast<const int8_t*>(Xq.get()),
                           se.get(), qn.get(), d, dp, chosen.get(), t - 1, dist2.get(), list.get(), cnt.get(),
                           surv.get(), scnt.get(), pb);
            else
                launch_pdl(fs_h, dim3(f_grid, Sy), b128, 0, s, pdl, X, reinterpret_cast<const __half*>(Xq.get()),
                           se.get(), d, dp, chosen.get(), t - 1, dist2.get(), list.get(), cnt.get(), surv.get(),
                           scnt.get(), pb);
            launch_pdl(pp_exact_kernel<T>, dim3(ex_grid, Sy), dim3(ex_warps * 32), ex_smem, s, pdl, X, d, chosen.get(),
                       t - 1, dist2.get(), near.get(), surv.get(), scnt.get(), csum.get(), 11, pb);
        } else {
            launch_pdl(pp_exact_kernel<T>, dim3(ex_grid, Sy), dim3(ex_warps * 32), ex_smem, s, pdl, X, d, chosen.get(),
                       t - 1, dist2.get(), near.get(), list.get(), cnt.get(), csum.get(), 11, pb);
        }
        // the first pass moves every point off +inf: its chunk sums are taken
        // afresh (later steps: pre-update sums corrected by the exact pass)
        if (t == 1)
            launch_pdl(fold_chunk_sum_kernel, dim3(nch, Sy), b256, 0, s, pdl, dist2.get(), N, csum.get(), bsum.get(),
                       t, pb);
        const int* skp = nullptr;
        if (fast) {
            launch_pdl(pp_pick_kernel, dim3(1, Sy), dim3(kPickThreads), pk_smem, s, pdl, dist2.get(), used.get(), N,
                       nch, csum.get(), bsum.get(), qbuf.get(), skip.get(), cnt.get(), d_raw.get(), KM - 1,
                       counter.get(), chosen.get(), t, nfall.get(), slack, filt ? scnt.get() : nullptr,
                       timing ? pstats.get() : nullptr, pk_smem ? 1 : 0, pb);
            skp = skip.get();
        }
        launch_pdl(fold_round_kernel, dim3(fr_grid, Sy), b256, 0, s, pdl, dist2.get(), N, csum.get(), ebin.get(),
                   R.get(), Rseg.get(), Eseg.get(), spred.get(), smask.get(), s0end.get(), skp, t, pb, nch);
        launch_pdl(pp_walk_pick_kernel, dim3(1, Sy), dim3(kWalkThreads), walk_smem, s, pdl, dist2.get(), used.get(), N,
                   nch, ebin.get(), spred.get(), R.get(), Rseg.get(), Eseg.get(), smask.get(), s0end.get(), csum.get(),
                   cnt.get(), sstart.get(), d_raw.get(), KM - 1, counter.get(), chosen.get(), t, walk_staged, skp, pb);
    }
    LAUNCH_OK("kmeans++");
    for (int y = 0; y < S; ++y)
        CUDA_OK(cudaMemcpyAsync(seqs[y].d_chosen, chosen.get() + static_cast<size_t>(y) * KM,
                                static_cast<size_t>(seqs[y].k) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    std::vector<int> h_cnt(S, 0);
    counter.download(h_cnt.data(), S, s);
    std::vector<unsigned> h_fall(S, 0);
    std::vector<unsigned long long> h_st(2 * S, 0);
    if (fast && timing) {
        nfall.download(h_fall.data(), S, s);
        pstats.download(h_st.data(), 2 * S, s);
    }
    ctx.sync();
    for (int y = 0; y < S; ++y) {
        if (seqs[y].draws_used) *seqs[y].draws_used = h_cnt[y];
        const int k = seqs[y].k;
        if (fast && timing && k > 1)
            std::fprintf(stderr,
                         "[kmeans++] N=%lld k=%d (sequence %d of %d): exact-walk fallbacks %u of %d steps; per step "
                         "%.0f filter candidates, %.0f exact folds (%s rows)\n",
                         N, k, y, S, h_fall[y], k - 1, static_cast<double>(h_st[2 * y]) / (k - 1),
                         static_cast<double>(h_st[2 * y + 1]) / (k - 1), filt ? (i8 ? "int8" : "fp16") : "no filter");
    }
#ifdef LCN_WALK_PROFILE
    if (std::getenv("LCN_WALK_STATS")) {
        unsigned long long h[16];
        CUDA_OK(cudaMemcpyFromSymbol(h, g_wt, sizeof(h)));
        const double n = h[5] ? static_cast<double>(h[5]) : 1.0;
        std::fprintf(stderr,
                     "[walk] cycles per launch: stage %.0f level1 %.0f (chunk0 %.0f, other chunks %.0f in %.1f calls; "
                     "segment folds %.0f in %.1f) search+pick %.0f\n",
                     h[0] / n, h[1] / n, h[8] / n, h[2] / n, h[3] / n, h[6] / n, h[7] / n, h[4] / n);
        CUDA_OK(cudaMemset(g_wt_ptr(), 0, sizeof(h)));
    }
#endif
}

template <typename T>
void kmeans_pp_device(Ctx& ctx, const T* X, long long N, int d, int k, uint64_t first,
                      const std::vector<unsigned long long>& raw, uint32_t* d_chosen, int* draws_used) {
    kmeans_pp_batch<T>(ctx, X, N, d, {PPSeq{k, first, raw, d_chosen, draws_used}});
}

// ---- Lloyd (kmeans.cpp:87-143) ---------------------------------------------
__global__ void count_changes_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, long long N,
                                     unsigned long long* __restrict__ changes) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < N; i += 256LL * gridDim.x) c += a[i] != b[i];
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(changes, c);
}
__global__ void count_kernel(const uint32_t* __restrict__ assign, long long N, int* __restrict__ counts) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < N) atomicAdd(&counts[assign[i]], 1);
}

__global__ void iota_kernel(uint32_t* p, long long n) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) p[i] = static_cast<uint32_t>(i);
}

// One CTA per cluster: per-dimension fold over the members in increasing
// point index (kmeans.cpp:106-114), then ctr = sum * (1/count).
template <typename T>
__global__ void centroid_kernel(const T* __restrict__ X, int d, const uint32_t* __restrict__ order,
                                const int* __restrict__ start, const int* __restrict__ counts,
                                double* __restrict__ ctr) {
    const int c = blockIdx.x;
    const int cnt = counts[c];
    if (cnt == 0) return;
    const int b = start[c];
    const double inv = __ddiv_rn(1.0, static_cast<double>(cnt));
    for (int kk = threadIdx.x; kk < d; kk += blockDim.x) {
        double s = 0.0;
        int p = 0;
        // 16 member rows loaded ahead of the (sequential) fold
        for (; p + 16 <= cnt; p += 16) {
            T v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = X[static_cast<long long>(order[b + p + u]) * d + kk];
#pragma unroll
            for (int u = 0; u < 16; ++u) s = xadd(s, static_cast<double>(v[u]));
        }
        for (; p < cnt; ++p) s = xadd(s, static_cast<double>(X[static_cast<long long>(order[b + p]) * d + kk]));
        ctr[static_cast<long long>(c) * d + kk] = xmul(s, inv);
    }
}

// Farthest point among clusters with count > 1 (kmeans.cpp:125-134): block
// partial argmax (value, lowest index).
template <typename T>
__global__ void farthest_partial_kernel(const T* __restrict__ X, long long N, int d, const double* __restrict__ ctr,
                                        const uint32_t* __restrict__ assign, const int* __restrict__ counts,
                                        double* __restrict__ pval, long long* __restrict__ pidx) {
    __shared__ double sv[256];
    __shared__ long long si[256];
    double best = -1.0;
    long long arg = -1;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < N; i += 256LL * gridDim.x) {
        uint32_t c = assign[i];
        if (counts[c] <= 1) continue;
        double d2 = sqdist_exact(X + i * d, ctr + static_cast<long long>(c) * d, d);
        if (d2 > best) { best = d2; arg = i; }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = arg;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            double ov = sv[threadIdx.x + o];
            long long oi = si[threadIdx.x + o];
            if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi >= 0 && (si[threadIdx.x] < 0 || oi < si[threadIdx.x]))) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pval[blockIdx.x] = sv[0];
        pidx[blockIdx.x] = si[0];
    }
}

template <typename T>
__global__ void reseed_apply_kernel(const T* __restrict__ X, int d, const double* __restrict__ pval,
                                    const long long* __restrict__ pidx, int nparts, double* __restrict__ ctr,
                                    uint32_t* __restrict__ assign, int* __restrict__ counts, int c,
                                    float* __restrict__ lb = nullptr) {
    __shared__ long long s_arg;
    if (threadIdx.x == 0) {
        double far = -1.0;
        long long arg = -1;
        for (int b = 0; b < nparts; ++b) {  // blocks cover increasing index ranges interleaved: keep lowest index
            if (pidx[b] < 0) continue;
            if (pval[b] > far || (pval[b] == far && pidx[b] < arg)) { far = pval[b]; arg = pidx[b]; }
        }
        if (arg < 0) arg = 0;  // far stays -1 -> arg = 0 (kmeans.cpp:126)
        s_arg = arg;
        counts[assign[arg]] -= 1;
        assign[arg] = static_cast<uint32_t>(c);
        counts[c] = 1;
        if (lb) lb[arg] = 0.0f;  // its bound was for another assignment: re-evaluate
    }
    __syncthreads();
    const long long arg = s_arg;
    for (int kk = threadIdx.x; kk < d; kk += blockDim.x) ctr[static_cast<long long>(c) * d + kk] = static_cast<double>(X[arg * d + kk]);
}


// ---- fast assignment: fp32 filter + exact fallback -------------------------
// For fp32 points with d <= kFD the argmin is first located with fp32 FMA
// tiles: v(c) = |c_f|^2 - 2 x.c_f (c_f = fp32(c)), so that the exact fold
// D(c) = |x|^2 + v(c) + err(c) with |err(c)| <= E(x) for every centroid
// (rigorous bound below). If the best and second-best v differ by more than
// 2 E(x), the best centroid is the exact argmin (no other centroid can tie or
// win); otherwise the point goes to the ambiguous list and gets the full
// exact fp64 scan with lowest-index ties. Results are identical to the exact
// kernel; the filter only skips work that cannot change them.
constexpr int kFB = 128;  // points per CTA = centroids per tile
constexpr int kFD = 128;  // max dimension of the filter path

struct FilterSmem {
    float A[kFD][kFB];     // point tile, feature-major
    float B[2][kFD][kFB];  // centroid tiles (double-buffered), feature-major
    float nc[2][kFB];      // |c_f|^2 rounded to fp32 (+inf for padding)
    double xn[kFB];        // |x|^2 (fp64)
};


// CfT[kk][c] = fp32(C[c][kk]) for c < k, 0 for padding; ncf[c] = fp32(sum c_f^2)
// (+inf for padding); cmax = max_c max(|c|^2, |c_f|^2) as fp64 bits.
__global__ void __launch_bounds__(128) filter_prep_kernel(const double* __restrict__ C, int k, int d, int Kp,
                                                          float* __restrict__ CfT, float* __restrict__ ncf,
                                                          unsigned long long* __restrict__ cmax) {
    __shared__ double r1[4], r2[4];
    const int c = blockIdx.x;
    double s1 = 0.0, s2 = 0.0;
    for (int kk = threadIdx.x; kk < d; kk += 128) {
        const double v = c < k ? C[static_cast<long long>(c) * d + kk] : 0.0;
        const float f = static_cast<float>(v);
        CfT[static_cast<long long>(kk) * Kp + c] = f;
        s1 += static_cast<double>(f) * static_cast<double>(f);
        s2 += v * v;
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = s1; r2[threadIdx.x >> 5] = s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        s1 = r1[0] + r1[1] + r1[2] + r1[3];
        s2 = r2[0] + r2[1] + r2[2] + r2[3];
        ncf[c] = c < k ? static_cast<float>(s1) : kPosInf;
        if (c < k) atomicMax(cmax, static_cast<unsigned long long>(__double_as_longlong(fmax(s1, s2))));
    }
}

__global__ void __launch_bounds__(256, 1) assign_filter_kernel(const float* __restrict__ X, long long N, int d,
                                                               const float* __restrict__ CfT, const float* __restrict__ ncf,
                                                               int Kp, const unsigned long long* __restrict__ cmax,
                                                               uint32_t* __restrict__ out, uint32_t* __restrict__ amb,
                                                               unsigned* __restrict__ namb) {
    extern __shared__ __align__(16) unsigned char dyn[];
    FilterSmem& sm = *reinterpret_cast<FilterSmem*>(dyn);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long p0 = static_cast<long long>(blockIdx.x) * kFB;
    const int ntile = Kp / kFB;
    auto load_b = [&](int buf, int c0) {
        for (int e = tid; e < d * (kFB / 4); e += 256) {
            const int kk = e / (kFB / 4), ch = e % (kFB / 4);
            cp_async16(&sm.B[buf][kk][ch * 4], CfT + static_cast<long long>(kk) * Kp + c0 + ch * 4);
        }
        if (tid < kFB / 4) cp_async16(&sm.nc[buf][tid * 4], ncf + c0 + tid * 4);
        cp_async_commit();
    };
    load_b(0, 0);
    // point tile, transposed to feature-major (a one-time load per CTA)
    for (int e = tid; e < kFB * d; e += 256) {
        const int pp = e % kFB, kk = e / kFB;
        const long long p = p0 + pp;
        sm.A[kk][pp] = p < N ? X[p * d + kk] : 0.0f;
    }
    __syncthreads();
    if (tid < kFB) {
        double sx = 0.0;
        for (int kk = 0; kk < d; ++kk) sx += static_cast<double>(sm.A[kk][tid]) * static_cast<double>(sm.A[kk][tid]);
        sm.xn[tid] = sx;
    }
    float v1[8], v2[8];
    int i1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { v1[i] = kPosInf; v2[i] = kPosInf; i1[i] = 0; }
    for (int t = 0; t < ntile; ++t) {
        const int buf = t & 1;
        if (t + 1 < ntile) {
            load_b(buf ^ 1, (t + 1) * kFB);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
        const float* Bb = &sm.B[buf][0][0];
#pragma unroll 4
        for (int kk = 0; kk < d; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&sm.A[kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&sm.A[kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(Bb + kk * kFB + tx * 4);
            const float4 b1 = *reinterpret_cast<const float4*>(Bb + kk * kFB + 64 + tx * 4);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int cl = j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4);
            const float nc = sm.nc[buf][cl];
            const int c = t * kFB + cl;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float v = fmaf(-2.0f, acc[i][j], nc);  // one rounding of |c_f|^2 - 2 x.c_f
                if (v < v1[i]) { v2[i] = v1[i]; v1[i] = v; i1[i] = c; }
                else if (v < v2[i]) v2[i] = v;
            }
        }
        __syncthreads();  // buffer `buf` is refilled by the next iteration's load
    }
    // merge the 16 column threads of each point (half-warp): best, index, second
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const float ov1 = __shfl_xor_sync(0xffffffffu, v1[i], o);
            const float ov2 = __shfl_xor_sync(0xffffffffu, v2[i], o);
            const int oi = __shfl_xor_sync(0xffffffffu, i1[i], o);
            if (ov1 < v1[i] || (ov1 == v1[i] && oi < i1[i])) {
                v2[i] = fminf(v1[i], ov2);
                v1[i] = ov1;
                i1[i] = oi;
            } else {
                v2[i] = fminf(ov1, v2[i]);
            }
        }
    }
    if (tx == 0) {
        const double u = 5.9604644775390625e-08;  // 2^-24
        const double g = d * u / (1.0 - d * u);    // gamma_d of the fp32 FMA dot
        const double C = sqrt(__longlong_as_double(*cmax)) * (1.0 + 1e-12);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int pp = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
            const long long p = p0 + pp;
            if (p >= N) continue;
            const double x = sqrt(sm.xn[pp]) * (1.0 + 1e-12);
            // c -> c_f (2u(x+C)C + u^2 C^2), |c_f|^2 -> fp32 (u C^2), dot (2 g x C),
            // final rounding (u (C^2 + 2 x C)), fp64 fold of D (<= 1e-13 (x+C)^2)
            const double E = 1.05 * ((2.0 * g + 4.0 * u) * x * C + 4.0 * u * C * C + u * u * C * C) +
                             1e-12 * (x + C) * (x + C);
            const double gap = static_cast<double>(v2[i]) - static_cast<double>(v1[i]);
            if (gap > 2.0 * E) out[p] = static_cast<uint32_t>(i1[i]);
            else amb[atomicAdd(namb, 1u)] = static_cast<uint32_t>(p);
        }
    }
}

cublasHandle_t cublas_of(Ctx& ctx);  // build.cu

// fp32 filter for d > 128 (configs[1] / [2]: d = 300), where neither the
// tensor-core filter (points in TMEM, d <= 128) nor the FMA register tiles
// (d <= 128 in shared memory) apply: the dots x.c_f for a chunk of points
// come from one fp32 GEMM (cuBLAS, CUBLAS_COMPUTE_32F_PEDANTIC: no TF32,
// whatever the environment says), a warp per point then keeps the best and
// second-best score v(c) = |c_f|^2 - 2 x.c_f and applies the same rigorous
// gap test as assign_filter_kernel, with gamma_{d+8} for a dot summed in
// any order (split-K included). Ambiguous points get the exact scan.
__global__ void __launch_bounds__(256) gemm_top2_kernel(const float* __restrict__ X, long long p0, long long np,
                                                        int d, const float* __restrict__ S, int Kp, int k,
                                                        const float* __restrict__ ncf,
                                                        const unsigned long long* __restrict__ cmax,
                                                        uint32_t* __restrict__ out, uint32_t* __restrict__ amb,
                                                        unsigned* __restrict__ namb) {
    const int lane = threadIdx.x & 31;
    const long long i = blockIdx.x * 8LL + (threadIdx.x >> 5);
    if (i >= np) return;
    const long long p = p0 + i;
    const float* sc = S + i * Kp;
    float v1 = kPosInf, v2 = kPosInf;
    int i1 = 0;
    for (int c = lane; c < k; c += 32) {
        const float v = fmaf(-2.0f, sc[c], ncf[c]);  // one rounding of |c_f|^2 - 2 x.c_f
        if (v < v1) { v2 = v1; v1 = v; i1 = c; }
        else if (v < v2) v2 = v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ov1 = __shfl_xor_sync(0xffffffffu, v1, o), ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i1, o);
        v2 = fminf(fminf(v2, ov2), fmaxf(v1, ov1));
        if (ov1 < v1 || (ov1 == v1 && oi < i1)) i1 = oi;
        v1 = fminf(v1, ov1);
    }
    double xn = 0.0;
    for (int kk = lane; kk < d; kk += 32) {
        const double xv = static_cast<double>(X[p * d + kk]);
        xn += xv * xv;
    }
    xn = warp_sum(xn);
    if (lane == 0) {
        const double u = 5.9604644775390625e-08;  // 2^-24
        const double g = (d + 8) * u / (1.0 - (d + 8) * u);
        const double Cn = sqrt(__longlong_as_double(*cmax)) * (1.0 + 1e-12);
        const double x = sqrt(xn) * (1.0 + 1e-12);
        const double E = 1.05 * ((2.0 * g + 4.0 * u) * x * Cn + 4.0 * u * Cn * Cn + u * u * Cn * Cn) +
                         1e-12 * (x + Cn) * (x + Cn);
        const double gap = static_cast<double>(v2) - static_cast<double>(v1);
        if (gap > 2.0 * E) out[p] = static_cast<uint32_t>(i1);
        else amb[atomicAdd(namb, 1u)] = static_cast<uint32_t>(p);
    }
}

void assign_gemm_filter(Ctx& ctx, const float* X, long long N, int d, const double* C, int k, uint32_t* out,
                        uint32_t* amb, unsigned* namb) {
    cudaStream_t s = ctx.stream;
    const int Kp = static_cast<int>(ceil_div(k, 32)) * 32;
    DevBuf<float> CfT(static_cast<size_t>(d) * Kp), ncf(Kp);
    DevBuf<unsigned long long> cmax(1);
    cmax.zero(s);
    filter_prep_kernel<<<Kp, 128, 0, s>>>(C, k, d, Kp, CfT.get(), ncf.get(), cmax.get());
    LAUNCH_OK("gemm filter prep");
    const long long chunk = std::max<long long>(1, std::min<long long>(N, (64LL << 20) / Kp));  // 256 MB of scores
    DevBuf<float> S(static_cast<size_t>(chunk) * Kp);
    cublasHandle_t h = cublas_of(ctx);
    const float one = 1.0f, zero = 0.0f;
    for (long long p0 = 0; p0 < N; p0 += chunk) {
        const long long np = std::min(chunk, N - p0);
        // S (Kp x np, column-major) = CfT^T-view (Kp x d) * X_chunk^T (d x np)
        if (cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, Kp, static_cast<int>(np), d, &one, CfT.get(), CUDA_R_32F, Kp,
                         X + p0 * d, CUDA_R_32F, d, &zero, S.get(), CUDA_R_32F, Kp, CUBLAS_COMPUTE_32F_PEDANTIC,
                         CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
            throw Status(100, "cublasGemmEx failed (assignment filter)");
        gemm_top2_kernel<<<static_cast<unsigned>(ceil_div(np, 8)), 256, 0, s>>>(X, p0, np, d, S.get(), Kp, k,
                                                                                ncf.get(), cmax.get(), out, amb,
                                                                                namb);
        LAUNCH_OK("gemm_top2_kernel");
    }
}

template <typename T>
void assign_device(Ctx& ctx, const T* X, long long N, int d, const double* C, int k, uint32_t* out) {
    if (N == 0) return;
    cudaStream_t s = ctx.stream;
    // fp32 filter for big problems with fp32 points: a GEMM + top-2 pass for
    // d > kFD (LCN_FILTER=exact: no filter there)
    const char* fsel0 = std::getenv("LCN_FILTER");
    if (std::is_same<T, float>::value && d > kFD && N * static_cast<long long>(k) >= (1LL << 22) &&
        !(fsel0 && std::string(fsel0) == "exact")) {
        DevBuf<uint32_t> amb(N);
        DevBuf<unsigned> namb(1);
        namb.zero(s);
        assign_gemm_filter(ctx, reinterpret_cast<const float*>(X), N, d, C, k, out, amb.get(), namb.get());
        unsigned h_amb = 0;
        namb.download(&h_amb, 1, s);
        ctx.sync();
        ctx.filter_ambiguous += h_amb;
        ctx.filter_points += N;
        if (h_amb)
            assign_exact_launch<T>(ctx, X, h_amb, d, C, k, out, nullptr, amb.get(), nullptr, nullptr);
        LAUNCH_OK("assign_exact_kernel (ambiguous, gemm filter)");
        return;
    }
    // fp32 filter for big problems (fp32 points, d <= kFD)
    if (std::is_same<T, float>::value && d <= kFD && N * static_cast<long long>(k) >= (1LL << 22)) {
        const int Kp = static_cast<int>(ceil_div(k, kFB)) * kFB;
        DevBuf<float> CfT(static_cast<size_t>(d) * Kp), ncf(Kp);
        DevBuf<unsigned long long> cmax(1);
        DevBuf<uint32_t> amb(N);
        DevBuf<unsigned> namb(1);
        cmax.zero(s);
        namb.zero(s);
        // tensor-core (tcgen05, 3xTF32) filter; the fp32 FMA filter when the
        // shape is not handled or LCN_FILTER=fma
        const char* fsel = std::getenv("LCN_FILTER");
        const bool fma_only = fsel && std::string(fsel) == "fma";
        if (fma_only || !assign_filter_tc(ctx, reinterpret_cast<const float*>(X), N, d, C, k, out, amb.get(),
                                          namb.get())) {
            filter_prep_kernel<<<Kp, 128, 0, s>>>(C, k, d, Kp, CfT.get(), ncf.get(), cmax.get());
            static std::atomic<bool> attr[64];  // set once per device; concurrent build jobs may race here (benign, idempotent)
            if (ctx.device >= 64 || !attr[ctx.device]) {
                CUDA_OK(cudaFuncSetAttribute(assign_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(FilterSmem))));
                if (ctx.device < 64) attr[ctx.device] = true;
            }
            assign_filter_kernel<<<ceil_div(N, kFB), 256, sizeof(FilterSmem), s>>>(
                reinterpret_cast<const float*>(X), N, d, CfT.get(), ncf.get(), Kp, cmax.get(), out, amb.get(),
                namb.get());
            LAUNCH_OK("assign_filter_kernel");
        }
        unsigned h_amb = 0;
        namb.download(&h_amb, 1, s);
        ctx.sync();
        ctx.filter_ambiguous += h_amb;
        ctx.filter_points += N;
        if (h_amb)
            assign_exact_launch<T>(ctx, X, h_amb, d, C, k, out, nullptr, amb.get(), nullptr, nullptr);
        LAUNCH_OK("assign_exact_kernel (ambiguous)");
        return;
    }
    assign_exact_launch<T>(ctx, X, N, d, C, k, out, nullptr, nullptr, nullptr, nullptr);
    LAUNCH_OK("assign_exact_kernel");
}

// ---- Lloyd with certified distance bounds (Hamerly) ------------------------
// After a full assignment every point carries ub >= its true distance to the
// chosen centroid and lb <= its true distance to every other centroid
// (assign_filter_tc / assign_exact_kernel). A Lloyd update moves centroid c
// by delta_c, so before the next assignment ub + delta_a and
// lb - max_{c != a} delta_c still bound the distances, and when
//   (ub + delta_a) (1 + 1e-9) < (lb - max delta) (1 - 1e-9)
// no other centroid can reach the assigned one: the reference's fp64 folds
// (within 1e-12 of the true squares) keep the same strict argmin
// (kmeans.cpp:76-82), so the point keeps its assignment with no tie possible.
// A failing point first tightens ub to its current distance (one row read);
// the rest are re-assigned by the tensor-core filter on a compacted list.
__global__ void centroid_shift_kernel(const double* __restrict__ cold, const double* __restrict__ cnew, int k, int d,
                                      double* __restrict__ delta) {
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (c >= k) return;
    double s2 = 0.0;
    for (int kk = lane; kk < d; kk += 32) {
        const double df = cnew[static_cast<long long>(c) * d + kk] - cold[static_cast<long long>(c) * d + kk];
        s2 += df * df;
    }
    s2 = warp_sum(s2);
    if (lane == 0) delta[c] = s2 > 0.0 ? __dsqrt_ru(s2) * (1.0 + 1e-12) : 0.0;
}

// largest and second-largest shift and the argmax (one CTA)
__global__ void __launch_bounds__(1024) shift_max_kernel(const double* __restrict__ delta, int k,
                                                         double* __restrict__ dstat) {
    __shared__ double m1s[32], m2s[32];
    __shared__ int a1s[32];
    double m1 = -1.0, m2 = -1.0;
    int a1 = -1;
    for (int c = threadIdx.x; c < k; c += 1024) {
        const double v = delta[c];
        if (v > m1) { m2 = m1; m1 = v; a1 = c; }
        else if (v > m2) m2 = v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double om1 = __shfl_xor_sync(0xffffffffu, m1, o), om2 = __shfl_xor_sync(0xffffffffu, m2, o);
        const int oa = __shfl_xor_sync(0xffffffffu, a1, o);
        m2 = fmax(fmax(m2, om2), fmin(m1, om1));
        if (om1 > m1) { m1 = om1; a1 = oa; }
    }
    if ((threadIdx.x & 31) == 0) {
        m1s[threadIdx.x >> 5] = m1;
        m2s[threadIdx.x >> 5] = m2;
        a1s[threadIdx.x >> 5] = a1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b1 = -1.0, b2 = -1.0;
        int ba = -1;
        for (int w = 0; w < 32; ++w) {
            b2 = fmax(fmax(b2, m2s[w]), fmin(b1, m1s[w]));
            if (m1s[w] > b1) { b1 = m1s[w]; ba = a1s[w]; }
        }
        dstat[0] = fmax(b1, 0.0);
        dstat[1] = fmax(b2, 0.0);
        dstat[2] = static_cast<double>(ba);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) lloyd_bounds_kernel(const T* __restrict__ X, long long N, int d,
                                                           const double* __restrict__ C,
                                                           const uint32_t* __restrict__ assign,
                                                           float* __restrict__ ub, float* __restrict__ lb,
                                                           const double* __restrict__ delta,
                                                           const double* __restrict__ dstat,
                                                           uint32_t* __restrict__ list, unsigned* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    const long long p = blockIdx.x * 256LL + threadIdx.x;
    const double dmax = dstat[0], dmax2 = dstat[1];
    const int amax = static_cast<int>(dstat[2]);
    uint32_t a = 0;
    double U = 0.0, L = 0.0;
    bool need = false;
    if (p < N) {
        a = assign[p];
        U = static_cast<double>(ub[p]) + delta[a];
        L = static_cast<double>(lb[p]) - (static_cast<int>(a) == amax ? dmax2 : dmax);
        need = !(U * (1.0 + 1e-9) < L * (1.0 - 1e-9));
        if (!need) {
            ub[p] = __double2float_ru(U);
            lb[p] = __double2float_rd(L);
        }
    }
    // tighten ub: the current distance to the assigned centroid, one
    // coalesced row read per failing point (any summation order: within
    // 1e-12 of the true square)
    unsigned m = __ballot_sync(0xffffffffu, need);
    bool still = false;
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const long long pj = __shfl_sync(0xffffffffu, p, j);
        const uint32_t aj = __shfl_sync(0xffffffffu, a, j);
        double s2 = 0.0;
        for (int kk = lane; kk < d; kk += 32) {
            const double df = static_cast<double>(X[pj * d + kk]) - C[static_cast<long long>(aj) * d + kk];
            s2 += df * df;
        }
        s2 = warp_sum(s2);
        if (lane == j) {
            const double Ut = __dsqrt_ru(s2 * (1.0 + 1e-12));
            if (Ut * (1.0 + 1e-9) < L * (1.0 - 1e-9)) {
                ub[p] = __double2float_ru(Ut);
                lb[p] = __double2float_rd(L);
            } else {
                still = true;
            }
        }
    }
    const unsigned sm = __ballot_sync(0xffffffffu, still);
    if (sm) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(count, static_cast<unsigned>(__popc(sm)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (still) list[base + __popc(sm & ((1u << lane) - 1u))] = static_cast<uint32_t>(p);
    }
}

// ---- Lloyd tile skipping (Elkan / Yinyang bounds per centroid tile) ---------
// Every full evaluation leaves, per point and tile of 128 centroids, a lower
// bound on the true distance to all of the tile's centroids (lbt, written
// by assign_filter_tc_kernel). After an update moving tile g's centroids by
// at most S_g, lbt - S_g still bounds them; a tile whose bound exceeds the
// point's upper bound ub + delta_a (its distance to its own centroid) holds
// no centroid that could be nearer (strictly, with margins), so it need not
// be evaluated. Points are taken in Lloyd's sorted order (grouped by
// centroid), and a cluster of 256 of them evaluates the union of their
// needed tiles: mostly the tiles of their own mixture component. The own
// tile always qualifies (its bound <= the distance to the own centroid), so
// the argmin over the evaluated tiles is the global one; ambiguous points
// still get the exact full scan.
__global__ void tile_shift_kernel(const double* __restrict__ delta, int k, int tn, const uint32_t* __restrict__ perm,
                                  double* __restrict__ tshift) {
    const int g = blockIdx.x, lane = threadIdx.x;
    double m = 0.0;
    for (int c = g * tn + lane; c < min(k, (g + 1) * tn); c += 32) m = fmax(m, delta[perm ? perm[c] : c]);
    m = warp_max(m);
    if (lane == 0) tshift[g] = m;
}

// Tile order of the centroids: each centroid's nearest among the first 32
// (the earliest k-means++ seeds, spread over the data) is its group; a
// stable sort by group packs nearby centroids into the same tiles.
__global__ void tile_group_kernel(const double* __restrict__ C, int k, int d, int G, uint32_t* __restrict__ grp) {
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (c >= k) return;
    double best = kPosInf;
    int arg = 0;
    for (int g = 0; g < G; ++g) {
        double s2 = 0.0;
        for (int kk = lane; kk < d; kk += 32) {
            const double df = C[static_cast<long long>(c) * d + kk] - C[static_cast<long long>(g) * d + kk];
            s2 += df * df;
        }
        s2 = warp_sum(s2);
        if (s2 < best) { best = s2; arg = g; }
    }
    if (lane == 0) grp[c] = static_cast<uint32_t>(arg);
}

__global__ void __launch_bounds__(256) tile_need_kernel(const uint32_t* __restrict__ order, long long N,
                                                        const uint32_t* __restrict__ assign,
                                                        const float* __restrict__ ub,
                                                        const double* __restrict__ delta,
                                                        const double* __restrict__ tshift, int ntile,
                                                        float* __restrict__ lbt,
                                                        unsigned long long* __restrict__ masks) {
    __shared__ unsigned long long wm[8];
    const long long p = blockIdx.x * 256LL + threadIdx.x;
    unsigned long long m = 0;
    if (p < N) {
        const long long q = order[p];
        const double U = (static_cast<double>(ub[q]) + delta[assign[q]]) * (1.0 + 1e-9);
        float* L = lbt + q * ntile * 2;
        for (int g = 0; g < ntile; ++g) {
            const double l = static_cast<double>(fminf(L[2 * g], L[2 * g + 1])) - tshift[g];
            const float lf = __double2float_rd(l * (1.0 - 1e-9));
            L[2 * g] = lf;
            L[2 * g + 1] = lf;
            if (!(static_cast<double>(lf) > U)) m |= 1ull << g;
        }
    }
    // OR over the block (the cluster's 256 points)
#pragma unroll
    for (int o = 16; o; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long all = 0;
        for (int w = 0; w < 8; ++w) all |= wm[w];
        masks[blockIdx.x] = all;
    }
}

__global__ void tile_count_kernel(const unsigned long long* __restrict__ masks, int ncl, int* __restrict__ cnt) {
    const int c = blockIdx.x * 256 + threadIdx.x;
    if (c < ncl) cnt[c] = __popcll(masks[c]);
}

__global__ void tile_fill_kernel(const unsigned long long* __restrict__ masks, int ncl, const int* __restrict__ off,
                                 int* __restrict__ tl) {
    const int c = blockIdx.x * 256 + threadIdx.x;
    if (c >= ncl) return;
    unsigned long long m = masks[c];
    int o = off[c];
    while (m) {
        tl[o++] = __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
    }
}

// Tensor-core assignment of the points rows[0 .. n) (all points when rows is
// null) with bounds; ambiguous points get the exact scan (and exact bounds).
template <typename T>
void assign_bounded(Ctx& ctx, const T* X, long long n, int d, const double* C, int k, uint32_t* out,
                    const uint32_t* rows, float* ub, float* lb, const int* tl_off = nullptr, const int* tl = nullptr,
                    float* lbt = nullptr, const uint32_t* perm = nullptr) {
    cudaStream_t s = ctx.stream;
    DevBuf<uint32_t> amb(n);
    DevBuf<unsigned> namb(1);
    namb.zero(s);
    if (!assign_filter_tc(ctx, reinterpret_cast<const float*>(X), n, d, C, k, out, amb.get(), namb.get(), nullptr, 0,
                          rows, ub, lb, tl_off, tl, lbt, perm))
        throw Status(100, "lloyd bounds: tensor-core filter unavailable for this shape");
    unsigned h_amb = 0;
    namb.download(&h_amb, 1, s);
    ctx.sync();
    ctx.filter_ambiguous += h_amb;
    ctx.filter_points += n;
    if (h_amb)
        assign_exact_launch<T>(ctx, X, h_amb, d, C, k, out, nullptr, amb.get(), ub, lb);
    LAUNCH_OK("assign_exact_kernel (ambiguous, bounds)");
}

PPSeq lloyd_seed_seq(uint64_t seed, long long N, int k, uint32_t* d_chosen) {
    // k-means++ init with the reference's engine and distributions (kmeans.cpp:93-94).
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<std::size_t> first(0, static_cast<std::size_t>(N - 1));
    PPSeq q;
    q.k = k;
    q.first = first(rng);
    q.raw.resize(k > 1 ? k - 1 : 0);
    for (auto& r : q.raw) r = rng();
    q.d_chosen = d_chosen;
    q.draws_used = nullptr;
    return q;
}

template <typename T>
void lloyd_device(Ctx& ctx, const T* X, long long N, int d, int k, int iters, uint64_t seed, double* d_ctr,
                  uint32_t* d_assign, const uint32_t* init_in) {
    if (N == 0) throw Status(2, "k-means on empty input");
    if (k == 0 || k > N) throw Status(2, "k-means: more buckets than points");
    cudaStream_t s = ctx.stream;
    DevBuf<uint32_t> init_buf(init_in ? 1 : k);
    const uint32_t* init = init_in;
    if (!init_in) {
        PhaseTimer pt(ctx, "  k-means++ seeding");
        kmeans_pp_batch<T>(ctx, X, N, d, {lloyd_seed_seq(seed, N, k, init_buf.get())});
        init = init_buf.get();
    }
    PhaseTimer pt_lloyd(ctx, "  lloyd iterations + final assign");
    // centroids = rows of the seeds (kmeans.cpp:99-100)
    {
        DevBuf<int> dummy_counts(k), dummy_start(k);
        std::vector<int> ones(k, 1), st(k);
        for (int c = 0; c < k; ++c) st[c] = c;
        dummy_counts.upload(ones.data(), k, s);
        dummy_start.upload(st.data(), k, s);
        centroid_kernel<T><<<k, 128, 0, s>>>(X, d, init, dummy_start.get(), dummy_counts.get(), d_ctr);
        LAUNCH_OK("centroid init");
        ctx.sync();
    }
    DevBuf<int> counts(k), start(k);
    DevBuf<uint32_t> keys_out(N), order(N), iota(N);
    iota_kernel<<<ceil_div(N, 256), 256, 0, s>>>(iota.get(), N);
    size_t tmp_sort = 0, tmp_scan = 0;
    int end_bit = 1;
    while ((1LL << end_bit) < k) ++end_bit;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, d_assign, keys_out.get(), iota.get(), order.get(),
                                    static_cast<int>(N), 0, end_bit, s);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, counts.get(), start.get(), k, s);
    DevBuf<unsigned char> tmp(std::max(tmp_sort, tmp_scan));
    const int fparts = std::min<long long>(ceil_div(N, 256), 4 * ctx.num_sms);
    DevBuf<double> pval(fparts);
    DevBuf<long long> pidx(fparts);
    std::vector<int> h_counts(k);
    // certified bounds (Hamerly) on the tensor-core path; LCN_LLOYD_BOUNDS=0
    // re-assigns every point every iteration
    const char* benv = std::getenv("LCN_LLOYD_BOUNDS");
    const char* fsel = std::getenv("LCN_FILTER");
    const bool bounds = std::is_same<T, float>::value && d <= 128 && N * static_cast<long long>(k) >= (1LL << 22) &&
                        !(benv && benv[0] == '0') && !(fsel && std::string(fsel) == "fma");
    DevBuf<float> ub(bounds ? N : 1), lb(bounds ? N : 1);
    DevBuf<double> cold(bounds ? static_cast<size_t>(k) * d : 1), delta(bounds ? k : 1), dstat(3);
    DevBuf<uint32_t> blist(bounds ? N : 1);
    DevBuf<unsigned> bcnt(1);
    long long reassigned = 0;
    // Sharded build (a communicator on the context): rank r assigns the
    // points [r S, (r + 1) S), S = ceil(N / world), and one all-gather gives
    // every rank the whole assignment; the centroid update, the reseeding and
    // the shifts then run identically on every rank. Every assignment is the
    // exact argmin, so the result is bit-identical for any world size.
    Comm* cm = ctx.comm && ctx.comm->world > 1 ? ctx.comm.get() : nullptr;
    const long long S = cm ? ceil_div(N, cm->world) : N;
    const long long lo = cm ? std::min(N, static_cast<long long>(cm->rank) * S) : 0;
    const long long Nr = cm ? std::min(N, lo + S) - lo : N;
    DevBuf<uint32_t> gsend(cm ? S : 1), grecv(cm ? S * cm->world : 1);
    auto gather_assign = [&] {
        if (!cm) return;
        CUDA_OK(cudaMemsetAsync(gsend.get(), 0, static_cast<size_t>(S) * 4, s));
        if (Nr)
            CUDA_OK(cudaMemcpyAsync(gsend.get(), d_assign + lo, static_cast<size_t>(Nr) * 4, cudaMemcpyDeviceToDevice,
                                    s));
        cm->allgather(gsend.get(), grecv.get(), static_cast<size_t>(S) * 4, s);
        CUDA_OK(cudaMemcpyAsync(d_assign, grecv.get(), static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s));
    };
    // tile skipping (bounds path, one rank, 8..64 tiles of 128 centroids;
    // LCN_LLOYD_TILES=0: every tile every time)
    const int ntile_c = assign_tc_tile_count(k);
    const char* tenv = std::getenv("LCN_LLOYD_TILES");
    const bool tiles = bounds && !cm && ntile_c >= 8 && ntile_c <= 64 && !(tenv && tenv[0] == '0');
    const int ncl = static_cast<int>(ceil_div(N, 256));
    DevBuf<float> lbt(tiles ? static_cast<size_t>(N) * ntile_c * 2 : 1);
    DevBuf<double> tshift(tiles ? ntile_c : 1);
    DevBuf<unsigned long long> tmask(tiles ? ncl : 1);
    DevBuf<int> tcnt(tiles ? ncl : 1), toff(tiles ? ncl + 1 : 1), tlst(tiles ? static_cast<size_t>(ncl) * ntile_c : 1);
    size_t tscan = 0;
    if (tiles) cub::DeviceScan::InclusiveSum(nullptr, tscan, tcnt.get(), toff.get() + 1, ncl, s);
    DevBuf<unsigned char> ttmp(std::max<size_t>(tscan, 1));
    long long tiles_eval = 0;
    DevBuf<uint32_t> tperm(tiles ? k : 1);
    if (tiles) {  // centroid tile order from the initial centroids (the seeds)
        DevBuf<uint32_t> grp(k), grp_s(k), idx(k);
        tile_group_kernel<<<ceil_div(k, 8), 256, 0, s>>>(d_ctr, k, d, std::min(k, 32), grp.get());
        iota_kernel<<<ceil_div(k, 256), 256, 0, s>>>(idx.get(), k);
        size_t ts = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, ts, grp.get(), grp_s.get(), idx.get(), tperm.get(), k, 0, 6, s);
        DevBuf<unsigned char> tt(std::max<size_t>(ts, 1));
        cub::DeviceRadixSort::SortPairs(tt.get(), ts, grp.get(), grp_s.get(), idx.get(), tperm.get(), k, 0, 6, s);
        LAUNCH_OK("lloyd tile order");
    }
    const char* tpenv = std::getenv("LCN_LLOYD_TILE_ORDER");
    const uint32_t* tp = tiles && !(tpenv && tpenv[0] == '0') ? tperm.get() : nullptr;
    const T* Xr = X + lo * d;
    uint32_t* ar = d_assign + lo;
    float* ubr = ub.get() + (bounds ? lo : 0);
    float* lbr = lb.get() + (bounds ? lo : 0);
    auto assign_step = [&](bool first) {
        if (tiles) {
            if (first) {
                assign_bounded<T>(ctx, X, N, d, d_ctr, k, d_assign, nullptr, ub.get(), lb.get(), nullptr, nullptr,
                                  lbt.get(), tp);
                reassigned += N;
                tiles_eval += static_cast<long long>(ncl) * ntile_c;
                return;
            }
            tile_shift_kernel<<<ntile_c, 32, 0, s>>>(delta.get(), k, 128, tp, tshift.get());
            tile_need_kernel<<<ncl, 256, 0, s>>>(order.get(), N, d_assign, ub.get(), delta.get(), tshift.get(), ntile_c,
                                                 lbt.get(), tmask.get());
            tile_count_kernel<<<ceil_div(ncl, 256), 256, 0, s>>>(tmask.get(), ncl, tcnt.get());
            CUDA_OK(cudaMemsetAsync(toff.get(), 0, sizeof(int), s));
            size_t t1 = ttmp.size();
            cub::DeviceScan::InclusiveSum(ttmp.get(), t1, tcnt.get(), toff.get() + 1, ncl, s);
            tile_fill_kernel<<<ceil_div(ncl, 256), 256, 0, s>>>(tmask.get(), ncl, toff.get(), tlst.get());
            LAUNCH_OK("lloyd tile lists");
            if (std::getenv("LCN_TIMING")) {
                int tot = 0;
                CUDA_OK(cudaMemcpyAsync(&tot, toff.get() + ncl, sizeof(int), cudaMemcpyDeviceToHost, s));
                ctx.sync();
                tiles_eval += tot;
            }
            assign_bounded<T>(ctx, X, N, d, d_ctr, k, d_assign, order.get(), ub.get(), lb.get(), toff.get(),
                              tlst.get(), lbt.get(), tp);
            reassigned += N;
            return;
        }
        if (!bounds) {
            if (Nr) assign_device<T>(ctx, Xr, Nr, d, d_ctr, k, ar);
            gather_assign();
            return;
        }
        if (first) {
            if (Nr) assign_bounded<T>(ctx, Xr, Nr, d, d_ctr, k, ar, nullptr, ubr, lbr);
            reassigned += Nr;
            gather_assign();
            return;
        }
        bcnt.zero(s);
        if (Nr)
            lloyd_bounds_kernel<T><<<ceil_div(Nr, 256), 256, 0, s>>>(Xr, Nr, d, d_ctr, ar, ubr, lbr, delta.get(),
                                                                    dstat.get(), blist.get(), bcnt.get());
        LAUNCH_OK("lloyd bounds");
        unsigned h = 0;
        bcnt.download(&h, 1, s);
        ctx.sync();
        reassigned += h;
        if (h) assign_bounded<T>(ctx, Xr, h, d, d_ctr, k, ar, blist.get(), ubr, lbr);
        gather_assign();
    };
    // Fixed point: when an assignment equals the previous one and the update
    // before it reseeded nothing, that update's centroids come back
    // bit-identical (same members, same fold order), so every later
    // iteration and the final assignment repeat this assignment: stop here
    // (the reference keeps iterating to the same result). LCN_LLOYD_EARLY_EXIT=0
    // runs every iteration.
    const char* eenv = std::getenv("LCN_LLOYD_EARLY_EXIT");
    const bool early_exit = !(eenv && eenv[0] == '0');
    DevBuf<uint32_t> prev(early_exit ? N : 1);
    DevBuf<unsigned long long> nchg(1);
    bool reseeded_prev = true;  // iteration 0 has no previous assignment
    int exit_it = -1;
    for (int it = 0; it < iters; ++it) {
        assign_step(it == 0);
        if (early_exit) {
            if (!reseeded_prev) {
                nchg.zero(s);
                count_changes_kernel<<<static_cast<unsigned>(std::min<long long>(ceil_div(N, 256), 4LL * ctx.num_sms)),
                                       256, 0, s>>>(d_assign, prev.get(), N, nchg.get());
                unsigned long long hc = 1;
                nchg.download(&hc, 1, s);
                ctx.sync();
                if (hc == 0) {
                    exit_it = it;
                    break;
                }
            }
            CUDA_OK(cudaMemcpyAsync(prev.get(), d_assign, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (bounds)
            CUDA_OK(cudaMemcpyAsync(cold.get(), d_ctr, static_cast<size_t>(k) * d * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
        counts.zero(s);
        count_kernel<<<ceil_div(N, 256), 256, 0, s>>>(d_assign, N, counts.get());
        size_t t1 = tmp.size();
        cub::DeviceScan::ExclusiveSum(tmp.get(), t1, counts.get(), start.get(), k, s);
        t1 = tmp.size();
        cub::DeviceRadixSort::SortPairs(tmp.get(), t1, d_assign, keys_out.get(), iota.get(), order.get(),
                                        static_cast<int>(N), 0, end_bit, s);
        centroid_kernel<T><<<k, 128, 0, s>>>(X, d, order.get(), start.get(), counts.get(), d_ctr);
        LAUNCH_OK("lloyd update");
        counts.download(h_counts.data(), k, s);
        ctx.sync();
        reseeded_prev = false;
        for (int c = 0; c < k; ++c) {
            if (h_counts[c] != 0) continue;
            reseeded_prev = true;
            farthest_partial_kernel<T><<<fparts, 256, 0, s>>>(X, N, d, d_ctr, d_assign, counts.get(), pval.get(), pidx.get());
            reseed_apply_kernel<T><<<1, 128, 0, s>>>(X, d, pval.get(), pidx.get(), fparts, d_ctr, d_assign, counts.get(), c,
                                                     bounds ? lb.get() : nullptr);
            LAUNCH_OK("reseed");
        }
        if (bounds) {
            centroid_shift_kernel<<<ceil_div(k, 8), 256, 0, s>>>(cold.get(), d_ctr, k, d, delta.get());
            shift_max_kernel<<<1, 1024, 0, s>>>(delta.get(), k, dstat.get());
            LAUNCH_OK("centroid shifts");
        }
    }
    if (exit_it < 0) assign_step(iters == 0);
    if (exit_it >= 0 && std::getenv("LCN_TIMING"))
        std::fprintf(stderr, "[lloyd] N=%lld k=%d: fixed point at iteration %d of %d (the rest skipped)\n", N, k,
                     exit_it, iters);
    if (tiles && std::getenv("LCN_TIMING"))
        std::fprintf(stderr, "[lloyd] N=%lld k=%d: tile skipping evaluated %lld of %lld cluster x tile blocks (%.1f%%)\n",
                     N, k, tiles_eval, static_cast<long long>(ncl) * ntile_c * (iters + 1),
                     100.0 * tiles_eval / (static_cast<double>(ncl) * ntile_c * (iters + 1)));
    if (bounds && std::getenv("LCN_TIMING"))
        std::fprintf(stderr, "[lloyd] N=%lld k=%d%s: %lld of %lld point assignments re-evaluated (%.1f%%)\n", N, k,
                     cm ? " (this rank's slice)" : "", reassigned, Nr * (iters + 1),
                     100.0 * reassigned / (static_cast<double>(std::max(Nr, 1LL)) * (iters + 1)));
}

#define LCNB_INST(T)                                                                                    \
    template void kmeans_pp_device<T>(Ctx&, const T*, long long, int, int, uint64_t,                    \
                                      const std::vector<unsigned long long>&, uint32_t*, int*);         \
    template void assign_device<T>(Ctx&, const T*, long long, int, const double*, int, uint32_t*);      \
    template void kmeans_pp_batch<T>(Ctx&, const T*, long long, int, const std::vector<PPSeq>&);          \
    template void lloyd_device<T>(Ctx&, const T*, long long, int, int, int, uint64_t, double*, uint32_t*,  \
                                  const uint32_t*);
LCNB_INST(double)
LCNB_INST(float)
#undef LCNB_INST

}  // namespace lcnb
