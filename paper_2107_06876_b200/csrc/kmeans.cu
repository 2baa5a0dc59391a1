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
                                                           const uint32_t* __restrict__ rows) {
    __shared__ double As[KC][TP + 1];
    __shared__ double Bs[KC][TC + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const long long p0 = static_cast<long long>(blockIdx.x) * TP;
    double best[4];
    int arg[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { best[i] = kPosInf; arg[i] = 0; }
    for (int c0 = 0; c0 < k; c0 += TC) {
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
            if (c < k)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (acc[i][j] < best[i]) { best[i] = acc[i][j]; arg[i] = c; }
        }
    }
    // (value, index) lexicographic min over the 16 threads sharing a point.
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double b = best[i];
        int a = arg[i];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            double ob = __shfl_xor_sync(0xffffffffu, b, o);
            int oa = __shfl_xor_sync(0xffffffffu, a, o);
            if (ob < b || (ob == b && oa < a)) { b = ob; a = oa; }
        }
        long long p = p0 + ty + 16 * i;
        if (tx == 0 && p < N) {
            const long long q = rows ? rows[p] : p;
            out[q] = static_cast<uint32_t>(a);
            if (best_out) best_out[q] = b;
        }
    }
}

// ---- k-means++ (kmeans.cpp:23-65) ------------------------------------------
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
__global__ void __launch_bounds__(256) pp_prune_kernel(long long N, int t, const double* __restrict__ dist2,
                                                       const uint32_t* __restrict__ near,
                                                       const double* __restrict__ dc, uint32_t* __restrict__ list,
                                                       unsigned* __restrict__ count) {
    const long long p = blockIdx.x * 256LL + threadIdx.x;
    bool need = p < N;
    if (need && t > 0) {
        const double D = dist2[p];
        if (D < kPosInf) {
            const double lb = dc[near[p]] * (1.0 - 1e-12);
            if (lb >= 2.0 * sqrt(D) * (1.0 + 1e-9)) need = false;
        }
    }
    // block-aggregated append: one global atomic per block (a single counter
    // hit by every warp serialises at L2)
    __shared__ unsigned wcnt[8], wbase[8], bbase;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (lane == 0) wcnt[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int w = 0; w < 8; ++w) {
            wbase[w] = tot;
            tot += wcnt[w];
        }
        bbase = tot ? atomicAdd(count, tot) : 0u;
    }
    __syncthreads();
    if (need) list[bbase + wbase[warp] + __popc(m & ((1u << lane) - 1u))] = static_cast<uint32_t>(p);
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
                                                       const unsigned* __restrict__ count) {
    extern __shared__ __align__(16) unsigned char dyn[];
    double* cs = reinterpret_cast<double*>(dyn);  // the new seed, fp64
    T* rows = reinterpret_cast<T*>(cs + d);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T* buf = rows + static_cast<size_t>(warp) * 32 * (d + 1);
    const long long last = chosen[t];
    for (int k = threadIdx.x; k < d; k += blockDim.x) cs[k] = static_cast<double>(X[last * d + k]);
    __syncthreads();
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
            if (acc < dist2[mine]) {
                dist2[mine] = acc;
                near[mine] = static_cast<uint32_t>(t);
            }
        }
        __syncwarp();
    }
}

// dc[j] = |x_{chosen[j]} - x_{chosen[t]}| for j < t (fp64, one warp per j)
template <typename T>
__global__ void __launch_bounds__(256) seed_dist_kernel(const T* __restrict__ X, int d,
                                                        const uint32_t* __restrict__ chosen, int t,
                                                        double* __restrict__ dc) {
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
struct FoldResult {
    double s;
    long long pick;
};

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

// ---- chunk-parallel exact fold ----------------------------------------------
// The fold over N values is cut into chunks of kFoldChunk. Most chunks lie
// inside one binade of the running sum, where the fold's result depends only
// on that binade: S_end = S_start + u_e * sum_j RN(x_j / u_e). So
//   A) approximate chunk sums (any order)            -> predicted start A_c
//   B) predicted binade e_c of each chunk (dirty if the interval
//      [A_c (1-1e-9), A_{c+1} (1+1e-9)] straddles a power of two)
//   C) the chunk's parity function R_c(e_c) = {inc[0], inc[1]} in parallel
//      (ties included), dirty only on huge x
//   D) one warp walks the chunks in order with the exact running sum: runs
//      of clean chunks whose actual binade matches e_c advance by a
//      parity-scan of their R_c, any other chunk is folded element-wise by
//      block_exact_fold.
// The prediction only decides which path a chunk takes; the walk re-checks
// the actual binade, so the result is exact regardless.
constexpr int kFoldChunk = 2048;

__global__ void fold_chunk_sum_kernel(const double* __restrict__ x, long long N, double* __restrict__ csum) {
    __shared__ double red[8];
    const long long b = static_cast<long long>(blockIdx.x) * kFoldChunk;
    const long long e = min(N, b + kFoldChunk);
    double s = 0.0;
    for (long long i = b + threadIdx.x; i < e; i += blockDim.x) s += x[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        csum[blockIdx.x] = t;
    }
}

__global__ void fold_plan_kernel(const double* __restrict__ csum, int nch, int* __restrict__ ebin) {
    // single block of 1024: blocked exclusive scan of the approximate sums
    __shared__ double tot[1024];
    const int per = (nch + 1023) / 1024;
    const int c0 = threadIdx.x * per, c1 = min(nch, c0 + per);
    double s = 0.0;
    for (int c = c0; c < c1; ++c) s += csum[c];
    tot[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        double v = threadIdx.x >= o ? tot[threadIdx.x - o] : 0.0;
        __syncthreads();
        tot[threadIdx.x] += v;
        __syncthreads();
    }
    double a = threadIdx.x ? tot[threadIdx.x - 1] : 0.0;
    for (int c = c0; c < c1; ++c) {
        double lo = a * (1.0 - 1e-9), hi = (a + csum[c]) * (1.0 + 1e-9);
        a += csum[c];
        int e = -100000;
        if (lo >= kMinNormal && hi < kPosInf && ilogb(lo) == ilogb(hi)) e = ilogb(lo);
        ebin[c] = e;
    }
}

__global__ void __launch_bounds__(256) fold_round_kernel(const double* __restrict__ x, long long N,
                                                         const int* __restrict__ ebin, longlong2* __restrict__ R) {
    constexpr int kPer = kFoldChunk / 256;  // contiguous elements per thread, in order
    __shared__ ParInc wred[8];
    __shared__ int bad_any;
    const int e = ebin[blockIdx.x];
    if (e == -100000) {
        if (threadIdx.x == 0) R[blockIdx.x] = make_longlong2(-1, -1);
        return;
    }
    if (threadIdx.x == 0) bad_any = 0;
    __syncthreads();
    const long long b = static_cast<long long>(blockIdx.x) * kFoldChunk + threadIdx.x * kPer;
    ParInc acc{0, 0};
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const long long i = b + j;
        if (i < N) {
            const double q = scale_to_grid(x[i], e);
            if (!(q < 9007199254740992.0)) bad = true;
            else acc = par_compose(acc, par_element(q));
        }
    }
    if (bad) bad_any = 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    acc = par_scan(acc, lane);
    if (lane == 31) wred[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        ParInc t{0, 0};
        for (int w = 0; w < 8; ++w) t = par_compose(t, wred[w]);
        R[blockIdx.x] = bad_any ? make_longlong2(-1, -1) : make_longlong2(t.i0, t.i1);
    }
}

// ---- block-wide exact fold of one staged chunk (kWalkThreads threads) -----
// Thread t owns elements [kSeg t, kSeg t + kSeg) of the chunk. While the running
// sum is normal in binade e, every thread composes its segment's parity
// function (ParInc) and a block scan gives each segment's start and end sums.
// The first segment that holds a huge element, leaves the binade, or (search)
// reaches the target is walked element by element by its owner, which
// publishes the exact stop; a stop element gets a real fp64 add and the fold
// restarts behind it. A chunk typically restarts once per binade change.
constexpr int kWalkThreads = 256;
constexpr int kSeg = kFoldChunk / kWalkThreads;

struct WalkShared {
    double buf[kFoldChunk];
    ParInc wsum[kWalkThreads / 32];
    int flag_min;
    int ev;           // 0: segment walked, no event; 1: real add at `stop`; 2: pick
    int stop;
    long long s_sig;  // significand before `stop` (ev 1) / after the segment (ev 0, 2)
    long long pick;
};

__device__ FoldResult block_exact_fold(WalkShared& sh, int cnt, long long base, double s, bool search,
                                       double target) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* xs = sh.buf;
    int a = 0;
    long long pick = -1;
    while (a < cnt) {
        if (!(s >= kMinNormal && s < kPosInf)) {  // zero / subnormal / inf: one real add
            const double va = xs[a];
            s = xadd(s, va);
            if (search && s >= target && va > 0.0) { pick = base + a; break; }
            ++a;
            continue;
        }
        const int e = dbl_exp(s);
        const long long S = dbl_sig(s);
        const int lo = max(a, kSeg * tid), hi = min(cnt, kSeg * tid + kSeg);
        ParInc f{0, 0};
        bool big = false;
        for (int i = lo; i < hi; ++i) {
            const double q = scale_to_grid(xs[i], e);
            if (!(q < 9007199254740992.0)) { big = true; break; }
            f = par_compose(f, par_element(q));
        }
        const ParInc inc = par_scan(f, lane);  // inclusive, within the warp
        if (lane == 31) sh.wsum[warp] = inc;
        if (tid == 0) sh.flag_min = kWalkThreads;
        __syncthreads();
        ParInc pre{0, 0};
        for (int w = 0; w < warp; ++w) pre = par_compose(pre, sh.wsum[w]);
        const ParInc up = par_shfl_up(inc, 1);
        const ParInc ex = par_compose(pre, lane ? up : ParInc{0, 0});  // before this segment
        const ParInc fe = par_compose(ex, f);                              // through this segment
        const long long s0 = S + ((S & 1) ? ex.i1 : ex.i0);
        const long long s1 = S + ((S & 1) ? fe.i1 : fe.i0);
        bool flag = lo < hi && (big || s1 >= kTwo53);
        if (search && lo < hi && s1 < kTwo53 && dbl_make(s1, e) >= target) flag = true;
        if (flag) atomicMin(&sh.flag_min, tid);
        __syncthreads();
        const int tf = sh.flag_min;
        if (tf == kWalkThreads) {  // no event: the rest of the chunk is one run
            if (tid == kWalkThreads - 1) sh.s_sig = s1;
            __syncthreads();
            s = dbl_make(sh.s_sig, e);
            break;
        }
        if (tid == tf) {
            long long cur = s0;
            int ev = 0, stop = hi;
            long long pk = -1;
            for (int i = lo; i < hi; ++i) {
                const double q = scale_to_grid(xs[i], e);
                if (!(q < 9007199254740992.0)) { ev = 1; stop = i; break; }
                const ParInc pe = par_element(q);
                const long long nx = cur + ((cur & 1) ? pe.i1 : pe.i0);
                if (nx >= kTwo53) { ev = 1; stop = i; break; }
                cur = nx;
                if (search && dbl_make(cur, e) >= target && xs[i] > 0.0) { ev = 2; pk = base + i; break; }
            }
            sh.ev = ev;
            sh.stop = stop;
            sh.s_sig = cur;
            sh.pick = pk;
        }
        __syncthreads();
        const int ev = sh.ev, stop = sh.stop;
        s = dbl_make(sh.s_sig, e);
        const long long pk = sh.pick;
        __syncthreads();  // shared state is rewritten by the next round
        if (ev == 2) { pick = pk; break; }
        if (ev == 0) { a = stop; continue; }
        const double vb = xs[stop];
        s = xadd(s, vb);
        if (search && s >= target && vb > 0.0) { pick = base + stop; break; }
        a = stop + 1;
    }
    return {s, pick};
}

// Stage chunk c of x into shared memory (all threads) and fold it.
__device__ __forceinline__ FoldResult fold_chunk_block(WalkShared& sh, const double* __restrict__ x, long long N,
                                                       int c, double s, bool search, double target) {
    const long long b = static_cast<long long>(c) * kFoldChunk;
    const int cnt = static_cast<int>(min(N - b, static_cast<long long>(kFoldChunk)));
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSeg; ++j) {
        const int i = threadIdx.x + j * kWalkThreads;
        sh.buf[i] = i < cnt ? x[b + i] : 0.0;
    }
    __syncthreads();
    return block_exact_fold(sh, cnt, b, s, search, target);
}

// D) walk + draw + pick for k-means++ step t (kmeans.cpp:35-62). raw[] holds
// the caller's engine draws in order; a step with total <= 0 consumes none
// (kmeans.cpp:42-47). Every warp runs the chunk walk redundantly (identical
// values, uniform control flow); chunks that need an element-wise fold use
// the whole block.
__global__ void __launch_bounds__(kWalkThreads) pp_walk_pick_kernel(
    double* __restrict__ dist2, unsigned char* __restrict__ used, long long N, int nch, const int* __restrict__ ebin,
    const longlong2* __restrict__ R, double* __restrict__ sstart, const unsigned long long* __restrict__ raw,
    int n_raw, int* __restrict__ draw_counter, uint32_t* __restrict__ chosen, int t, int staged) {
    __shared__ WalkShared sh;
    extern __shared__ __align__(16) unsigned char wdyn[];
    const int lane = threadIdx.x & 31;
    const bool w0 = threadIdx.x < 32;
    // chunk plans and the running-sum table in shared memory when they fit:
    // one memory latency for all plans instead of one per 32-chunk group
    if (staged) {
        longlong2* Rs = reinterpret_cast<longlong2*>(wdyn);
        double* ss = reinterpret_cast<double*>(Rs + nch);
        int* es = reinterpret_cast<int*>(ss + nch + 1);
        for (int c = threadIdx.x; c < nch; c += kWalkThreads) {
            Rs[c] = R[c];
            es[c] = ebin[c];
        }
        __syncthreads();
        R = Rs;
        ebin = es;
        sstart = ss;
    }
    double S = 0.0;
    // 32 chunks per step: a run of clean chunks in the running sum's binade
    // advances by an exact parity scan of their R_c
    for (int cb = 0; cb < nch; cb += 32) {
        const int c_l = cb + lane;
        const int e_l = c_l < nch ? ebin[c_l] : 0;
        const longlong2 r2 = c_l < nch ? R[c_l] : make_longlong2(-1, -1);
        const ParInc r_l{r2.x, r2.y};
        const int cnt = min(32, nch - cb);
        int k = 0;
        while (k < cnt) {
            const bool normal = S >= kMinNormal && S < kPosInf;
            const int eS = normal ? dbl_exp(S) : -100001;
            const long long Si = normal ? dbl_sig(S) : 0;
            const bool in = lane >= k && lane < cnt;
            const bool ok = in && normal && e_l == eS && r_l.i0 >= 0;
            const unsigned notok = __ballot_sync(0xffffffffu, in && !ok);
            int fb = notok ? __ffs(notok) - 1 : cnt;
            const bool run = lane >= k && lane < fb;
            const ParInc pf = par_scan(run ? r_l : ParInc{0, 0}, lane);
            const long long P = (Si & 1) ? pf.i1 : pf.i0;
            // a chunk whose end leaves the binade is folded element-wise
            const unsigned cross = __ballot_sync(0xffffffffu, run && Si + P >= kTwo53);
            if (cross) fb = min(fb, __ffs(cross) - 1);
            const long long Pprev = __shfl_up_sync(0xffffffffu, P, 1);
            const long long Pex = lane > k ? Pprev : 0;
            if (w0 && lane >= k && lane < fb) sstart[c_l] = dbl_make(Si + Pex, eS);
            if (fb > k) S = dbl_make(Si + __shfl_sync(0xffffffffu, P, fb - 1), eS);
            if (fb < cnt) {
                const int c = cb + fb;
                if (threadIdx.x == 0) sstart[c] = S;
                S = fold_chunk_block(sh, dist2, N, c, S, false, 0.0).s;
                k = fb + 1;
            } else {
                k = cnt;
            }
        }
    }
    if (threadIdx.x == 0) sstart[nch] = S;
    __syncthreads();
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
        __syncthreads();
        if (threadIdx.x == 0) sh.flag_min = nch;
        __syncthreads();
        for (int c = threadIdx.x; c < nch; c += kWalkThreads)
            if (sstart[c + 1] >= target) {
                atomicMin(&sh.flag_min, c);
                break;
            }
        __syncthreads();
        const int cstar = sh.flag_min;
        pick = -1;
        // the running sum reaches the target inside chunk cstar (an element
        // that raises it is > 0); later chunks only as a guard
        double sc = cstar < nch ? sstart[cstar] : 0.0;
        for (int cc = cstar; cc < nch && pick < 0; ++cc) {
            const FoldResult sr = fold_chunk_block(sh, dist2, N, cc, sc, true, target);
            pick = sr.pick;
            sc = sr.s;
        }
        if (pick < 0) pick = N - 1;
        __syncthreads();
        if (threadIdx.x == 0) *draw_counter = di + 1;
    }
    if (threadIdx.x == 0) {
        chosen[t] = static_cast<uint32_t>(pick);
        if (pick < N) {
            dist2[pick] = 0.0;
            used[pick] = 1;
        }
    }
}

__global__ void fill_kernel(double* p, long long n, double v) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) p[i] = v;
}

template <typename T>
void kmeans_pp_device(Ctx& ctx, const T* X, long long N, int d, int k, uint64_t first,
                      const std::vector<unsigned long long>& raw, uint32_t* d_chosen, int* draws_used) {
    cudaStream_t s = ctx.stream;
    const int nch = ceil_div(N, kFoldChunk);
    DevBuf<double> dist2(N), csum(nch), sstart(nch + 1);
    DevBuf<int> ebin(nch);
    DevBuf<longlong2> R(nch);
    DevBuf<unsigned char> used(N);
    // walk: chunk plans + running-sum table staged in shared memory if they fit
    size_t walk_smem = static_cast<size_t>(nch) * (sizeof(longlong2) + sizeof(double) + sizeof(int)) + sizeof(double);
    int walk_staged = walk_smem + sizeof(WalkShared) <= 200 * 1024;
    if (walk_staged)
        CUDA_OK(cudaFuncSetAttribute(pp_walk_pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(walk_smem)));
    else
        walk_smem = 0;
    DevBuf<uint32_t> near(N), list(N);
    DevBuf<unsigned> cnt(1);
    DevBuf<double> dc(std::max(k, 1));
    // exact-pass geometry: warps per CTA so one CTA's row buffers stay <= 96 KB
    int ex_warps = 4;
    while (ex_warps > 1 && static_cast<size_t>(ex_warps) * 32 * (d + 1) * sizeof(T) > 96 * 1024) ex_warps >>= 1;
    const size_t ex_smem = static_cast<size_t>(d) * 8 + static_cast<size_t>(ex_warps) * 32 * (d + 1) * sizeof(T);
    if (ex_smem > 200 * 1024) throw Status(2, "k-means++: dimension too large for the exact seeding pass");
    CUDA_OK(cudaFuncSetAttribute(pp_exact_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(ex_smem)));
    int ex_occ = 1;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ex_occ, pp_exact_kernel<T>, ex_warps * 32, ex_smem));
    const int ex_grid = std::max(1, ex_occ) * ctx.num_sms;
    DevBuf<unsigned long long> d_raw(raw.size() ? raw.size() : 1);
    DevBuf<int> counter(1);
    used.zero(s);
    near.zero(s);
    counter.zero(s);
    if (!raw.empty()) d_raw.upload(raw.data(), raw.size(), s);
    fill_kernel<<<ceil_div(N, 256), 256, 0, s>>>(dist2.get(), N, kPosInf);
    uint32_t f32 = static_cast<uint32_t>(first);
    unsigned char one = 1;
    CUDA_OK(cudaMemcpyAsync(d_chosen, &f32, 4, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(used.get() + first, &one, 1, cudaMemcpyHostToDevice, s));
    for (int t = 1; t < k; ++t) {
        if (t > 1) seed_dist_kernel<T><<<ceil_div(t - 1, 8), 256, 0, s>>>(X, d, d_chosen, t - 1, dc.get());
        cnt.zero(s);
        pp_prune_kernel<<<ceil_div(N, 256), 256, 0, s>>>(N, t - 1, dist2.get(), near.get(), dc.get(), list.get(),
                                                         cnt.get());
        pp_exact_kernel<T><<<ex_grid, ex_warps * 32, ex_smem, s>>>(X, d, d_chosen, t - 1, dist2.get(), near.get(),
                                                                   list.get(), cnt.get());
        fold_chunk_sum_kernel<<<nch, 256, 0, s>>>(dist2.get(), N, csum.get());
        fold_plan_kernel<<<1, 1024, 0, s>>>(csum.get(), nch, ebin.get());
        fold_round_kernel<<<nch, 256, 0, s>>>(dist2.get(), N, ebin.get(), R.get());
        pp_walk_pick_kernel<<<1, kWalkThreads, walk_smem, s>>>(dist2.get(), used.get(), N, nch, ebin.get(), R.get(),
                                                               sstart.get(), d_raw.get(), static_cast<int>(raw.size()),
                                                               counter.get(), d_chosen, t, walk_staged);
    }
    LAUNCH_OK("kmeans++");
    if (draws_used) counter.download(draws_used, 1, s);
    ctx.sync();
}

// ---- Lloyd (kmeans.cpp:87-143) ---------------------------------------------
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
                                    uint32_t* __restrict__ assign, int* __restrict__ counts, int c) {
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

template <typename T>
void assign_device(Ctx& ctx, const T* X, long long N, int d, const double* C, int k, uint32_t* out) {
    if (N == 0) return;
    cudaStream_t s = ctx.stream;
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
            static bool attr[64] = {};
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
            assign_exact_kernel<T><<<ceil_div(static_cast<long long>(h_amb), TP), 256, 0, s>>>(X, h_amb, d, C, k, out,
                                                                                                nullptr, amb.get());
        LAUNCH_OK("assign_exact_kernel (ambiguous)");
        return;
    }
    assign_exact_kernel<T><<<ceil_div(N, TP), 256, 0, s>>>(X, N, d, C, k, out, nullptr, nullptr);
    LAUNCH_OK("assign_exact_kernel");
}

template <typename T>
void lloyd_device(Ctx& ctx, const T* X, long long N, int d, int k, int iters, uint64_t seed, double* d_ctr,
                  uint32_t* d_assign) {
    if (N == 0) throw Status(2, "k-means on empty input");
    if (k == 0 || k > N) throw Status(2, "k-means: more buckets than points");
    cudaStream_t s = ctx.stream;
    // k-means++ init with the reference's engine and distributions (kmeans.cpp:93-94).
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<std::size_t> first(0, static_cast<std::size_t>(N - 1));
    uint64_t f = first(rng);
    std::vector<unsigned long long> raw(k > 1 ? k - 1 : 0);
    for (auto& r : raw) r = rng();
    DevBuf<uint32_t> init(k);
    {
        PhaseTimer pt(ctx, "  k-means++ seeding");
        kmeans_pp_device<T>(ctx, X, N, d, k, f, raw, init.get(), nullptr);
    }
    PhaseTimer pt_lloyd(ctx, "  lloyd iterations + final assign");
    // centroids = rows of the seeds (kmeans.cpp:99-100)
    {
        DevBuf<int> dummy_counts(k), dummy_start(k);
        std::vector<int> ones(k, 1), st(k);
        for (int c = 0; c < k; ++c) st[c] = c;
        dummy_counts.upload(ones.data(), k, s);
        dummy_start.upload(st.data(), k, s);
        centroid_kernel<T><<<k, 128, 0, s>>>(X, d, init.get(), dummy_start.get(), dummy_counts.get(), d_ctr);
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
    for (int it = 0; it < iters; ++it) {
        assign_device<T>(ctx, X, N, d, d_ctr, k, d_assign);
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
        for (int c = 0; c < k; ++c) {
            if (h_counts[c] != 0) continue;
            farthest_partial_kernel<T><<<fparts, 256, 0, s>>>(X, N, d, d_ctr, d_assign, counts.get(), pval.get(), pidx.get());
            reseed_apply_kernel<T><<<1, 128, 0, s>>>(X, d, pval.get(), pidx.get(), fparts, d_ctr, d_assign, counts.get(), c);
            LAUNCH_OK("reseed");
        }
    }
    assign_device<T>(ctx, X, N, d, d_ctr, k, d_assign);
}

#define LCNB_INST(T)                                                                                    \
    template void kmeans_pp_device<T>(Ctx&, const T*, long long, int, int, uint64_t,                    \
                                      const std::vector<unsigned long long>&, uint32_t*, int*);         \
    template void assign_device<T>(Ctx&, const T*, long long, int, const double*, int, uint32_t*);      \
    template void lloyd_device<T>(Ctx&, const T*, long long, int, int, int, uint64_t, double*, uint32_t*);
LCNB_INST(double)
LCNB_INST(float)
#undef LCNB_INST

}  // namespace lcnb
