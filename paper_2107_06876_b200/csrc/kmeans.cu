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

#include <random>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "kmeans.cuh"
#include "tiles.cuh"

namespace lcnb {

// ---- assign_nearest (kmeans.cpp:67-85) -------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) assign_exact_kernel(const T* __restrict__ X, long long N, int d,
                                                           const double* __restrict__ Cm, int k,
                                                           uint32_t* __restrict__ out, double* __restrict__ best_out) {
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
            load_slab<T>(As, X, nullptr, p0, N, d, k0);
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
            out[p] = static_cast<uint32_t>(a);
            if (best_out) best_out[p] = b;
        }
    }
}

// ---- k-means++ (kmeans.cpp:23-65) ------------------------------------------
// dist2[i] = min(dist2[i], sqdist(x_i, x_last)), strict < as kmeans.cpp:38.
template <typename T>
__global__ void __launch_bounds__(256) pp_update_kernel(const T* __restrict__ X, long long N, int d,
                                                        const uint32_t* __restrict__ chosen, int t,
                                                        double* __restrict__ dist2) {
    __shared__ double As[KC][TP + 1];
    __shared__ double Cs[KC];
    const long long p0 = static_cast<long long>(blockIdx.x) * TP;
    const long long last = chosen[t];
    // 4 threads per point would break the sequential fold; one thread folds
    // one point, slabs staged for coalescing.
    double acc = 0.0;
    const int r = threadIdx.x;  // blockDim = 64
    for (int k0 = 0; k0 < d; k0 += KC) {
        load_slab<T>(As, X, nullptr, p0, N, d, k0);
        if (threadIdx.x < KC) Cs[threadIdx.x] = k0 + threadIdx.x < d ? static_cast<double>(X[last * d + k0 + threadIdx.x]) : 0.0;
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            double df = xsub(As[kk][r], Cs[kk]);
            acc = xadd(acc, xmul(df, df));
        }
        __syncthreads();
    }
    long long p = p0 + r;
    if (p < N && acc < dist2[p]) dist2[p] = acc;
}

// Exact emulation of the sequential fp64 fold s_{i+1} = fl(s_i + x_i) by one
// warp, 32 elements at a time. While s is a normal number in the binade
// [2^e, 2^(e+1)) its grid is u = 2^(e-52) and fl(s + x) = s + u * RN(x/u)
// (x >= 0); the per-lane integers RN(x/u) are prefix-summed exactly in int64.
// A lane leaves the fast path when its rounding is a tie (parity-dependent),
// when x/u is huge, or when the running sum would reach 2^(e+1); that element
// is added with a real fp64 add and the binade is recomputed.
// With search, also returns the first index whose running sum is >= target
// and whose element is > 0 (kmeans.cpp:51-58).
struct FoldResult {
    double s;
    long long pick;
};

constexpr double kMinNormal = 2.2250738585072014e-308;
constexpr long long kTwo53 = 1LL << 53;

__device__ FoldResult warp_exact_fold(const double* __restrict__ x, long long begin, long long end, double s,
                                      bool search, double target) {
    const int lane = threadIdx.x & 31;
    long long pick = -1;
    for (long long base = begin; base < end; base += 32) {
        const int cnt = static_cast<int>(min(32LL, end - base));
        const double v = lane < cnt ? x[base + lane] : 0.0;
        int a = 0;
        while (a < cnt) {
            if (!(s >= kMinNormal && s < kPosInf)) {  // zero / subnormal / inf: real add
                double va = __shfl_sync(0xffffffffu, v, a);
                s = xadd(s, va);
                if (search && pick < 0 && s >= target && va > 0.0) pick = base + a;
                ++a;
                continue;
            }
            const int e = ilogb(s);
            const long long S = static_cast<long long>(scalbn(s, 52 - e));
            const bool mine = lane >= a && lane < cnt;
            double q = mine ? scalbn(v, 52 - e) : 0.0;
            const bool big = !(q < 9007199254740992.0);
            long long r = 0;
            bool tie = false;
            if (mine && !big) {
                double K = floor(q), f = q - K;
                r = static_cast<long long>(K) + (f > 0.5 ? 1 : 0);
                tie = (f == 0.5);
            } else if (big) {
                r = kTwo53;
            }
            long long P = r;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                long long t = __shfl_up_sync(0xffffffffu, P, o);
                if (lane >= o) P += t;
            }
            const bool bad = mine && (big || tie || S + P >= kTwo53);
            const unsigned bm = __ballot_sync(0xffffffffu, bad);
            const int fb = bm ? __ffs(bm) - 1 : cnt;
            if (search && pick < 0) {
                bool hit = false;
                if (lane >= a && lane < fb) hit = scalbn(static_cast<double>(S + P), e - 52) >= target && v > 0.0;
                const unsigned hm = __ballot_sync(0xffffffffu, hit);
                if (hm) pick = base + __ffs(hm) - 1;
            }
            const long long Pacc = fb > a ? __shfl_sync(0xffffffffu, P, fb - 1) : 0;
            s = scalbn(static_cast<double>(S + Pacc), e - 52);
            if (fb < cnt) {
                double vb = __shfl_sync(0xffffffffu, v, fb);
                s = xadd(s, vb);
                if (search && pick < 0 && s >= target && vb > 0.0) pick = base + fb;
                a = fb + 1;
            } else {
                a = cnt;
            }
        }
        if (search && pick >= 0) break;
    }
    return {s, pick};
}

// ---- chunk-parallel exact fold ----------------------------------------------
// The fold over N values is cut into chunks of kFoldChunk. Most chunks lie
// inside one binade of the running sum, where the fold's result depends only
// on that binade: S_end = S_start + u_e * sum_j RN(x_j / u_e). So
//   A) approximate chunk sums (any order)            -> predicted start A_c
//   B) predicted binade e_c of each chunk (dirty if the interval
//      [A_c (1-1e-9), A_{c+1} (1+1e-9)] straddles a power of two)
//   C) integer rounding sums R_c(e_c) in parallel, dirty on ties / huge x
//   D) one warp walks the chunks in order with the exact running sum: a clean
//      chunk whose actual binade matches e_c advances by u * R_c exactly,
//      any other chunk is folded element-wise by warp_exact_fold.
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

__global__ void fold_round_kernel(const double* __restrict__ x, long long N, const int* __restrict__ ebin,
                                  long long* __restrict__ R) {
    __shared__ long long red[8];
    __shared__ int bad_any;
    const int e = ebin[blockIdx.x];
    if (e == -100000) {
        if (threadIdx.x == 0) R[blockIdx.x] = -1;
        return;
    }
    if (threadIdx.x == 0) bad_any = 0;
    __syncthreads();
    const long long b = static_cast<long long>(blockIdx.x) * kFoldChunk;
    const long long en = min(N, b + kFoldChunk);
    long long r = 0;
    bool bad = false;
    for (long long i = b + threadIdx.x; i < en; i += blockDim.x) {
        double q = scalbn(x[i], 52 - e);
        if (!(q < 9007199254740992.0)) { bad = true; continue; }
        double K = floor(q), f = q - K;
        if (f == 0.5) bad = true;
        r += static_cast<long long>(K) + (f > 0.5 ? 1 : 0);
    }
    if (bad) bad_any = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        R[blockIdx.x] = bad_any ? -1 : t;
    }
}

// D) walk + draw + pick for k-means++ step t (kmeans.cpp:35-62). raw[] holds
// the caller's engine draws in order; a step with total <= 0 consumes none
// (kmeans.cpp:42-47).
__global__ void pp_walk_pick_kernel(double* __restrict__ dist2, unsigned char* __restrict__ used, long long N, int nch,
                                    const int* __restrict__ ebin, const long long* __restrict__ R,
                                    double* __restrict__ sstart, const unsigned long long* __restrict__ raw, int n_raw,
                                    int* __restrict__ draw_counter, uint32_t* __restrict__ chosen, int t) {
    const int lane = threadIdx.x;
    double S = 0.0;
    for (int cb = 0; cb < nch; cb += 32) {
        const int c_l = cb + lane;
        const int e_l = c_l < nch ? ebin[c_l] : 0;
        const long long r_l = c_l < nch ? R[c_l] : -1;
        const int cnt = min(32, nch - cb);
        for (int k = 0; k < cnt; ++k) {
            const int c = cb + k;
            if (lane == 0) sstart[c] = S;
            const int e = __shfl_sync(0xffffffffu, e_l, k);
            const long long Rc = __shfl_sync(0xffffffffu, r_l, k);
            bool fast = Rc >= 0 && S >= kMinNormal && S < kPosInf && ilogb(S) == e;
            long long Si = 0;
            if (fast) {
                Si = static_cast<long long>(scalbn(S, 52 - e));
                fast = Si + Rc < kTwo53;
            }
            if (fast) {
                S = scalbn(static_cast<double>(Si + Rc), e - 52);
            } else {
                const long long b = static_cast<long long>(c) * kFoldChunk;
                S = warp_exact_fold(dist2, b, min(N, b + kFoldChunk), S, false, 0.0).s;
            }
        }
    }
    if (lane == 0) sstart[nch] = S;
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
        // first chunk whose running sum reaches the target (the sum is monotone)
        int cstar = nch;
        for (int cb = 0; cb < nch; cb += 32) {
            const int c_l = cb + lane;
            const bool hit = c_l < nch && sstart[c_l + 1] >= target;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) { cstar = cb + __ffs(m) - 1; break; }
        }
        pick = -1;
        if (cstar < nch) {
            FoldResult sr = warp_exact_fold(dist2, static_cast<long long>(cstar) * kFoldChunk, N, sstart[cstar], true, target);
            pick = sr.pick;
        }
        if (pick < 0) pick = N - 1;
        if (lane == 0) *draw_counter = di + 1;
    }
    __syncwarp();
    if (lane == 0) {
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
    DevBuf<long long> R(nch);
    DevBuf<unsigned char> used(N);
    DevBuf<unsigned long long> d_raw(raw.size() ? raw.size() : 1);
    DevBuf<int> counter(1);
    used.zero(s);
    counter.zero(s);
    if (!raw.empty()) d_raw.upload(raw.data(), raw.size(), s);
    fill_kernel<<<ceil_div(N, 256), 256, 0, s>>>(dist2.get(), N, kPosInf);
    uint32_t f32 = static_cast<uint32_t>(first);
    unsigned char one = 1;
    CUDA_OK(cudaMemcpyAsync(d_chosen, &f32, 4, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(used.get() + first, &one, 1, cudaMemcpyHostToDevice, s));
    for (int t = 1; t < k; ++t) {
        pp_update_kernel<T><<<ceil_div(N, TP), TP, 0, s>>>(X, N, d, d_chosen, t - 1, dist2.get());
        fold_chunk_sum_kernel<<<nch, 256, 0, s>>>(dist2.get(), N, csum.get());
        fold_plan_kernel<<<1, 1024, 0, s>>>(csum.get(), nch, ebin.get());
        fold_round_kernel<<<nch, 256, 0, s>>>(dist2.get(), N, ebin.get(), R.get());
        pp_walk_pick_kernel<<<1, 32, 0, s>>>(dist2.get(), used.get(), N, nch, ebin.get(), R.get(), sstart.get(),
                                             d_raw.get(), static_cast<int>(raw.size()), counter.get(), d_chosen, t);
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
        for (int p = 0; p < cnt; ++p) s = xadd(s, static_cast<double>(X[static_cast<long long>(order[b + p]) * d + kk]));
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

template <typename T>
void assign_device(Ctx& ctx, const T* X, long long N, int d, const double* C, int k, uint32_t* out) {
    if (N == 0) return;
    assign_exact_kernel<T><<<ceil_div(N, TP), 256, 0, ctx.stream>>>(X, N, d, C, k, out, nullptr);
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
    kmeans_pp_device<T>(ctx, X, N, d, k, f, raw, init.get(), nullptr);
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
