// Batched small LCN problems (configs[4]): many
// independent problems of a few hundred points, one CTA per problem, the
// whole pipeline in two ragged launches:
//
//   bat_kmeans_kernel  per problem: k-means LSH of the union (1 band,
//                      lsh.cpp:245-283 -> lloyd, kmeans.cpp:23-143) and the
//                      k-means landmarks (select_landmarks, nystrom.cpp:28-48),
//                      both bit-exact to the reference (the same sequential
//                      fp64 folds, the caller engine's draws), then the
//                      landmark kernel matrix A (nystrom.cpp:88-93)
//   host               per problem: the long-double LDL^T of A + jitter (the
//                      reference's own precision, nystrom.cpp:99-124) ->
//                      A_j^-1 (10 x 10), shared with the big path
//   bat_solve_kernel   per problem: U, V (kernel_block, nystrom.cpp:52-64),
//                      W = A_j^-1 V with the reference's residual test
//                      (a failing problem goes back to the host for the next
//                      jitter level), K_sp and delta on the bucket blocks
//                      (sparse_kernel.cpp:51-117), the log-stabilised LCN
//                      Sinkhorn loop (sinkhorn.cpp:104-188 over
//                      operator.cpp:123-224) and the distance (sinkhorn.cpp:178-183)
//
// Points stay in global memory (L1-resident per CTA); the per-problem
// vectors live in shared memory; U, V/W and delta in a per-problem global
// scratch. Error behaviour per problem: the status of the reference's first
// throw (NegativeKernelError, StabilizationError, FactorizationError).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <optional>
#include <random>

#include "common.cuh"
#include "ctx.cuh"
#include "kmeans.cuh"
#include "op.cuh"

namespace lcnb {
namespace {

constexpr int kBT = 256;        // threads per problem CTA (solve)
constexpr int kKT = 128;        // threads per problem CTA (k-means: several CTAs per SM hide the serial folds)
constexpr int kBMaxK = 16;      // clusters / landmarks per problem
constexpr int kBMaxD = 32;      // features
constexpr int kBMaxN = 1024;    // points per problem (n + m)
constexpr int kNeedJitter = 50; // status: residual test failed at this jitter level

struct BatProb {
    long long nnz;         // support size (sum over buckets of n_b m_b)
    long long row0;        // first row of the problem in X (n sources, then m targets)
    int n, m;
    uint32_t lsh_first, lm_first;  // k-means++ first indices (host engine)
    long long lsh_raw, lm_raw;     // offsets of the engine's raw draws
    long long scr;                 // scratch offset (doubles): U n x l, V l x m, W l x m, delta nnz
};

__device__ __forceinline__ long long s_nnz_of(const BatProb& p) { return p.nnz; }

// sqdist with the reference's separate roundings (kmeans.cpp:12-19)
__device__ __forceinline__ double bat_sqdist(const double* __restrict__ x, const double* __restrict__ y, int d) {
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < d; ++k) {
        const double df = xsub(x[k], y[k]);
        s = xadd(s, xmul(df, df));
    }
    return s;
}

// the same fold with the point held in registers (DP >= d, predicated): the
// hot loops of the k-means compare one point against many centres
template <int DP>
__device__ __forceinline__ void bat_load(const double* __restrict__ x, int d, double (&v)[DP]) {
#pragma unroll
    for (int k = 0; k < DP; ++k) v[k] = k < d ? x[k] : 0.0;
}
template <int DP>
__device__ __forceinline__ double bat_sqdist_reg(const double (&v)[DP], const double* __restrict__ y, int d) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < DP; ++k)
        if (k < d) {
            const double df = xsub(v[k], y[k]);
            s = xadd(s, xmul(df, df));
        }
    return s;
}

// cost_value (geometry.cpp:45-76) for the kinds this path takes
__device__ __forceinline__ double bat_cost(int kind, const double* x, const double* y, int d) {
    const double s = bat_sqdist(x, y, d);
    return kind == 0 ? __dsqrt_rn(s) : s;
}

struct BatKm {  // one lloyd call, shared memory
    double* dist2;    // N
    double* prefix;   // N
    uint32_t* assign; // N
    uint32_t* order;  // N: members grouped by cluster, point order inside
    double* ctr;      // k x d
    double* sums;     // k x d
    int* counts;      // k
    int* start;       // k + 1
    uint32_t* chosen; // k
};

// kmeans_pp_indices (kmeans.cpp:23-65): first = the engine's first index,
// raw = its later 64-bit draws (one per step with total > 0).
template <int DP>
__device__ void cta_kmeanspp(const double* __restrict__ X, int N, int d, int k, uint32_t first,
                             const unsigned long long* __restrict__ raw, BatKm& s) {
    __shared__ double target_s;
    __shared__ int pick_s, mode_s;
    const int tid = threadIdx.x;
    for (int i = tid; i < N; i += kKT) s.dist2[i] = kPosInf;
    if (tid == 0) s.chosen[0] = first;
    __syncthreads();
    int draw = 0;
    for (int t = 1; t < k; ++t) {
        const double* last = X + static_cast<long long>(s.chosen[t - 1]) * d;
        double lv[DP];
        bat_load<DP>(last, d, lv);
        for (int i = tid; i < N; i += kKT) {
            const double d2 = bat_sqdist_reg<DP>(lv, X + static_cast<long long>(i) * d, d);  // same fold (x - y)^2
            if (d2 < s.dist2[i]) s.dist2[i] = d2;
        }
        __syncthreads();
        if (tid == 0) {
            double total = 0.0;  // left fold in index order (kmeans.cpp:39)
            for (int i = 0; i < N; ++i) s.prefix[i] = total = xadd(total, s.dist2[i]);
            if (total <= 0.0) {
                mode_s = 0;
            } else {
                // uniform_real_distribution(0, total): generate_canonical = u 2^-64,
                // clamped below 1; (b - a) c + a (kmeans.cpp:49-50)
                double c = __ull2double_rn(raw[draw++]) * 5.421010862427522e-20;
                if (c >= 1.0) c = 0.99999999999999989;
                target_s = xadd(xmul(c, xsub(total, 0.0)), 0.0);
                mode_s = 1;
            }
            pick_s = N;
        }
        __syncthreads();
        if (mode_s == 1) {
            // first i with running sum >= target and dist2 > 0 (kmeans.cpp:51-58)
            const double target = target_s;
            for (int i = tid; i < N; i += kKT)
                if (s.prefix[i] >= target && s.dist2[i] > 0.0) {
                    atomicMin(&pick_s, i);
                    break;
                }
        } else {
            // first unused index (kmeans.cpp:42-47), no draw
            for (int i = tid; i < N; i += kKT) {
                bool used = false;
                for (int c = 0; c < t; ++c) used |= s.chosen[c] == static_cast<uint32_t>(i);
                if (!used) {
                    atomicMin(&pick_s, i);
                    break;
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            const int pick = pick_s < N ? pick_s : N - 1;
            s.chosen[t] = static_cast<uint32_t>(pick);
            s.dist2[pick] = 0.0;
        }
        __syncthreads();
    }
}

// assign_nearest (kmeans.cpp:67-85): strict < over c = 0..k-1
template <int DP>
__device__ void cta_assign(const double* __restrict__ X, int N, int d, int k, BatKm& s) {
    for (int i = threadIdx.x; i < N; i += kKT) {
        double xv[DP];
        bat_load<DP>(X + static_cast<long long>(i) * d, d, xv);
        double best = kPosInf;
        uint32_t arg = 0;
        for (int c = 0; c < k; ++c) {
            const double d2 = bat_sqdist_reg<DP>(xv, s.ctr + c * d, d);
            if (d2 < best) {
                best = d2;
                arg = static_cast<uint32_t>(c);
            }
        }
        s.assign[i] = arg;
    }
    __syncthreads();
}

// lloyd (kmeans.cpp:87-143)
template <int DP>
__device__ void cta_lloyd(const double* __restrict__ X, int N, int d, int k, int iters, uint32_t first,
                          const unsigned long long* __restrict__ raw, BatKm& s) {
    const int tid = threadIdx.x;
    cta_kmeanspp<DP>(X, N, d, k, first, raw, s);
    for (int e = tid; e < k * d; e += kKT) s.ctr[e] = X[static_cast<long long>(s.chosen[e / d]) * d + e % d];
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        cta_assign<DP>(X, N, d, k, s);
        for (int c = tid; c < k; c += kKT) s.counts[c] = 0;
        __syncthreads();
        for (int i = tid; i < N; i += kKT) atomicAdd(&s.counts[s.assign[i]], 1);
        __syncthreads();
        if (tid < 32) {
            // members of each cluster in point order: a stable partition,
            // 32 points at a time (lanes of a cluster ranked by lane)
            if (tid == 0) {
                int acc = 0;
                for (int c = 0; c < k; ++c) {
                    s.start[c] = acc;
                    acc += s.counts[c];
                }
                s.start[k] = acc;
            }
            __syncwarp();
            int cur = tid < k ? s.start[tid] : 0;  // lane c: next slot of cluster c
            for (int b0 = 0; b0 < N; b0 += 32) {
                const int i = b0 + tid;
                const uint32_t c = i < N ? s.assign[i] : 0xffffffffu;
                const unsigned grp = __match_any_sync(0xffffffffu, c);
                const int base = __shfl_sync(0xffffffffu, cur, static_cast<int>(c < 32 ? c : 0));
                if (i < N) s.order[base + __popc(grp & ((1u << tid) - 1u))] = static_cast<uint32_t>(i);
                // advance each cluster's cursor by its members in this chunk
                for (int cc = 0; cc < k; ++cc) {
                    const unsigned mc = __ballot_sync(0xffffffffu, c == static_cast<uint32_t>(cc));
                    if (tid == cc) cur += __popc(mc);
                }
            }
        }
        __syncthreads();
        // sums in point order per (cluster, feature), then s * (1 / count)
        // (kmeans.cpp:106-121)
        for (int e = tid; e < k * d; e += kKT) {
            const int c = e / d, kk = e % d;
            if (s.counts[c] == 0) continue;
            double acc = 0.0;
            for (int r = s.start[c]; r < s.start[c + 1]; ++r)
                acc = xadd(acc, X[static_cast<long long>(s.order[r]) * d + kk]);
            s.sums[e] = xmul(acc, __ddiv_rn(1.0, static_cast<double>(s.counts[c])));
        }
        __syncthreads();
        for (int e = tid; e < k * d; e += kKT)
            if (s.counts[e / d] != 0) s.ctr[e] = s.sums[e];
        __syncthreads();
        if (tid == 0) {  // empty clusters: the farthest point, first max (kmeans.cpp:122-139)
            for (int c = 0; c < k; ++c) {
                if (s.counts[c] != 0) continue;
                double far = -1.0;
                int arg = 0;
                for (int i = 0; i < N; ++i) {
                    if (s.counts[s.assign[i]] <= 1) continue;
                    const double d2 = bat_sqdist(X + static_cast<long long>(i) * d, s.ctr + s.assign[i] * d, d);
                    if (d2 > far) {
                        far = d2;
                        arg = i;
                    }
                }
                for (int kk = 0; kk < d; ++kk) s.ctr[c * d + kk] = X[static_cast<long long>(arg) * d + kk];
                --s.counts[s.assign[arg]];
                s.assign[arg] = static_cast<uint32_t>(c);
                s.counts[c] = 1;
            }
        }
        __syncthreads();
    }
    cta_assign<DP>(X, N, d, k, s);
}

// Per problem: LSH bucket ids (k-means of the union, fn_seed(seed, 0, 0)),
// landmarks (k-means of the union, 10 iterations) and A = exp(-c(L, L) / lambda).
template <int DP>
__global__ void __launch_bounds__(kKT, 8) bat_kmeans_kernel(const double* __restrict__ X, int d,
                                                         const BatProb* __restrict__ probs,
                                                         const unsigned long long* __restrict__ raw, int buckets,
                                                         int kmeans_iters, int l, int kind, double lambda,
                                                         uint32_t* __restrict__ bucket_out,
                                                         double* __restrict__ lm_out, double* __restrict__ a_out,
                                                         unsigned long long* __restrict__ nnz_out) {
    extern __shared__ __align__(16) unsigned char bdyn[];
    const BatProb pr = probs[blockIdx.x];
    const int N = pr.n + pr.m;
    const double* Xp = X + pr.row0 * d;
    BatKm s;
    s.dist2 = reinterpret_cast<double*>(bdyn);
    s.prefix = s.dist2 + N;
    s.ctr = s.prefix + N;
    s.sums = s.ctr + kBMaxK * d;
    s.assign = reinterpret_cast<uint32_t*>(s.sums + kBMaxK * d);
    s.order = s.assign + N;
    s.counts = reinterpret_cast<int*>(s.order + N);
    s.start = s.counts + kBMaxK;
    s.chosen = reinterpret_cast<uint32_t*>(s.start + kBMaxK + 1);
    __shared__ int bcnt[2][kBMaxK];
    const int tid = threadIdx.x;

    // LSH: one band, one function (lsh.cpp:264-276)
    cta_lloyd<DP>(Xp, N, d, buckets, kmeans_iters, pr.lsh_first, raw + pr.lsh_raw, s);
    for (int i = tid; i < N; i += kKT) bucket_out[pr.row0 + i] = s.assign[i];
    if (tid < kBMaxK) bcnt[0][tid] = bcnt[1][tid] = 0;
    __syncthreads();
    for (int i = tid; i < N; i += kKT) atomicAdd(&bcnt[i < pr.n ? 0 : 1][s.assign[i]], 1);
    __syncthreads();
    if (tid == 0) {
        unsigned long long nnz = 0;
        for (int b = 0; b < buckets; ++b) nnz += static_cast<unsigned long long>(bcnt[0][b]) * bcnt[1][b];
        nnz_out[blockIdx.x] = nnz;
    }
    __syncthreads();

    // landmarks: lloyd(union, l, 10, seed) centroids (nystrom.cpp:35-37)
    cta_lloyd<DP>(Xp, N, d, l, 10, pr.lm_first, raw + pr.lm_raw, s);
    double* L = lm_out + static_cast<long long>(blockIdx.x) * l * d;
    for (int e = tid; e < l * d; e += kKT) L[e] = s.ctr[e];
    // A_ab = exp(-c(L_a, L_b) / lambda) (nystrom.cpp:88-93: division)
    double* A = a_out + static_cast<long long>(blockIdx.x) * l * l;
    for (int e = tid; e < l * l; e += kKT)
        A[e] = exp(-bat_cost(kind, s.ctr + (e / l) * d, s.ctr + (e % l) * d, d) / lambda);
}

// ---- solve ------------------------------------------------------------------
struct BatSolveSmem {
    double *log_s, *log_t, *kt, *kt2, *tt, *rowm;  // vectors
    int *p_ord, *q_ord, *p_rank, *q_rank;    // sources / targets grouped by bucket, rank inside
    int *p_start, *q_start;                  // bucket offsets (buckets + 1)
    unsigned long long* blk;                 // delta block offsets (buckets + 1)
};

__device__ __forceinline__ double block_max(double v, double* red) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < kBT / 32; ++w) r = fmax(r, red[w]);
    return r;
}
__device__ __forceinline__ bool block_any(bool v, int* flag) {
    __syncthreads();
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    if (v) *flag = 1;
    __syncthreads();
    return *flag != 0;
}
// l sums over the block (thread partials v[0..l)), returned in out[0..l)
__device__ __forceinline__ void block_sums(double* v, int l, double* red, double* out) {
    __syncthreads();
    for (int a = 0; a < l; ++a) {
        double x = v[a];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) red[a * (kBT / 32) + (threadIdx.x >> 5)] = x;
    }
    __syncthreads();
    if (threadIdx.x < l) {
        double x = 0.0;
        for (int w = 0; w < kBT / 32; ++w) x += red[threadIdx.x * (kBT / 32) + w];
        out[threadIdx.x] = x;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kBT, 4) bat_solve_kernel(
    const double* __restrict__ X, int d, const BatProb* __restrict__ probs, const int* __restrict__ todo,
    const uint32_t* __restrict__ bucket, const double* __restrict__ lm, const double* __restrict__ ainv,
    const double* __restrict__ aj, int buckets, int l, int kind, double lambda, int iters,
    double* __restrict__ scratch, double* __restrict__ dist_out, int* __restrict__ status_out,
    int* __restrict__ iters_out) {
    extern __shared__ __align__(16) unsigned char bdyn[];
    __shared__ double red[kBMaxK * (kBT / 32)];
    __shared__ double mid[kBMaxK];
    __shared__ int flag;
    const int pi = todo ? todo[blockIdx.x] : static_cast<int>(blockIdx.x);
    const BatProb pr = probs[pi];
    const int n = pr.n, m = pr.m, N = n + m, tid = threadIdx.x;
    const double* P = X + pr.row0 * d;
    const double* Q = P + static_cast<long long>(n) * d;
    const uint32_t* bk = bucket + pr.row0;
    const double* L = lm + static_cast<long long>(pi) * l * d;
    const double* Ai = ainv + static_cast<long long>(pi) * l * l;
    const double* Aj = aj + static_cast<long long>(pi) * l * l;
    double* U = scratch + pr.scr;            // n x l
    double* V = U + static_cast<long long>(n) * l;  // l x m
    double* W = V + static_cast<long long>(l) * m;  // l x m
    double* D = W + static_cast<long long>(l) * m;  // delta, bucket blocks row-major
    double* DT = D + s_nnz_of(pr);                  // delta, bucket blocks transposed (column pass)
    BatSolveSmem s;
    s.log_s = reinterpret_cast<double*>(bdyn);
    s.log_t = s.log_s + n;
    s.kt = s.log_t + m;
    s.kt2 = s.kt + n;
    s.tt = s.kt2 + m;
    s.rowm = s.tt + std::max(n, m);
    s.blk = reinterpret_cast<unsigned long long*>(s.rowm + n);
    s.p_ord = reinterpret_cast<int*>(s.blk + buckets + 1);
    s.q_ord = s.p_ord + n;
    s.p_rank = s.q_ord + m;
    s.q_rank = s.p_rank + n;
    s.p_start = s.q_rank + m;
    s.q_start = s.p_start + buckets + 1;
    const double inv = 1.0 / lambda;
    auto fail = [&](int st) {
        if (tid == 0) {
            status_out[pi] = st;
            dist_out[pi] = std::numeric_limits<double>::quiet_NaN();
        }
    };

    // bucket layout: sources / targets grouped by bucket in point order
    if (tid == 0) {
        for (int b = 0; b <= buckets; ++b) s.p_start[b] = s.q_start[b] = 0;
        for (int i = 0; i < n; ++i) ++s.p_start[bk[i] + 1];
        for (int j = 0; j < m; ++j) ++s.q_start[bk[n + j] + 1];
        for (int b = 0; b < buckets; ++b) {
            s.p_start[b + 1] += s.p_start[b];
            s.q_start[b + 1] += s.q_start[b];
        }
        unsigned long long off = 0;
        for (int b = 0; b < buckets; ++b) {
            s.blk[b] = off;
            off += static_cast<unsigned long long>(s.p_start[b + 1] - s.p_start[b]) * (s.q_start[b + 1] - s.q_start[b]);
        }
        s.blk[buckets] = off;
        for (int b = 0; b < buckets; ++b) {  // cursors in p_rank / q_rank (reused)
            s.p_rank[b] = s.p_start[b];
            s.q_rank[b] = s.q_start[b];
        }
        for (int i = 0; i < n; ++i) s.p_ord[s.p_rank[bk[i]]++] = i;
        for (int j = 0; j < m; ++j) s.q_ord[s.q_rank[bk[n + j]]++] = j;
        for (int b = 0; b < buckets; ++b) {
            for (int r = s.p_start[b]; r < s.p_start[b + 1]; ++r) s.p_rank[s.p_ord[r]] = r - s.p_start[b];
            for (int r = s.q_start[b]; r < s.q_start[b + 1]; ++r) s.q_rank[s.q_ord[r]] = r - s.q_start[b];
        }
    }
    // U = exp(-c(p, L) * (1 / lambda)), V = exp(-c(L, q) * (1 / lambda)) (nystrom.cpp:52-64)
    for (int e = tid; e < n * l; e += kBT)
        U[e] = exp(-bat_cost(kind, P + static_cast<long long>(e / l) * d, L + (e % l) * d, d) * inv);
    double vmax = 0.0;
    for (int e = tid; e < l * m; e += kBT) {
        V[e] = exp(-bat_cost(kind, L + (e / m) * d, Q + static_cast<long long>(e % m) * d, d) * inv);
        vmax = fmax(vmax, fabs(V[e]));
    }
    vmax = block_max(vmax, red);
    // W = A_j^-1 V and the residual max |A_j W - V| <= 1e-6 max(max|V|, 1e-300) (nystrom.cpp:110-112)
    bool bad = false;
    for (int e = tid; e < l * m; e += kBT) {
        const int a = e / m, j = e % m;
        double w = 0.0;
        for (int b = 0; b < l; ++b) w += Ai[a * l + b] * V[b * m + j];
        W[e] = w;
        bad |= !isfinite(w);
    }
    __syncthreads();
    double resid = 0.0;
    for (int e = tid; e < l * m; e += kBT) {
        const int a = e / m, j = e % m;
        double r = -V[e];
        for (int b = 0; b < l; ++b) r += Aj[a * l + b] * W[b * m + j];
        resid = fmax(resid, fabs(r));
    }
    resid = block_max(resid, red);
    if (block_any(bad, &flag) || !(resid <= 1e-6 * fmax(vmax, 1e-300))) {
        fail(kNeedJitter);
        return;
    }
    // K_sp (log K = 0 - c * (1 / lambda), sparse_kernel.cpp:71-77) and
    // delta = exp(log K) - (U W)_ij on the support (sparse_kernel.cpp:96-110)
    bool over = false;
    for (int b = 0; b < buckets; ++b) {
        const int nb = s.p_start[b + 1] - s.p_start[b], mb = s.q_start[b + 1] - s.q_start[b];
        for (int e = tid; e < nb * mb; e += kBT) {
            const int i = s.p_ord[s.p_start[b] + e / mb], j = s.q_ord[s.q_start[b] + e % mb];
            const double lk = 0.0 - bat_cost(kind, P + static_cast<long long>(i) * d, Q + static_cast<long long>(j) * d, d) * inv;
            const double ex = exp(lk);
            if (isinf(ex)) over = true;
            double nys = 0.0;
            for (int a = 0; a < l; ++a) nys += U[i * l + a] * W[a * m + j];
            D[s.blk[b] + e] = ex - nys;
            DT[s.blk[b] + static_cast<long long>(e % mb) * nb + e / mb] = ex - nys;
        }
    }
    if (block_any(over, &flag)) {
        fail(3);  // StabilizationError: kernel value overflows linear space
        return;
    }

    // ---- Sinkhorn (sinkhorn.cpp:104-188), uniform marginals, tol 0 ----------
    // Every check the reference makes (non-finite log scalings, zero linear
    // scalings, non-positive Nystrom / LCN row sums, an exact fixed point)
    // goes into per-pass flags that are read at the barriers the data flow
    // needs anyway: five barriers per half-iteration.
    const double lp = log(1.0 / n), lq = log(1.0 / m);
    __shared__ int f_nf, f_zero, f_nys, f_neg, f_ne;
    // one LCN log matvec (operator.cpp:148-176): in[len_in] are log scalings,
    // out[len_out] = hi + log(Fo mid + delta tt), mid = Fi^T tt, tt = exp(in - hi).
    // src: when given, in[k] = base - src[k] is formed on the fly (the
    // s-update / t-update of sinkhorn.cpp:151-156) and checked for finiteness.
    auto pass = [&](double* in, const double* src, double base, int len_in, int len_out, const double* Fi,
                    int fi_rs, int fi_cs, const double* Fo, int fo_rs, int fo_cs, const double* Dm, bool rows,
                    double* out) -> int {
        if (tid == 0) f_nf = f_zero = f_nys = f_neg = 0;
        double hi = -kPosInf;
        bool nf = false;
        for (int k2 = tid; k2 < len_in; k2 += kBT) {
            double v = in[k2];
            if (src) {
                v = base - src[k2];
                in[k2] = v;
                nf |= !isfinite(v);
            }
            hi = fmax(hi, v);
        }
        if (nf) f_nf = 1;
        hi = block_max(hi, red);  // 2 barriers
        if (f_nf) return 3;       // StabilizationError: non-finite scaling
        bool zero = false;
        for (int k2 = tid; k2 < len_in; k2 += kBT) {
            const double t = exp(in[k2] - hi);
            s.tt[k2] = t;
            zero |= !(t > 0.0);
        }
        if (zero) f_zero = 1;
        __syncthreads();  // 1 barrier: tt complete
        // mid_a = sum_k Fi(k, a) tt_k: warp w owns landmarks a = w, w + 8, ...
        for (int a = tid >> 5; a < l; a += kBT / 32) {
            double acc = 0.0;
            for (int k2 = tid & 31; k2 < len_in; k2 += 32)
                acc += Fi[static_cast<long long>(k2) * fi_rs + a * fi_cs] * s.tt[k2];
            acc = warp_sum(acc);
            if ((tid & 31) == 0) mid[a] = acc;
        }
        __syncthreads();  // 1 barrier: mid complete
        bool nys = false, neg = false;
        for (int o = tid; o < len_out; o += kBT) {
            double y = 0.0;
            for (int a = 0; a < l; ++a) y += Fo[static_cast<long long>(o) * fo_rs + a * fo_cs] * mid[a];
            nys |= !(y > 0.0);  // nys_matvec (nystrom.cpp:157-160) when every tt > 0
            const int b = rows ? bk[o] : bk[n + o];
            const int ob = rows ? s.q_start[b] : s.p_start[b];
            const int nbk = (rows ? s.q_start[b + 1] : s.p_start[b + 1]) - ob;
            const int* ord = rows ? s.q_ord : s.p_ord;
            const double* Dr = Dm + s.blk[b] + static_cast<long long>(rows ? s.p_rank[o] : s.q_rank[o]) * nbk;
            double c = 0.0;
            for (int r = 0; r < nbk; ++r) c += Dr[r] * s.tt[ord[ob + r]];
            y += c;
            neg |= !(y > 0.0);
            out[o] = hi + log(y);
        }
        if (nys) f_nys = 1;
        if (neg) f_neg = 1;
        __syncthreads();  // 1 barrier: out complete, flags final
        if (f_neg || (f_nys && !f_zero)) return 4;  // NegativeKernelError
        return 0;
    };
    for (int j = tid; j < m; j += kBT) s.log_t[j] = 0.0;
    __syncthreads();
    // kt = log_matvec(log t = 0)
    int st = pass(s.log_t, nullptr, 0.0, m, n, W, 1, m, U, l, 1, D, true, s.kt);
    if (st) {
        fail(st);
        return;
    }
    int it = 0;
    while (it < iters) {
        ++it;
        // log s = log p - kt, then kts = log_matvec_t(log s)
        if ((st = pass(s.log_s, s.kt, lp, n, m, U, l, 1, W, 1, m, DT, false, s.kt2))) {
            fail(st);
            return;
        }
        // log t = log q - kts, then kt = log_matvec(log t)
        if ((st = pass(s.log_t, s.kt2, lq, m, n, W, 1, m, U, l, 1, D, true, s.kt))) {
            fail(st);
            return;
        }
        // err = sum |exp(log s + kt) - p| <= tol = 0 only at an exact fixed point
        if (tid == 0) f_ne = 0;
        __syncthreads();
        bool ne = false;
        for (int i = tid; i < n; i += kBT) ne |= exp(s.log_s[i] + s.kt[i]) != 1.0 / n;
        if (ne) f_ne = 1;
        __syncthreads();
        if (!f_ne) break;
    }
    for (int i = tid; i < n; i += kBT) s.rowm[i] = exp(s.log_s[i] + s.kt[i]);
    __syncthreads();
    // distance = lambda (<log s, P1> + <log t, q>) (sinkhorn.cpp:178-183)
    double acc = 0.0;
    for (int i = tid; i < n; i += kBT) acc += s.log_s[i] * s.rowm[i];
    for (int j = tid; j < m; j += kBT) acc += s.log_t[j] * (1.0 / m);
    acc = warp_sum(acc);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kBT / 32; ++w) t += red[w];
        mid[0] = t;
    }
    __syncthreads();
    if (tid == 0) {
        status_out[pi] = 0;
        dist_out[pi] = lambda * mid[0];
        iters_out[pi] = it;
    }
}

}  // namespace

// Host driver (see the file comment).
void batched_lcn(Ctx& ctx, const double* h_X, size_t rows, int d, int nprob, const int* h_n, const int* h_m,
                 int kind, double lambda, int buckets, int kmeans_iters, const uint64_t* lsh_seeds, int l,
                 const uint64_t* lm_seeds, int iters, double* dist_out, int* status_out, int* iters_out) {
    if (kind != 0 && kind != 3) throw Status(2, "batched LCN: cost must be euclidean or squared euclidean");
    if (d < 1 || d > kBMaxD) throw Status(2, "batched LCN: 1 <= d <= 32 on this path");
    if (buckets < 2 || buckets > kBMaxK || l < 1 || l > kBMaxK)
        throw Status(2, "batched LCN: buckets in [2, 16] and landmarks in [1, 16] on this path");
    if (!(lambda > 0.0)) throw Status(2, "build_factors: lambda must be positive");
    cudaStream_t s = ctx.stream;
    std::vector<BatProb> pr(nprob);
    // the caller engines' draws per problem (fixed slots: buckets - 1 for the
    // LSH k-means++, then l - 1 for the landmark one), independent problems
    const long long slot = static_cast<long long>(buckets - 1) + (l - 1);
    std::vector<unsigned long long> raw(std::max<long long>(static_cast<long long>(nprob) * slot, 1));
    long long row = 0;
    for (int k = 0; k < nprob; ++k) {
        const int N = h_n[k] + h_m[k];
        if (h_n[k] < 1 || h_m[k] < 1 || N > kBMaxN) throw Status(2, "batched LCN: 1 <= n, m and n + m <= 1024");
        if (buckets > N) throw Status(2, "hash_kmeans: more buckets than points");
        if (l > N) throw Status(2, "select_landmarks: l out of range");
        pr[k].row0 = row;
        pr[k].n = h_n[k];
        pr[k].m = h_m[k];
        row += N;
    }
#pragma omp parallel for schedule(static)
    for (int k = 0; k < nprob; ++k) {
        const int N = h_n[k] + h_m[k];
        auto draws = [&](uint64_t seed, int kk, uint32_t& first, long long off) {
            std::mt19937_64 rng(seed);
            std::uniform_int_distribution<std::size_t> fst(0, static_cast<std::size_t>(N - 1));
            first = static_cast<uint32_t>(fst(rng));
            for (int t = 0; t < kk - 1; ++t) raw[off + t] = rng();
        };
        pr[k].lsh_raw = static_cast<long long>(k) * slot;
        pr[k].lm_raw = pr[k].lsh_raw + (buckets - 1);
        draws(fn_seed(lsh_seeds[k], 0, 0), buckets, pr[k].lsh_first, pr[k].lsh_raw);
        draws(lm_seeds[k], l, pr[k].lm_first, pr[k].lm_raw);
    }
    if (static_cast<size_t>(row) != rows) throw Status(1, "batched LCN: row count does not match n + m totals");
    std::optional<PhaseTimer> pt;
    pt.emplace(ctx, "batched: upload");
    DevBuf<double> X(rows * d);
    X.upload(h_X, rows * d, s);
    DevBuf<unsigned long long> draws(std::max<size_t>(raw.size(), 1));
    if (!raw.empty()) draws.upload(raw.data(), raw.size(), s);
    DevBuf<BatProb> dprob(nprob);
    dprob.upload(pr.data(), nprob, s);
    DevBuf<uint32_t> bucket(rows);
    DevBuf<double> lm(static_cast<size_t>(nprob) * l * d), A(static_cast<size_t>(nprob) * l * l);
    DevBuf<unsigned long long> nnz(nprob);
    int maxN = 1;
    for (int k = 0; k < nprob; ++k) maxN = std::max(maxN, h_n[k] + h_m[k]);
    // shared memory sized by the batch's largest problem (more CTAs per SM)
    const size_t km_smem = static_cast<size_t>(maxN) * (8 + 8 + 4 + 4) + 2 * kBMaxK * static_cast<size_t>(d) * 8 +
                           (3 * kBMaxK + 2) * 4 + 64;
    auto kmk = d <= 16 ? bat_kmeans_kernel<16> : bat_kmeans_kernel<32>;
    allow_max_dyn_smem(kmk);
    pt.emplace(ctx, "batched: k-means LSH + landmarks (device)");
    kmk<<<nprob, kKT, km_smem, s>>>(X.get(), d, dprob.get(), draws.get(), buckets, kmeans_iters, l, kind, lambda,
                                    bucket.get(), lm.get(), A.get(), nnz.get());
    LAUNCH_OK("bat_kmeans_kernel");
    std::vector<double> hA(static_cast<size_t>(nprob) * l * l);
    std::vector<unsigned long long> hnnz(nprob);
    A.download(hA.data(), hA.size(), s);
    nnz.download(hnnz.data(), nprob, s);
    ctx.sync();
    long long scr = 0;
    for (int k = 0; k < nprob; ++k) {
        pr[k].scr = scr;
        pr[k].nnz = static_cast<long long>(hnnz[k]);
        scr += static_cast<long long>(pr[k].n) * l + 2LL * l * pr[k].m + 2LL * static_cast<long long>(hnnz[k]);
    }
    dprob.upload(pr.data(), nprob, s);
    DevBuf<double> scratch(std::max<long long>(scr, 1));
    DevBuf<double> dAinv(hA.size()), dAj(hA.size()), ddist(nprob);
    DevBuf<int> dstat(nprob), diters(nprob), dtodo(nprob);
    std::vector<double> hAinv(hA.size()), hAj(hA.size());
    std::vector<int> level(nprob, 0), todo(nprob), hstat(nprob, kNeedJitter);
    for (int k = 0; k < nprob; ++k) todo[k] = k;
    const size_t sv_smem = static_cast<size_t>(maxN) * 8 * 6 + (kBMaxK + 1) * 8 + static_cast<size_t>(maxN) * 8 +
                           (kBMaxK + 1) * 8 + 64;
    allow_max_dyn_smem(bat_solve_kernel);
    // jitter schedule rel = 0, 1e-10, then rel * 10 while <= 1.1e-4 (nystrom.cpp:99)
    std::vector<double> rels;
    for (double rel = 0.0; rel <= 1.1e-4; rel = (rel == 0.0 ? 1e-10 : rel * 10.0)) rels.push_back(rel);
    const int kLevels = static_cast<int>(rels.size());
    auto rel_of = [&](int lv) { return rels[lv]; };
    while (!todo.empty()) {
        pt.emplace(ctx, "batched: LDL^T + inverse (host, long double)");
        // host: LDL^T of A + rel * trace / l in long double, inverse (shared with the big path)
        std::vector<int> launch;
#pragma omp parallel for schedule(dynamic, 64)
        for (long long ii = 0; ii < static_cast<long long>(todo.size()); ++ii) {
            const int k = todo[ii];
            for (; level[k] < kLevels; ++level[k]) {
                if (nystrom_inverse_host(hA.data() + static_cast<size_t>(k) * l * l, l, rel_of(level[k]),
                                         hAinv.data() + static_cast<size_t>(k) * l * l,
                                         hAj.data() + static_cast<size_t>(k) * l * l))
                    break;
            }
        }
        for (int k : todo) {
            if (level[k] >= kLevels) hstat[k] = 5;  // FactorizationError
            else launch.push_back(k);
        }
        if (launch.empty()) break;
        pt.emplace(ctx, "batched: factors, correction, Sinkhorn (device)");
        dAinv.upload(hAinv.data(), hAinv.size(), s);
        dAj.upload(hAj.data(), hAj.size(), s);
        dtodo.upload(launch.data(), launch.size(), s);
        bat_solve_kernel<<<static_cast<unsigned>(launch.size()), kBT, sv_smem, s>>>(
            X.get(), d, dprob.get(), dtodo.get(), bucket.get(), lm.get(), dAinv.get(), dAj.get(), buckets, l, kind,
            lambda, iters, scratch.get(), ddist.get(), dstat.get(), diters.get());
        LAUNCH_OK("bat_solve_kernel");
        std::vector<int> st(nprob);
        dstat.download(st.data(), nprob, s);
        ctx.sync();
        todo.clear();
        for (int k : launch) {
            hstat[k] = st[k];
            if (st[k] == kNeedJitter) {
                ++level[k];
                todo.push_back(k);
            }
        }
    }
    pt.reset();
    ddist.download(dist_out, nprob, s);
    std::vector<int> it(nprob);
    diters.download(it.data(), nprob, s);
    ctx.sync();
    for (int k = 0; k < nprob; ++k) {
        status_out[k] = hstat[k] == kNeedJitter ? 5 : hstat[k];
        if (status_out[k]) dist_out[k] = std::numeric_limits<double>::quiet_NaN();
        if (iters_out) iters_out[k] = status_out[k] ? 0 : it[k];
    }
}

}  // namespace lcnb
