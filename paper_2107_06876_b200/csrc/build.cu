// Operator construction on the device:
//   * k-means LSH bucket ids (lsh.cpp:245-283 via lloyd_device);
//   * the bucket-blocked layout of K_sp: with k-means LSH
//     every within-bucket (source, target) pair is a neighbour
//     (lsh.cpp:222-239), so band b's support is the union of dense
//     n_bucket x m_bucket blocks; pairs already present in an earlier band are
//     masked (the sort+unique of NeighborPairs::from_pairs, lsh.cpp:163-177);
//   * K_sp values log K = 0 - c(x_i, y_j) * (1/lambda) (sparse_kernel.cpp:71-77);
//   * Nystrom factors U, A, V, W = A^-1 V (nystrom.cpp:53-125) with the
//     long-double factorisation and jitter schedule on the host and the
//     l x m products on the device;
//   * the LCN correction delta = exp(log K) - (U W)_ij at the support
//     (sparse_kernel.cpp:82-117).
#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cublas_v2.h>
#include <omp.h>
#include <cmath>
#include <limits>
#include <numeric>
#include <optional>
#include <functional>
#include <mutex>
#include <thread>
#include <exception>
#include <deque>
#include <random>

#include "kmeans.cuh"
#include "op.cuh"
#include "tc_block.cuh"
#include "tiles.cuh"

namespace lcnb {

PhaseTimer::PhaseTimer(Ctx& c, const char* n) : ctx(c), name(n), t0(0), on(std::getenv("LCN_TIMING") != nullptr) {
    if (on) {
        ctx.sync();
        t0 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
}
PhaseTimer::~PhaseTimer() {
    if (on) {
        cudaStreamSynchronize(ctx.stream);
        double t1 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
        std::fprintf(stderr, "[lcn timing] %-36s %10.2f ms", name, t1 - t0);
        if (ctx.filter_points)
            std::fprintf(stderr, "   (assign filter: %lld of %lld points to the exact scan)", ctx.filter_ambiguous,
                         ctx.filter_points);
        std::fprintf(stderr, "\n");
        ctx.filter_points = ctx.filter_ambiguous = 0;
    }
}

BandView Op::view(int b) const {
    const Band& B = bands[b];
    return {B.src_order.get(), B.tgt_order.get(), B.src_start.get(), B.tgt_start.get(), B.blk_off.get(),
            B.blkT_off.get(), B.src_bucket.get(), B.tgt_bucket.get(), B.src_local.get(), B.tgt_local.get(), B.src_pos.get(),
            B.tgt_pos.get()};
}

BandSet Op::bandset() const {
    BandSet s{};
    s.bands = static_cast<int>(bands.size());
    for (int b = 0; b < s.bands; ++b) {
        s.src_bucket[b] = bands[b].src_bucket.get();
        s.tgt_bucket[b] = bands[b].tgt_bucket.get();
    }
    return s;
}

// ---------------------------------------------------------------------------
// Band layout
// ---------------------------------------------------------------------------
namespace {

__global__ void hist_kernel(const uint32_t* __restrict__ ids, long long n, uint32_t* __restrict__ counts) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) atomicAdd(&counts[ids[i]], 1u);
}

__global__ void iota32_kernel(uint32_t* p, long long n) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) p[i] = static_cast<uint32_t>(i);
}

__global__ void local_pos_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ ids,
                                 const uint32_t* __restrict__ start, long long n, uint32_t* __restrict__ local,
                                 uint32_t* __restrict__ pos) {
    long long p = blockIdx.x * 256LL + threadIdx.x;
    if (p < n) {
        uint32_t i = order[p];
        local[i] = static_cast<uint32_t>(p - start[ids[i]]);
        pos[i] = static_cast<uint32_t>(p);
    }
}

// order / pos arrays carry 16 spare entries: the iteration kernels bulk-copy
// 16-byte-aligned supersets of their ranges.
void stable_group(Ctx& ctx, const uint32_t* d_ids, size_t n, size_t nb, DevBuf<uint32_t>& order,
                  DevBuf<uint32_t>& start, std::vector<uint32_t>& h_start, DevBuf<uint32_t>& local,
                  DevBuf<uint32_t>& pos) {
    cudaStream_t s = ctx.stream;
    order.resize(n + 16);
    order.zero(s);
    pos.resize(n + 16);
    pos.zero(s);
    local.resize(std::max<size_t>(n, 1));
    start.resize(nb + 1);
    DevBuf<uint32_t> counts(nb + 1), iota(std::max<size_t>(n, 1)), keys(std::max<size_t>(n, 1));
    counts.zero(s);
    if (n) {
        hist_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_ids, n, counts.get());
        iota32_kernel<<<ceil_div(n, 256), 256, 0, s>>>(iota.get(), n);
    }
    std::vector<uint32_t> h_counts(nb + 1);
    counts.download(h_counts.data(), nb, s);
    ctx.sync();
    h_start.assign(nb + 1, 0);
    for (size_t b = 0; b < nb; ++b) h_start[b + 1] = h_start[b] + h_counts[b];
    start.upload(h_start.data(), nb + 1, s);
    if (n) {
        int end_bit = 1;
        while ((1ull << end_bit) < nb) ++end_bit;
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, d_ids, keys.get(), iota.get(), order.get(), static_cast<int>(n),
                                        0, end_bit, s);
        DevBuf<unsigned char> t(tmp);
        cub::DeviceRadixSort::SortPairs(t.get(), tmp, d_ids, keys.get(), iota.get(), order.get(), static_cast<int>(n),
                                        0, end_bit, s);
        local_pos_kernel<<<ceil_div(n, 256), 256, 0, s>>>(order.get(), d_ids, start.get(), n, local.get(), pos.get());
        LAUNCH_OK("stable_group");
    }
    ctx.sync();
}

}  // namespace

void build_band_layout(Ctx& ctx, Band& B, const uint32_t* d_src_bucket, const uint32_t* d_tgt_bucket, size_t n,
                       size_t m, size_t nb) {
    cudaStream_t s = ctx.stream;
    B.nb = nb;
    B.src_bucket.resize(std::max<size_t>(n, 1));
    B.tgt_bucket.resize(std::max<size_t>(m, 1));
    if (n) CUDA_OK(cudaMemcpyAsync(B.src_bucket.get(), d_src_bucket, n * 4, cudaMemcpyDeviceToDevice, s));
    if (m) CUDA_OK(cudaMemcpyAsync(B.tgt_bucket.get(), d_tgt_bucket, m * 4, cudaMemcpyDeviceToDevice, s));
    stable_group(ctx, B.src_bucket.get(), n, nb, B.src_order, B.src_start, B.h_src_start, B.src_local, B.src_pos);
    stable_group(ctx, B.tgt_bucket.get(), m, nb, B.tgt_order, B.tgt_start, B.h_tgt_start, B.tgt_local, B.tgt_pos);
    B.h_blk_off.assign(nb + 1, 0);
    B.h_blkT_off.assign(nb + 1, 0);
    std::vector<uint32_t> work;
    B.real_entries = 0;
    for (size_t b = 0; b < nb; ++b) {
        unsigned long long nbk = B.h_src_start[b + 1] - B.h_src_start[b];
        unsigned long long mbk = B.h_tgt_start[b + 1] - B.h_tgt_start[b];
        // rows padded to a multiple of 4 entries: every block row starts 16-byte
        // aligned so the iteration kernels stream it as float4 / double2x2.
        // ... and every block starts on a 128-byte line (32 entries) so the
        // bulk-copy chunks of the streaming kernels are line aligned.
        B.h_blk_off[b + 1] = (B.h_blk_off[b] + nbk * row_stride(mbk) + 31ull) & ~31ull;
        B.h_blkT_off[b + 1] = (B.h_blkT_off[b] + mbk * row_stride(nbk) + 31ull) & ~31ull;
        B.real_entries += nbk * mbk;
        if (nbk && mbk) work.push_back(static_cast<uint32_t>(b));
    }
    // largest blocks first: better tail balance for the per-bucket kernels
    std::stable_sort(work.begin(), work.end(), [&](uint32_t x, uint32_t y) {
        auto sz = [&](uint32_t k) {
            return static_cast<unsigned long long>(B.h_src_start[k + 1] - B.h_src_start[k]) *
                   (B.h_tgt_start[k + 1] - B.h_tgt_start[k]);
        };
        return sz(x) > sz(y);
    });
    B.entries = B.h_blk_off[nb];
    B.entriesT = B.h_blkT_off[nb];
    B.blk_off.upload(B.h_blk_off.data(), nb + 1, s);
    B.blkT_off.upload(B.h_blkT_off.data(), nb + 1, s);
    B.n_work = work.size();
    B.work.resize(std::max<size_t>(work.size(), 1));
    if (!work.empty()) B.work.upload(work.data(), work.size(), s);
    ctx.sync();
}

namespace {
__global__ void compose_kernel(uint64_t* __restrict__ comp, const uint32_t* __restrict__ a, long long n, uint64_t radix) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) comp[i] = comp[i] * radix + a[i];
}
__global__ void narrow_kernel(uint32_t* __restrict__ out, const uint64_t* __restrict__ in, long long n) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) out[i] = static_cast<uint32_t>(in[i]);
}
}  // namespace

// Independent build stages (the k-means of each LSH band, the landmark
// k-means) run concurrently: one host thread and one non-blocking stream per
// job, each on its own copy of the context. Their seeding walks are
// latency-bound single-CTA kernels, so the jobs overlap well. Results do not
// depend on the overlap (every job is deterministic on its own).
void* cublas_pool_take(int device);
void cublas_pool_give(int device, void* h);
void run_jobs(Ctx& ctx, std::vector<std::function<void(Ctx&)>>& jobs) {
    if (jobs.size() == 1) {
        jobs[0](ctx);
        return;
    }
    ctx.sync();  // inputs are ready on the caller's stream
    std::vector<Ctx> ctxs(jobs.size(), ctx);
    std::vector<std::exception_ptr> errs(jobs.size());
    for (auto& c : ctxs) {
        c.own_stream = nullptr;
        c.comm.reset();
        c.cublas = nullptr;  // a job that needs one creates its own (released below)
        CUDA_OK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    }
    std::vector<std::thread> th;
    for (size_t i = 0; i < jobs.size(); ++i)
        th.emplace_back([&, i] {
            try {
                CUDA_OK(cudaSetDevice(ctx.device));
                alloc_stream() = ctxs[i].stream;
                jobs[i](ctxs[i]);
                CUDA_OK(cudaStreamSynchronize(ctxs[i].stream));
            } catch (...) {
                errs[i] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& c : ctxs) {
        cublas_pool_give(c.device, c.cublas);  // back to the pool, not destroyed
        cudaStreamDestroy(c.stream);
    }
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

namespace {

// cross_polytope_bucket (lsh.cpp:55-71) for a 64-point tile per CTA: every
// v = x . proj(:, c) is folded over the features in increasing order with
// separate multiply and add (bit-identical to the reference loop), and the
// argmax over [v || -v] keeps the first maximum, i.e. the lexicographic
// (value desc, index asc) winner. Rt is half x d, Rt[c*d + k] = proj(k, c).
template <typename T>
__global__ void __launch_bounds__(256) cp_hash_kernel(const T* __restrict__ X, long long N, int d,
                                                      const double* __restrict__ Rt, int half, uint64_t radix,
                                                      uint64_t* __restrict__ comp) {
    __shared__ double As[KC][TP + 1];
    __shared__ double Bs[KC][TC + 1];
    const long long r0 = blockIdx.x * static_cast<long long>(TP);
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double best[4];
    uint32_t arg[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) best[i] = -CUDART_INF, arg[i] = 0xffffffffu;
    auto better = [](double v, uint32_t a, double bv, uint32_t ba) { return v > bv || (v == bv && a < ba); };
    for (int c0 = 0; c0 < half; c0 += TC) {
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        for (int k0 = 0; k0 < d; k0 += KC) {
            load_slab<T>(As, X, nullptr, r0, N, d, k0);
            load_slab<double>(Bs, Rt, nullptr, c0, half, d, k0);
            __syncthreads();
            tile_fold<1>(As, Bs, ty, tx, acc);
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double bv = -CUDART_INF;
            uint32_t ba = 0xffffffffu;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = c0 + tx + 16 * j;
                if (c >= half) continue;
                if (better(acc[i][j], c, bv, ba)) bv = acc[i][j], ba = c;
                if (better(-acc[i][j], c + half, bv, ba)) bv = -acc[i][j], ba = c + half;
            }
#pragma unroll
            for (int o = 8; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const uint32_t oa = __shfl_xor_sync(0xffffffffu, ba, o);
                if (better(ov, oa, bv, ba)) bv = ov, ba = oa;
            }
            if (better(bv, ba, best[i], arg[i])) best[i] = bv, arg[i] = ba;
        }
    }
    if (tx == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const long long r = r0 + ty + 16 * i;
            if (r < N) comp[r] = comp[r] * radix + (arg[i] == 0xffffffffu ? 0u : arg[i]);
        }
}

__global__ void seq_kernel(uint32_t* __restrict__ p, long long n) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) p[i] = static_cast<uint32_t>(i);
}

template <typename T>
__global__ void gather_rows_kernel(T* __restrict__ out, const T* __restrict__ X, const uint32_t* __restrict__ idx,
                                   long long cnt, int d) {
    const long long e = blockIdx.x * 256LL + threadIdx.x;
    if (e < cnt * d) {
        const long long r = e / d;
        out[e] = X[static_cast<long long>(idx[r]) * d + (e - r * d)];
    }
}

__global__ void child_count_kernel(const uint32_t* __restrict__ a, long long n, int k, int* __restrict__ counts) {
    __shared__ int loc[64];
    for (int c = threadIdx.x; c < k; c += blockDim.x) loc[c] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) atomicAdd(&loc[a[i]], 1);
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x)
        if (loc[c]) atomicAdd(&counts[c], loc[c]);
}

// One CTA per leaf: every point of leaf segment blockIdx.x gets the leaf id.
__global__ void leaf_fill_kernel(uint32_t* __restrict__ assign, const uint32_t* __restrict__ idx,
                                 const long long* __restrict__ seg) {
    const long long off = seg[2 * blockIdx.x], len = seg[2 * blockIdx.x + 1];
    for (long long e = threadIdx.x; e < len; e += blockDim.x) assign[idx[off + e]] = blockIdx.x;
}

// hierarchical_assign (lsh.cpp:107-143): FIFO queue of clusters, a cluster
// becomes a leaf once queue + leaves + 1 >= target (or it has < 2 points),
// otherwise lloyd(k = min(branching, size), iters, mix64(seed ^ ++splits))
// on its points splits it and the non-empty children are queued in child
// order. Clusters are contiguous segments of a device permutation; a split
// gathers its points, runs lloyd_device, and stable-sorts the segment by
// child (the push_back order of lsh.cpp:134-135), so only the k child sizes
// come back to the host for the queue.
// Returns the leaf count: with branching > 2 the last split can overshoot the
// target, and leaf ids >= target then flow into the composite ids exactly as
// in the reference.
template <typename T>
long long hier_assign_device(Ctx& ctx, const T* X, long long N, int d, int target, int branching, int iters,
                             uint64_t seed, uint32_t* assign) {
    if (branching < 2) throw Status(2, "lsh: branching must be >= 2");
    if (branching > 64) throw Status(2, "lsh: branching > 64 is not supported on this path");
    cudaStream_t s = ctx.stream;
    DevBuf<uint32_t> idx(N), idx2(N), keys(N), keys2(N);
    DevBuf<T> sub(static_cast<size_t>(N) * d);
    DevBuf<double> ctr(static_cast<size_t>(branching) * d);
    DevBuf<int> counts(branching);
    seq_kernel<<<ceil_div(N, 256), 256, 0, s>>>(idx.get(), N);
    int end_bit = 1;
    while ((1LL << end_bit) < branching) ++end_bit;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.get(), keys2.get(), idx.get(), idx2.get(),
                                    static_cast<int>(N), 0, end_bit, s);
    DevBuf<unsigned char> tmp(tmp_bytes);
    std::deque<std::pair<long long, long long>> queue{{0, N}};
    std::vector<long long> leaves;  // (off, len) pairs
    uint64_t splits = 0;
    std::vector<int> h_counts(branching);
    while (!queue.empty()) {
        const auto [off, len] = queue.front();
        queue.pop_front();
        const size_t live = queue.size() + leaves.size() / 2 + 1;
        if (live >= static_cast<size_t>(target) || len < 2) {
            leaves.push_back(off);
            leaves.push_back(len);
            continue;
        }
        const int k = static_cast<int>(std::min<long long>(branching, len));
        gather_rows_kernel<T><<<ceil_div(len * d, 256), 256, 0, s>>>(sub.get(), X, idx.get() + off, len, d);
        LAUNCH_OK("hierarchical gather");
        lloyd_device<T>(ctx, sub.get(), len, d, k, iters, mix64(seed ^ ++splits), ctr.get(), keys.get());
        size_t need = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, need, keys.get(), keys2.get(), idx.get() + off, idx2.get(),
                                        static_cast<int>(len), 0, end_bit, s);
        if (need > tmp_bytes) throw Status(6, "hierarchical k-means: sort scratch too small");
        cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, keys.get(), keys2.get(), idx.get() + off, idx2.get(),
                                        static_cast<int>(len), 0, end_bit, s);
        CUDA_OK(cudaMemcpyAsync(idx.get() + off, idx2.get(), len * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        CUDA_OK(cudaMemsetAsync(counts.get(), 0, k * sizeof(int), s));
        child_count_kernel<<<static_cast<unsigned>(std::min<long long>(ceil_div(len, 256), 4LL * ctx.num_sms)), 256,
                             0, s>>>(keys.get(), len, k, counts.get());
        LAUNCH_OK("hierarchical child counts");
        counts.download(h_counts.data(), k, s);
        ctx.sync();
        long long at = off;
        for (int c = 0; c < k; ++c) {
            if (h_counts[c] > 0) queue.emplace_back(at, h_counts[c]);
            at += h_counts[c];
        }
    }
    const long long nleaves = static_cast<long long>(leaves.size() / 2);
    DevBuf<long long> seg(leaves.size());
    seg.upload(leaves.data(), leaves.size(), s);
    leaf_fill_kernel<<<static_cast<unsigned>(nleaves), 256, 0, s>>>(assign, idx.get(), seg.get());
    LAUNCH_OK("hierarchical leaf ids");
    ctx.sync();
    return nleaves;
}

// hash_cross_polytope's projection (lsh.cpp:85-89): proj is d x half filled
// row-major from normal_distribution<double>(0, 1) over mt19937_64(seed);
// returned transposed (half x d) for the tile loads.
std::vector<double> cp_projection(uint64_t seed, size_t d, size_t half) {
    std::vector<double> proj(d * half), t(d * half);
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (double& v : proj) v = gauss(rng);
    for (size_t k = 0; k < d; ++k)
        for (size_t c = 0; c < half; ++c) t[c * d + k] = proj[k * half + c];
    return t;
}

}  // namespace

// cross_polytope_bucket (lsh.cpp:55-71) for n device points against an
// explicit host projection (d x half, row-major as DenseMatrix).
void cross_polytope_buckets_device(Ctx& ctx, const double* X, long long N, int d, const double* h_proj, int half,
                                   uint32_t* out) {
    cudaStream_t s = ctx.stream;
    std::vector<double> t(static_cast<size_t>(d) * half);
    for (int k = 0; k < d; ++k)
        for (int c = 0; c < half; ++c) t[static_cast<size_t>(c) * d + k] = h_proj[static_cast<size_t>(k) * half + c];
    DevBuf<double> Rt(t.size());
    Rt.upload(t.data(), t.size(), s);
    DevBuf<uint64_t> comp(N);
    comp.zero(s);
    cp_hash_kernel<double><<<static_cast<unsigned>(ceil_div(N, TP)), 256, 0, s>>>(X, N, d, Rt.get(), half, 1,
                                                                                  comp.get());
    narrow_kernel<<<ceil_div(N, 256), 256, 0, s>>>(out, comp.get(), N);
    LAUNCH_OK("cross-polytope buckets");
    ctx.sync();
}

// lsh_neighbor_pairs (lsh.cpp:245-283) up to the bucket ids, per band, of the
// union [p; q]:
//   * cross-polytope: hash_cross_polytope of p and of q with the same
//     projections (lsh.cpp:73-103) — the per-point hash does not depend on
//     which set the point is in, so the union is hashed in one pass;
//   * k-means / hierarchical k-means: hash_kmeans of the union
//     (lsh.cpp:145-158) with fn_seed(seed, band, fn).
// Composite ids are mixed-radix over the r functions. Bands run as concurrent
// jobs, together with `extra` (the landmark k-means) when given.
void lsh_bucket_ids(Ctx& ctx, const double* d_union, const float* d_union32, size_t n, size_t m, size_t d,
                    const LshParams& cfg, std::vector<DevBuf<uint32_t>>& ids, size_t& range,
                    const std::function<void(Ctx&)>& extra, const ExtraSeeding* extra_seed, bool early_extra) {
    const size_t N = n + m;
    const int bands = cfg.bands, rows = cfg.rows, buckets = cfg.buckets;
    if (bands < 1 || rows < 1) throw Status(2, "lsh: bands and rows_per_band must be >= 1");
    if (buckets < 2) throw Status(2, "lsh: buckets_per_fn must be >= 2");
    if (cfg.scheme < 0 || cfg.scheme > 2) throw Status(2, "unknown LSH scheme");
    if (cfg.scheme == 0) {
        if (buckets % 2 != 0) throw Status(2, "cross-polytope needs an even bucket count");
    } else {
        if (static_cast<size_t>(buckets) > N) throw Status(2, "hash_kmeans: more buckets than points");
    }
    double r = std::pow(static_cast<double>(buckets), rows);
    if (r > 4294967295.0) throw Status(2, "lsh: composite bucket range exceeds 2^32 on this path");
    range = static_cast<size_t>(r);
    ids.clear();
    ids.resize(bands);
    // per band: an upper bound on its composite ids (hierarchical leaves can
    // exceed buckets - 1, see hier_assign_device)
    std::vector<double> band_bound(bands, 0.0);
    // k-means scheme: every band function's k-means++ seeding (and the
    // landmark k-means', when given) runs as one batched step chain first;
    // the per-band jobs then run Lloyd from those seeds
    // early_extra: the extra job (the landmark k-means, and the Nystrom
    // factors when the caller adds them) starts now on its own thread and
    // stream, concurrently with the bands' seeding chain and Lloyd jobs;
    // its host-side LDL^T and its device work fill the seeding chain's gaps
    struct ExtraThread {
        std::thread th;
        Ctx c;
        std::exception_ptr err;
        bool on = false;
        ~ExtraThread() {
            if (th.joinable()) th.join();
            if (on) {
                cublas_pool_give(c.device, c.cublas);
                cudaStreamDestroy(c.stream);
            }
        }
    } xt;
    if (extra && early_extra) {
        ctx.sync();  // inputs are ready on the caller's stream
        xt.c = ctx;
        xt.c.own_stream = nullptr;
        xt.c.comm.reset();
        xt.c.cublas = nullptr;
        CUDA_OK(cudaStreamCreateWithFlags(&xt.c.stream, cudaStreamNonBlocking));
        xt.on = true;
        xt.th = std::thread([&] {
            try {
                CUDA_OK(cudaSetDevice(ctx.device));
                alloc_stream() = xt.c.stream;
                extra(xt.c);
                CUDA_OK(cudaStreamSynchronize(xt.c.stream));
            } catch (...) {
                xt.err = std::current_exception();
            }
        });
    }
    std::vector<DevBuf<uint32_t>> inits;
    const bool xseed = extra_seed && extra_seed->k > 0 && static_cast<size_t>(extra_seed->k) <= N && extra_seed->out;
    if (cfg.scheme == 1 || xseed) {
        PhaseTimer pt(ctx, "k-means++ seeding (batched chain)");
        std::vector<PPSeq> seqs;
        if (cfg.scheme == 1) {
            inits.resize(static_cast<size_t>(bands) * rows);
            for (int b = 0; b < bands; ++b)
                for (int fn = 0; fn < rows; ++fn) {
                    auto& ib = inits[static_cast<size_t>(b) * rows + fn];
                    ib.resize(buckets);
                    seqs.push_back(
                        lloyd_seed_seq(fn_seed(cfg.seed, b, fn), static_cast<long long>(N), buckets, ib.get()));
                }
        }
        if (xseed)
            seqs.push_back(lloyd_seed_seq(extra_seed->seed, static_cast<long long>(N), extra_seed->k, extra_seed->out));
        if (d_union32)
            kmeans_pp_batch<float>(ctx, d_union32, static_cast<long long>(N), static_cast<int>(d), seqs);
        else
            kmeans_pp_batch<double>(ctx, d_union, static_cast<long long>(N), static_cast<int>(d), seqs);
    }
    std::vector<std::function<void(Ctx&)>> jobs;
    for (int b = 0; b < bands; ++b)
        jobs.push_back([&, b](Ctx& jc) {
            cudaStream_t s = jc.stream;
            double bound = 0.0;
            DevBuf<uint64_t> comp(N);
            comp.zero(s);
            const uint64_t radix = static_cast<uint64_t>(buckets);
            if (cfg.scheme == 0) {
                const int half = buckets / 2;
                DevBuf<double> Rt(static_cast<size_t>(half) * d);
                for (int fn = 0; fn < rows; ++fn) {
                    PhaseTimer pt(jc, "lsh cross-polytope (one band function)");
                    const std::vector<double> h = cp_projection(fn_seed(cfg.seed, b, fn), d, half);
                    Rt.upload(h.data(), h.size(), s);
                    const unsigned grid = static_cast<unsigned>(ceil_div(N, TP));
                    if (d_union32)
                        cp_hash_kernel<float><<<grid, 256, 0, s>>>(d_union32, N, static_cast<int>(d), Rt.get(), half,
                                                                  radix, comp.get());
                    else
                        cp_hash_kernel<double><<<grid, 256, 0, s>>>(d_union, N, static_cast<int>(d), Rt.get(), half,
                                                                   radix, comp.get());
                    LAUNCH_OK("cross-polytope hash");
                    jc.sync();  // h is reused by the next function's upload
                }
            } else {
                DevBuf<double> ctr(static_cast<size_t>(buckets) * d);
                DevBuf<uint32_t> assign(N);
                for (int fn = 0; fn < rows; ++fn) {
                    PhaseTimer pt(jc, "lsh k-means (one band function)");
                    const uint64_t sd = fn_seed(cfg.seed, b, fn);
                    const long long NN = static_cast<long long>(N);
                    long long leaves = buckets;
                    if (cfg.scheme == 2) {
                        if (d_union32)
                            leaves = hier_assign_device<float>(jc, d_union32, NN, static_cast<int>(d), buckets,
                                                               cfg.branching, cfg.iters, sd, assign.get());
                        else
                            leaves = hier_assign_device<double>(jc, d_union, NN, static_cast<int>(d), buckets,
                                                                cfg.branching, cfg.iters, sd, assign.get());
                    } else if (d_union32) {
                        lloyd_device<float>(jc, d_union32, NN, static_cast<int>(d), buckets, cfg.iters, sd, ctr.get(),
                                            assign.get(), inits[static_cast<size_t>(b) * rows + fn].get());
                    } else {
                        lloyd_device<double>(jc, d_union, NN, static_cast<int>(d), buckets, cfg.iters, sd, ctr.get(),
                                             assign.get(), inits[static_cast<size_t>(b) * rows + fn].get());
                    }
                    compose_kernel<<<ceil_div(N, 256), 256, 0, s>>>(comp.get(), assign.get(), N, radix);
                    bound = bound * static_cast<double>(radix) + static_cast<double>(leaves - 1);
                }
            }
            band_bound[b] = bound;
            DevBuf<uint32_t> out(N);
            narrow_kernel<<<ceil_div(N, 256), 256, 0, s>>>(out.get(), comp.get(), N);
            LAUNCH_OK("lsh ids");
            jc.sync();
            ids[b] = std::move(out);
        });
    if (extra && !early_extra) jobs.push_back(extra);
    if (ctx.comm && ctx.comm->world > 1) {
        // sharded build: the k-means assignments are split over the ranks
        // (lloyd_device's all-gather), so the jobs run one after the other on
        // this context, the communicator's calls in the same order on every rank
        for (auto& j : jobs) j(ctx);
        ctx.sync();
    } else {
        run_jobs(ctx, jobs);
    }
    if (xt.on) {
        xt.th.join();
        if (xt.err) std::rethrow_exception(xt.err);
    }
    ctx.sync();
    for (double bb : band_bound) {
        if (bb + 1.0 > 4294967295.0) throw Status(2, "lsh: composite bucket range exceeds 2^32 on this path");
        range = std::max(range, static_cast<size_t>(bb) + 1);
    }
}

// ---------------------------------------------------------------------------
// Tiled kernels with epilogues
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ double cost_from_fold(int kind, double acc, double nx, double ny, int* bad) {
    if (kind == 0) return __dsqrt_rn(acc);
    if (kind == 3) return acc;
    if (kind == 1) return -acc;
    if (nx == 0.0 || ny == 0.0) {
        atomicOr(bad, 1);
        return 0.0;
    }
    double c = __ddiv_rn(acc, __dsqrt_rn(xmul(nx, ny)));
    c = c > 1.0 ? 1.0 : c;
    c = c < -1.0 ? -1.0 : c;
    return __dsqrt_rn(xsub(1.0, c));
}

// Band blocks: tile = (bucket, r0, c0) of bucket's n_b x m_b block.
template <int MODE, class Epi>
__global__ void __launch_bounds__(256) band_tile_kernel(const int4* __restrict__ tiles, BandView bv,
                                                        const double* __restrict__ A, const double* __restrict__ B,
                                                        int d, Epi epi) {
    __shared__ double As[KC][TP + 1];
    __shared__ double Bs[KC][TC + 1];
    const int4 t = tiles[blockIdx.x];
    const int b = t.x, r0 = t.y, c0 = t.z;
    const uint32_t sb = bv.src_start[b], nb = bv.src_start[b + 1] - sb;
    const uint32_t tb = bv.tgt_start[b], mb = bv.tgt_start[b + 1] - tb;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += KC) {
        load_slab<double>(As, A, bv.src_order + sb, r0, nb, d, k0);
        load_slab<double>(Bs, B, bv.tgt_order + tb, c0, mb, d, k0);
        __syncthreads();
        tile_fold<MODE>(As, Bs, ty, tx, acc);
        __syncthreads();
    }
    double tmax = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t r = r0 + ty + 16 * i;
        if (r >= nb) continue;
        const uint32_t si = bv.src_order[sb + r];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t c = c0 + tx + 16 * j;
            if (c < mb) {
                const double v = epi(bv.blk_off[b] + static_cast<unsigned long long>(r) * row_stride(mb) + c, si,
                                     bv.tgt_order[tb + c], acc[i][j]);
                if constexpr (Epi::kReduce) tmax = fmax(tmax, v);
            }
        }
    }
    // one atomic per warp (a per-element atomic on one address serialises)
    if constexpr (Epi::kReduce) {
        tmax = warp_max(tmax);
        if ((threadIdx.x & 31) == 0) atomicMax(epi.maxbits, static_cast<unsigned long long>(__double_as_longlong(tmax)));
    }
}

// Dense: rows of A (na) against rows of B (nb).
template <int MODE, class Epi>
__global__ void __launch_bounds__(256) dense_tile_kernel(const double* __restrict__ A, long long na,
                                                         const double* __restrict__ B, long long nbr, int d, Epi epi) {
    __shared__ double As[KC][TP + 1];
    __shared__ double Bs[KC][TC + 1];
    const long long r0 = static_cast<long long>(blockIdx.x) * TP, c0 = static_cast<long long>(blockIdx.y) * TC;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += KC) {
        load_slab<double>(As, A, nullptr, r0, na, d, k0);
        load_slab<double>(Bs, B, nullptr, c0, nbr, d, k0);
        __syncthreads();
        tile_fold<MODE>(As, Bs, ty, tx, acc);
        __syncthreads();
    }
    double tmax = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        long long r = r0 + ty + 16 * i;
        if (r >= na) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            long long c = c0 + tx + 16 * j;
            if (c < nbr) {
                const double v = epi(r, c, acc[i][j]);
                if constexpr (Epi::kReduce) tmax = fmax(tmax, v);
            }
        }
    }
    if constexpr (Epi::kReduce) {
        tmax = warp_max(tmax);
        if ((threadIdx.x & 31) == 0) atomicMax(epi.maxbits, static_cast<unsigned long long>(__double_as_longlong(tmax)));
    }
}

// log K^sp at a block entry, -inf where an earlier band already holds the
// pair (sparse_kernel.cpp:76: logvals = 0.0 - cost * inv).
struct EpiLogK {
    static constexpr bool kReduce = false;
    double* out;
    BandSet bs;
    int band;
    int kind;
    double inv;
    const double* norms;  // union norms (cosine only), targets offset by n
    long long n;
    int* bad;
    __device__ double operator()(unsigned long long idx, uint32_t i, uint32_t j, double acc) const {
        for (int b = 0; b < band; ++b)
            if (bs.src_bucket[b][i] == bs.tgt_bucket[b][j]) {
                out[idx] = kNegInf;
                return 0.0;
            }
        double nx = norms ? norms[i] : 0.0, ny = norms ? norms[n + j] : 0.0;
        double c = cost_from_fold(kind, acc, nx, ny, bad);
        out[idx] = xsub(0.0, xmul(c, inv));
        return 0.0;
    }
};

// exp(-c * inv) (kernel_block, nystrom.cpp:53-64) or exp(-c / lambda)
// (the landmark Gram matrix A, nystrom.cpp:91-95).
struct EpiExp {
    static constexpr bool kReduce = false;
    double* out;
    long long ld;
    int kind;
    double scale;
    bool divide;
    const double* na;
    const double* nb;
    int* bad;
    __device__ double operator()(long long r, long long c, double acc) const {
        double c0 = cost_from_fold(kind, acc, na ? na[r] : 0.0, nb ? nb[c] : 0.0, bad);
        out[r * ld + c] = divide ? exp(__ddiv_rn(-c0, scale)) : exp(xmul(-c0, scale));
        return 0.0;
    }
};

// dense cost (build_cost, geometry.cpp:113-130): c of every pair
struct EpiDenseCost {
    static constexpr bool kReduce = false;
    double* out;
    long long ld;
    int kind;
    const double* na;
    const double* nb;
    int* bad;
    __device__ double operator()(long long r, long long c, double acc) const {
        out[r * ld + c] = cost_from_fold(kind, acc, na ? na[r] : 0.0, nb ? nb[c] : 0.0, bad);
        return 0.0;
    }
};

// dense log K (build_cost + build_kernel, geometry.cpp:113-144):
// logk = 0.0 - c * inv with c the sequential-fold cost of the pair
struct EpiDenseLogK {
    static constexpr bool kReduce = false;
    double* out;
    long long ld;
    int kind;
    double inv;
    const double* na;
    const double* nb;
    int* bad;
    __device__ double operator()(long long r, long long c, double acc) const {
        const double cst = cost_from_fold(kind, acc, na ? na[r] : 0.0, nb ? nb[c] : 0.0, bad);
        out[r * ld + c] = xsub(0.0, xmul(cst, inv));
        return 0.0;
    }
};

struct EpiStore {
    static constexpr bool kReduce = false;
    double* out;
    long long ld;
    int* bad;
    __device__ double operator()(long long r, long long c, double acc) const {
        if (!isfinite(acc)) atomicOr(bad, 1);
        out[r * ld + c] = acc;
        return 0.0;
    }
};

// max |(A_j W) - V| with the transposed storage: acc = (A_j W)_{c r}.
struct EpiResid {
    static constexpr bool kReduce = true;  // max |.| reduced per warp by the tile kernel
    const double* vt;
    long long ld;
    unsigned long long* maxbits;
    __device__ double operator()(long long r, long long c, double acc) const {
        double e = fabs(acc - vt[r * ld + c]);
        if (!(e <= 1.79e308)) e = kPosInf;
        return e;
    }
};

// delta = exp(log K) - (U W)_ij (sparse_kernel.cpp:100-109); acc is the
// sequential fold sum_a u_ia w_aj of NystromFactors::entry (nystrom.cpp:127-132).
struct EpiDelta {
    static constexpr bool kReduce = true;
    double* delta;
    const double* logk;
    unsigned long long* maxbits;
    int* overflow;
    __device__ double operator()(unsigned long long idx, uint32_t, uint32_t, double nys) const {
        double lk = logk[idx];
        if (lk == kNegInf) {  // masked duplicate of an earlier band
            delta[idx] = 0.0;
            return 0.0;
        }
        double exact = exp(lk);
        if (isinf(exact)) {
            atomicOr(overflow, 1);
            delta[idx] = 0.0;
            return 0.0;
        }
        double dv = exact - nys;
        delta[idx] = dv;
        return fabs(dv);
    }
};

__global__ void fill_value_kernel(double* __restrict__ p, unsigned long long n, double v) {
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 256ull * gridDim.x) p[i] = v;
}
void fill_value(Ctx& ctx, double* p, unsigned long long n, double v) {
    if (n) fill_value_kernel<<<std::min<long long>(ceil_div(n, 256), 16 * ctx.num_sms), 256, 0, ctx.stream>>>(p, n, v);
}

__global__ void norms_kernel(const double* __restrict__ X, long long N, int d, double* __restrict__ out) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < N) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = xadd(s, xmul(X[i * d + k], X[i * d + k]));
        out[i] = s;
    }
}

std::vector<int4> band_tiles(const Band& B) {
    std::vector<int4> tiles;
    for (size_t b = 0; b < B.nb; ++b) {
        int nbk = B.h_src_start[b + 1] - B.h_src_start[b];
        int mbk = B.h_tgt_start[b + 1] - B.h_tgt_start[b];
        for (int r0 = 0; r0 < nbk; r0 += TP)
            for (int c0 = 0; c0 < mbk; c0 += TC) tiles.push_back(make_int4(static_cast<int>(b), r0, c0, 0));
    }
    return tiles;
}

template <int MODE, class Epi>
void launch_band_tiles(Ctx& ctx, const Band& B, BandView bv, const double* A, const double* Bm, int d, Epi epi) {
    std::vector<int4> tiles = band_tiles(B);
    if (tiles.empty()) return;
    DevBuf<int4> dt;
    dt.upload(tiles.data(), tiles.size(), ctx.stream);
    for (size_t off = 0; off < tiles.size(); off += 1u << 30) {
        unsigned cnt = static_cast<unsigned>(std::min<size_t>(tiles.size() - off, 1u << 30));
        band_tile_kernel<MODE, Epi><<<cnt, 256, 0, ctx.stream>>>(dt.get() + off, bv, A, Bm, d, epi);
    }
    LAUNCH_OK("band_tile_kernel");
    ctx.sync();
}

template <int MODE, class Epi>
void launch_dense_tiles(Ctx& ctx, const double* A, long long na, const double* B, long long nb, int d, Epi epi) {
    if (na == 0 || nb == 0) return;
    dim3 grid(ceil_div(na, TP), ceil_div(nb, TC));
    dense_tile_kernel<MODE, Epi><<<grid, 256, 0, ctx.stream>>>(A, na, B, nb, d, epi);
    LAUNCH_OK("dense_tile_kernel");
}

const double* union_norms(Op& op, cudaStream_t st = nullptr) {
    if (op.cost != 2) return nullptr;
    if (op.norms.size() != op.n + op.m) {
        op.norms.resize(op.n + op.m);
        norms_kernel<<<ceil_div(op.n + op.m, 256), 256, 0, st ? st : op.ctx->stream>>>(op.X.get(), op.n + op.m, op.d,
                                                                                      op.norms.get());
        LAUNCH_OK("norms");
    }
    return op.norms.get();
}

int read_flag(Ctx& ctx, DevBuf<int>& f) {
    int h = 0;
    f.download(&h, 1, ctx.stream);
    ctx.sync();
    return h;
}

// ---- tensor-core build contractions (tc_block.cuh), fp32 storage ----------
// The cost from an FP32-accurate dot product and exact fp64 norms:
// |x - y|^2 = |x|^2 + |y|^2 - 2 x.y (cost_value, geometry.cpp:45-76).
__device__ __forceinline__ double tc_cost(int kind, float dot, double nx, double ny, int* bad) {
    const double dd = static_cast<double>(dot);
    if (kind == 1) return -dd;
    if (kind == 2) {
        if (nx == 0.0 || ny == 0.0) {
            atomicOr(bad, 1);
            return 0.0;
        }
        double c = dd / sqrt(nx * ny);
        c = c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
        return sqrt(1.0 - c);
    }
    const double sq = fmax(nx + ny - 2.0 * dd, 0.0);
    return kind == 0 ? sqrt(sq) : sq;
}

// log K^sp of band block entries (EpiLogK on the tensor cores): items
// {row tile, column tile, bucket}; -inf where an earlier band holds the pair.
// Per-column inputs are read in the band's target order (coalesced along a
// warp's lanes): the centred norms and, for each earlier band, the bucket of
// the target at that position.
struct TcEpiLogK {
    static constexpr int kRB = 4;  // rows per load batch
    double* out;
    BandView bv;
    int band, kind;
    double inv;
    const double* nrm;  // union norms |x|^2 (targets offset by n): uncentred kinds (dot, cosine)
    long long n;
    const double* cn_src;  // |x - c_b|^2 per source position (distance kinds, centred)
    const double* cn_tgt;
    const uint32_t* prev_src;  // band x n: earlier bands' bucket of the source at each position
    const uint32_t* prev_tgt;  // band x m: same for targets
    long long pn, pm;
    const uint32_t* a_first;
    const uint32_t* b_first;
    int* bad;
    struct Item {
        uint32_t sb, nb, tb, mb, r0, c0;
        unsigned long long off;
    };
    struct Row {
        bool valid;
        uint32_t p, pb0;
        double nx;
        double* o;
    };
    struct Pre {
        double ny;
        bool masked;
    };
    __device__ Item item(const int4& it) const {
        Item I;
        const int b = it.z;
        I.sb = bv.src_start[b];
        I.nb = bv.src_start[b + 1] - I.sb;
        I.tb = bv.tgt_start[b];
        I.mb = bv.tgt_start[b + 1] - I.tb;
        I.r0 = (it.x - a_first[b]) * tcb::kM;
        I.c0 = (it.y - b_first[b]) * tcb::kM;
        I.off = bv.blk_off[b];
        return I;
    }
    __device__ Row row(const Item& I, int rr) const {
        Row R{};
        const uint32_t r = I.r0 + rr;
        R.valid = r < I.nb;
        if (!R.valid) return R;
        R.p = I.sb + r;
        R.nx = cn_src ? cn_src[R.p] : nrm[bv.src_order[R.p]];
        R.pb0 = band > 0 ? prev_src[R.p] : 0u;
        R.o = out + I.off + static_cast<unsigned long long>(r) * row_stride(I.mb);
        return R;
    }
    __device__ Pre pre(const Item& I, const Row& R, int c) const {
        Pre P{0.0, false};
        const uint32_t cc = I.c0 + c;
        if (!R.valid || cc >= I.mb) return P;
        const uint32_t q = I.tb + cc;
        P.ny = cn_tgt ? cn_tgt[q] : nrm[n + bv.tgt_order[q]];
        if (band > 0) P.masked = prev_tgt[q] == R.pb0;
        for (int bb = 1; bb < band && !P.masked; ++bb) P.masked = prev_tgt[bb * pm + q] == prev_src[bb * pn + R.p];
        return P;
    }
    __device__ void apply(const Item& I, const Row& R, const Pre& P, int c, float dot) {
        const uint32_t cc = I.c0 + c;
        if (!R.valid || cc >= I.mb) return;
        R.o[cc] = P.masked ? kNegInf : 0.0 - tc_cost(kind, dot, R.nx, P.ny, bad) * inv;
    }
    __device__ void finish() {}
};

// delta = exp(log K) - (U W)_ij (sparse_kernel.cpp:100-109) with (U W)_ij
// the FP32-accurate dot of U's row and W's column
struct TcEpiDelta {
    static constexpr int kRB = 8;
    double* delta;
    const double* logk;
    BandView bv;
    const uint32_t* a_first;
    const uint32_t* b_first;
    unsigned long long* maxbits;
    int* overflow;
    double mx = 0.0;
    struct Item {
        uint32_t nb, mb, r0, c0;
        unsigned long long off;
    };
    struct Row {
        bool valid;
        unsigned long long base;
    };
    struct Pre {
        double lk;
    };
    __device__ Item item(const int4& it) const {
        Item I;
        const int b = it.z;
        I.nb = bv.src_start[b + 1] - bv.src_start[b];
        I.mb = bv.tgt_start[b + 1] - bv.tgt_start[b];
        I.r0 = (it.x - a_first[b]) * tcb::kM;
        I.c0 = (it.y - b_first[b]) * tcb::kM;
        I.off = bv.blk_off[b];
        return I;
    }
    __device__ Row row(const Item& I, int rr) const {
        Row R{};
        const uint32_t r = I.r0 + rr;
        R.valid = r < I.nb;
        R.base = I.off + static_cast<unsigned long long>(r) * row_stride(I.mb) + I.c0;
        return R;
    }
    __device__ Pre pre(const Item& I, const Row& R, int c) const {
        return Pre{R.valid && I.c0 + c < I.mb ? logk[R.base + c] : kNegInf};
    }
    __device__ void apply(const Item& I, const Row& R, const Pre& P, int c, float dot) {
        if (!R.valid || I.c0 + c >= I.mb) return;
        double dv = 0.0;
        if (P.lk != kNegInf) {  // masked duplicate of an earlier band: 0
            const double exact = exp(P.lk);
            if (isinf(exact)) atomicOr(overflow, 1);
            else dv = exact - static_cast<double>(dot);
        }
        delta[R.base + c] = dv;
        mx = fmax(mx, fabs(dv));
    }
    __device__ void finish() {
        const double w = warp_max(mx);
        if ((threadIdx.x & 31) == 0 && w > 0.0) atomicMax(maxbits, static_cast<unsigned long long>(__double_as_longlong(w)));
    }
};

// exp(-c * (1/lambda)) of a dense point x landmark block (kernel_block,
// nystrom.cpp:53-64): items {row tile, column tile}
struct TcEpiExp {
    static constexpr int kRB = 8;
    double* out;
    long long ld, nrows, ncols;
    int kind;
    double inv;
    const double* na;
    const double* nb;
    int* bad;
    struct Item {
        long long r0, c0;
    };
    struct Row {
        bool valid;
        double nx;
        double* o;
    };
    struct Pre {
        double ny;
    };
    __device__ Item item(const int4& it) const {
        return Item{static_cast<long long>(it.x) * tcb::kM, static_cast<long long>(it.y) * tcb::kM};
    }
    __device__ Row row(const Item& I, int rr) const {
        Row R{};
        const long long r = I.r0 + rr;
        R.valid = r < nrows;
        if (!R.valid) return R;
        R.nx = na[r];
        R.o = out + r * ld;
        return R;
    }
    __device__ Pre pre(const Item& I, const Row&, int c) const {
        return Pre{I.c0 + c < ncols ? nb[I.c0 + c] : 0.0};
    }
    __device__ void apply(const Item& I, const Row& R, const Pre& P, int c, float dot) {
        const long long cc = I.c0 + c;
        if (R.valid && cc < ncols) R.o[cc] = exp(-tc_cost(kind, dot, R.nx, P.ny, bad) * inv);
    }
    __device__ void finish() {}
};

// earlier bands' bucket of each position of band b's source / target order
__global__ void prev_bucket_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ bucket,
                                   long long count, uint32_t* __restrict__ out) {
    const long long p = blockIdx.x * 256LL + threadIdx.x;
    if (p < count) out[p] = bucket[order[p]];
}

// part: 1 K^sp distance blocks, 2 U / V blocks, 4 delta SDDMM. LCN_TC_PARTS
// (bit mask) overrides the default 1 | 4. U and V stay on the exact fp64
// tiles: the Nystrom product U A^-1 V cancels 5-40x against K,
// so the 3xTF32 dot's ~1e-5 relative error in U's entries (the |x|^2 + |l|^2 -
// 2 x.l cancellation, uncentrable across all landmarks) grows to ~1e-4 in the
// plan; measured at configs[3] x 0.005: sp_vals max error 9.2e-5 with U/V on
// the tensor cores, 1.9e-6 without (profiles/tc_build_r02.json). K^sp blocks
// are centred per bucket and delta absorbs its own dot error, so both keep
// ~1e-6.
bool use_tc_build(const Op& op, int part) {
    if (op.fp64 || op.ctx->exact_build || op.cost < 0 || op.cost > 3) return false;
    const char* e = std::getenv("LCN_TC_PARTS");
    return ((e && *e ? std::atoi(e) : 5) & part) != 0;
}

template <typename T>
void tc_pack(Ctx& ctx, const T* X, long long ld, int d, const uint32_t* idx, const std::vector<tcb::PackTile>& tiles,
             DevBuf<unsigned char>& out, const double* centers = nullptr) {
    const int KB = static_cast<int>(ceil_div(d, 32));
    out.resize(std::max<size_t>(tiles.size(), 1) * KB * tcb::kKBlock);
    if (tiles.empty()) return;
    DevBuf<tcb::PackTile> dt;
    dt.upload(tiles.data(), tiles.size(), ctx.stream);
    for (size_t o = 0; o < tiles.size(); o += 65535u * 512u) {
        const unsigned cnt = static_cast<unsigned>(std::min<size_t>(tiles.size() - o, 65535u * 512u));
        tcb::tcb_pack_kernel<T><<<dim3(cnt, KB), 256, 0, ctx.stream>>>(X, ld, d, idx, dt.get() + o, KB, centers,
                                                                      out.get() + o * KB * tcb::kKBlock);
    }
    LAUNCH_OK("tcb_pack_kernel");
    ctx.sync();  // dt leaves scope
}

template <class Epi>
void tc_run(Ctx& ctx, const DevBuf<unsigned char>& A, const DevBuf<unsigned char>& B, int d,
            const std::vector<int4>& items, Epi epi) {
    if (items.empty()) return;
    static std::atomic<bool> attr[64];  // per instantiation and device
    if (ctx.device >= 64 || !attr[ctx.device]) {
        CUDA_OK(cudaFuncSetAttribute(tcb::tcb_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, tcb::kSmem));
        if (ctx.device < 64) attr[ctx.device] = true;
    }
    DevBuf<int4> di;
    di.upload(items.data(), items.size(), ctx.stream);
    const int grid = static_cast<int>(std::min<size_t>(items.size(), static_cast<size_t>(ctx.num_sms)));
    // LCN_TCB_TRACE: global-timer stamps of CTA 0's first 16 items (pipeline study)
    const bool tr = std::getenv("LCN_TCB_TRACE") != nullptr;
    DevBuf<unsigned long long> trace(tr ? 128 : 0);
    if (tr) trace.zero(ctx.stream);
    tcb::tcb_kernel<Epi><<<grid, tcb::kThreads, tcb::kSmem, ctx.stream>>>(A.get(), B.get(),
                                                                         static_cast<int>(ceil_div(d, 32)), di.get(),
                                                                         static_cast<int>(items.size()), epi,
                                                                         tr ? trace.get() : nullptr);
    LAUNCH_OK("tcb_kernel");
    ctx.sync();
    if (tr) {
        unsigned long long h[128];
        trace.download(h, 128, ctx.stream);
        ctx.sync();
        std::fprintf(stderr, "[tcb trace] items %zu grid %d KB %d (ns from producer start: prod kb0, mma kb0, mma kbN, epi start, epi end, mma acc free)\n",
                     items.size(), grid, static_cast<int>(ceil_div(d, 32)));
        const unsigned long long t0 = h[0];
        for (int i = 0; i < 16 && h[i * 8]; ++i)
            std::fprintf(stderr, "[tcb trace] item %2d: %8lld %8lld %8lld %8lld %8lld %8lld\n", i,
                         (long long)(h[i * 8] - t0), (long long)(h[i * 8 + 1] - t0), (long long)(h[i * 8 + 2] - t0),
                         (long long)(h[i * 8 + 3] - t0), (long long)(h[i * 8 + 4] - t0), (long long)(h[i * 8 + 5] - t0));
    }
}

// Packed tiles and items of one band's bucket blocks: sources in 128-row
// tiles of src_order, targets in 128-row tiles of tgt_order, one item per
// (row tile, column tile) of every nonempty block.
struct TcBandTiles {
    bool centered = false;  // distance blocks: points minus their bucket's source mean
    std::vector<tcb::PackTile> a, b;
    std::vector<uint32_t> a_first, b_first;
    std::vector<int4> items;
    DevBuf<uint32_t> d_a_first, d_b_first;
};
void tc_band_tiles(Ctx& ctx, const Band& B, TcBandTiles& T) {
    T.a_first.assign(B.nb + 1, 0);
    T.b_first.assign(B.nb + 1, 0);
    for (size_t k = 0; k < B.nb; ++k) {
        const uint32_t sb = B.h_src_start[k], nbk = B.h_src_start[k + 1] - sb;
        const uint32_t tb = B.h_tgt_start[k], mbk = B.h_tgt_start[k + 1] - tb;
        T.a_first[k] = static_cast<uint32_t>(T.a.size());
        T.b_first[k] = static_cast<uint32_t>(T.b.size());
        if (nbk == 0 || mbk == 0) continue;
        const uint32_t cen = T.centered ? static_cast<uint32_t>(k) : ~0u;
        for (uint32_t r0 = 0; r0 < nbk; r0 += tcb::kM)
            T.a.push_back({sb + r0, std::min<uint32_t>(tcb::kM, nbk - r0), cen});
        for (uint32_t c0 = 0; c0 < mbk; c0 += tcb::kM)
            T.b.push_back({tb + c0, std::min<uint32_t>(tcb::kM, mbk - c0), cen});
        for (uint32_t ra = T.a_first[k]; ra < T.a.size(); ++ra)
            for (uint32_t cb = T.b_first[k]; cb < T.b.size(); ++cb)
                T.items.push_back(make_int4(static_cast<int>(ra), static_cast<int>(cb), static_cast<int>(k), 0));
    }
    T.d_a_first.upload(T.a_first.data(), T.a_first.size(), ctx.stream);
    T.d_b_first.upload(T.b_first.data(), T.b_first.size(), ctx.stream);
}

// |x|^2 of every union point (fp64 sequential fold), for the tensor-core costs
const double* union_sqnorms(Op& op, cudaStream_t st = nullptr) {
    if (op.norms.size() != op.n + op.m) {
        op.norms.resize(op.n + op.m);
        norms_kernel<<<ceil_div(op.n + op.m, 256), 256, 0, st ? st : op.ctx->stream>>>(op.X.get(), op.n + op.m, op.d,
                                                                                      op.norms.get());
        LAUNCH_OK("norms");
    }
    return op.norms.get();
}

// Bucket centers for the distance blocks: the fp64 mean of each bucket's
// sources. |x - y|^2 is translation invariant, and centred vectors of one
// bucket are nearly orthogonal, so the fp32 tensor-core accumulator never
// carries the large |x|^2 + |y|^2 terms the cancellation would amplify.
template <typename T>
__global__ void bucket_center_kernel(const T* __restrict__ X, int d, const uint32_t* __restrict__ order,
                                     const uint32_t* __restrict__ start, double* __restrict__ centers) {
    const uint32_t b = blockIdx.x, s0 = start[b], s1 = start[b + 1];
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double acc = 0.0;
        for (uint32_t p = s0; p < s1; ++p) acc += static_cast<double>(X[static_cast<long long>(order[p]) * d + k]);
        centers[static_cast<long long>(b) * d + k] = s1 > s0 ? acc / static_cast<double>(s1 - s0) : 0.0;
    }
}
// |x - c_b|^2 per position of a bucket order (one warp per position)
template <typename T>
__global__ void centered_norms_kernel(const T* __restrict__ X, int d, const uint32_t* __restrict__ order,
                                      const uint32_t* __restrict__ bucket, long long count,
                                      const double* __restrict__ centers, double* __restrict__ out) {
    const long long p = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= count) return;
    const long long i = order[p];
    const double* c = centers + static_cast<long long>(bucket[i]) * d;
    double acc = 0.0;
    for (int k = lane; k < d; k += 32) {
        const double v = static_cast<double>(X[i * d + k]) - c[k];
        acc += v * v;
    }
    acc = warp_sum(acc);
    if (lane == 0) out[p] = acc;
}

struct BandCenters {
    DevBuf<double> centers, cn_src, cn_tgt;
};
template <typename T>
void band_centers_t(Ctx& ctx, const T* P, const T* Q, int d, const Band& B, BandCenters& C) {
    cudaStream_t s = ctx.stream;
    const size_t n = B.src_order.size(), m = B.tgt_order.size();
    C.centers.resize(std::max<size_t>(B.nb * d, 1));
    C.cn_src.resize(std::max<size_t>(n, 1));
    C.cn_tgt.resize(std::max<size_t>(m, 1));
    if (B.nb) bucket_center_kernel<T><<<B.nb, 128, 0, s>>>(P, d, B.src_order.get(), B.src_start.get(), C.centers.get());
    if (n) centered_norms_kernel<T><<<ceil_div(n * 32, 256), 256, 0, s>>>(P, d, B.src_order.get(), B.src_bucket.get(),
                                                                          static_cast<long long>(n), C.centers.get(),
                                                                          C.cn_src.get());
    if (m) centered_norms_kernel<T><<<ceil_div(m * 32, 256), 256, 0, s>>>(Q, d, B.tgt_order.get(), B.tgt_bucket.get(),
                                                                          static_cast<long long>(m), C.centers.get(),
                                                                          C.cn_tgt.get());
    LAUNCH_OK("band centers");
}

// pack rows of the union points (fp32 copy when exact, else fp64)
void tc_pack_points(Op& op, bool targets, const uint32_t* idx, const std::vector<tcb::PackTile>& tiles,
                    DevBuf<unsigned char>& out, const double* centers = nullptr) {
    const long long off = targets ? static_cast<long long>(op.n * op.d) : 0;
    if (op.X32.size())
        tc_pack<float>(*op.ctx, op.X32.get() + off, op.d, static_cast<int>(op.d), idx, tiles, out, centers);
    else
        tc_pack<double>(*op.ctx, op.X.get() + off, op.d, static_cast<int>(op.d), idx, tiles, out, centers);
}
void band_centers(Op& op, const Band& B, BandCenters& C) {
    if (op.X32.size())
        band_centers_t<float>(*op.ctx, op.X32.get(), op.X32.get() + op.n * op.d, static_cast<int>(op.d), B, C);
    else
        band_centers_t<double>(*op.ctx, op.P(), op.Q(), static_cast<int>(op.d), B, C);
}

}  // namespace

void build_sparse_values(Op& op) {
    Ctx& ctx = *op.ctx;
    PhaseTimer pt(ctx, "K_sp bucket blocks");
    const double* nrm = union_norms(op);
    DevBuf<int> bad(1);
    bad.zero(ctx.stream);
    op.val64.clear();
    op.stored = 0;
    const bool dot = op.cost == 1 || op.cost == 2;  // negative-dot / cosine fold x.y, else (x-y)^2
    const bool tc = use_tc_build(op, 1);
    for (size_t b = 0; b < op.bands.size(); ++b) {
        DevBuf<double> v(std::max<unsigned long long>(op.bands[b].entries, 1));
        fill_value(ctx, v.get(), op.bands[b].entries, kNegInf);  // row padding: log K = -inf
        if (tc) {  // within-bucket distance blocks on the tensor cores (3xTF32)
            const Band& B = op.bands[b];
            TcBandTiles T;
            T.centered = op.cost == 0 || op.cost == 3;  // translation-invariant costs
            tc_band_tiles(ctx, B, T);
            BandCenters BC;
            if (T.centered) band_centers(op, B, BC);
            DevBuf<unsigned char> pa, pb;
            tc_pack_points(op, false, B.src_order.get(), T.a, pa, BC.centers.get());
            tc_pack_points(op, true, B.tgt_order.get(), T.b, pb, BC.centers.get());
            const size_t n = op.n, m = op.m;
            DevBuf<uint32_t> prev_src(std::max<size_t>(b * n, 1)), prev_tgt(std::max<size_t>(b * m, 1));
            for (size_t bb = 0; bb < b; ++bb) {
                if (n) prev_bucket_kernel<<<ceil_div(n, 256), 256, 0, ctx.stream>>>(
                    B.src_order.get(), op.bands[bb].src_bucket.get(), static_cast<long long>(n), prev_src.get() + bb * n);
                if (m) prev_bucket_kernel<<<ceil_div(m, 256), 256, 0, ctx.stream>>>(
                    B.tgt_order.get(), op.bands[bb].tgt_bucket.get(), static_cast<long long>(m), prev_tgt.get() + bb * m);
            }
            TcEpiLogK epi{v.get(), op.view(static_cast<int>(b)), static_cast<int>(b), op.cost, 1.0 / op.lambda,
                          union_sqnorms(op), static_cast<long long>(n), T.centered ? BC.cn_src.get() : nullptr,
                          T.centered ? BC.cn_tgt.get() : nullptr, prev_src.get(), prev_tgt.get(),
                          static_cast<long long>(n), static_cast<long long>(m), T.d_a_first.get(), T.d_b_first.get(),
                          bad.get()};
            tc_run(ctx, pa, pb, static_cast<int>(op.d), T.items, epi);
            op.stored += B.real_entries;
            op.val64.push_back(std::move(v));
            continue;
        }
        EpiLogK epi{v.get(), op.bandset(), static_cast<int>(b), op.cost, 1.0 / op.lambda, nrm,
                    static_cast<long long>(op.n), bad.get()};
        if (dot)
            launch_band_tiles<1>(ctx, op.bands[b], op.view(static_cast<int>(b)), op.P(), op.Q(), static_cast<int>(op.d), epi);
        else
            launch_band_tiles<0>(ctx, op.bands[b], op.view(static_cast<int>(b)), op.P(), op.Q(), static_cast<int>(op.d), epi);
        op.stored += op.bands[b].real_entries;
        op.val64.push_back(std::move(v));
    }
    if (read_flag(ctx, bad)) throw Status(2, "cosine-derived cost undefined for zero vectors");
}

// ---------------------------------------------------------------------------
// Nystrom factors (nystrom.cpp:28-125)
// ---------------------------------------------------------------------------
namespace {

using LD = long double;

// Symmetric diagonal-pivoted LDL^T in long double (the factorisation the
// reference takes from Eigen::LDLT<long double>, nystrom.cpp:108).
struct HostLdlt {
    size_t l;
    std::vector<LD> f;
    std::vector<size_t> perm;
    bool ok = true;
    HostLdlt(const std::vector<LD>& a, size_t n) : l(n), f(a), perm(n) {
        std::iota(perm.begin(), perm.end(), size_t{0});
        std::vector<LD> w(l);
        for (size_t k = 0; k < l; ++k) {
            size_t piv = k;
            LD best = std::fabs(f[k * l + k]);
            for (size_t i = k + 1; i < l; ++i)
                if (std::fabs(f[i * l + i]) > best) { best = std::fabs(f[i * l + i]); piv = i; }
            if (piv != k) {
                for (size_t c = 0; c < l; ++c) std::swap(f[k * l + c], f[piv * l + c]);
                for (size_t r = 0; r < l; ++r) std::swap(f[r * l + k], f[r * l + piv]);
                std::swap(perm[k], perm[piv]);
            }
            for (size_t j = 0; j < k; ++j) w[j] = f[j * l + j] * f[k * l + j];
            LD dk = f[k * l + k];
            for (size_t j = 0; j < k; ++j) dk -= f[k * l + j] * w[j];
            f[k * l + k] = dk;
            // row updates in parallel down to short columns (each entry's
            // operation order is unchanged: bit-identical for any team)
#pragma omp parallel for schedule(static) if ((l - k) * k > 8192)
            for (long long ii = static_cast<long long>(k) + 1; ii < static_cast<long long>(l); ++ii) {
                const size_t i = static_cast<size_t>(ii);
                LD v = f[i * l + k];
                for (size_t j = 0; j < k; ++j) v -= f[i * l + j] * w[j];
                f[i * l + k] = v;
            }
            if (std::fabs(dk) > 0) {
                for (size_t i = k + 1; i < l; ++i) f[i * l + k] /= dk;
            } else {
                for (size_t i = k + 1; i < l; ++i)
                    if (f[i * l + k] != 0) ok = false;
            }
        }
    }
    void solve(LD* b) const {
        std::vector<LD> y(l);
        for (size_t k = 0; k < l; ++k) y[k] = b[perm[k]];
        for (size_t i = 0; i < l; ++i)
            for (size_t j = 0; j < i; ++j) y[i] -= f[i * l + j] * y[j];
        for (size_t i = 0; i < l; ++i) {
            LD dv = f[i * l + i];
            y[i] = std::fabs(dv) > std::numeric_limits<LD>::min() ? y[i] / dv : 0;
        }
        for (size_t ii = l; ii-- > 0;)
            for (size_t j = ii + 1; j < l; ++j) y[ii] -= f[j * l + ii] * y[j];
        for (size_t k = 0; k < l; ++k) b[perm[k]] = y[k];
    }
};

}  // namespace

// One jitter level of build_factors' factorisation (nystrom.cpp:96-108) for a
// small l x l landmark matrix A (fp64, row-major): A_j = A + rel * trace(A)/l
// on the diagonal in long double, its diagonal-pivoted LDL^T and inverse.
// false when the factorisation fails or the inverse is not finite (the
// reference moves to the next level then); the caller tests the residual.
bool nystrom_inverse_host(const double* A, int l, double rel, double* ainv, double* aj_out) {
    const size_t L = static_cast<size_t>(l);
    std::vector<LD> a(L * L);
    LD trace = 0.0L;
    for (size_t i = 0; i < L * L; ++i) a[i] = static_cast<LD>(A[i]);
    for (size_t i = 0; i < L; ++i) trace += a[i * L + i];
    const LD jitter_unit = trace / static_cast<LD>(L);
    for (size_t i = 0; i < L; ++i) a[i * L + i] += rel * jitter_unit;
    HostLdlt fac(a, L);
    if (!fac.ok) return false;
    std::vector<LD> e(L);
    for (size_t c = 0; c < L; ++c) {
        std::fill(e.begin(), e.end(), 0.0L);
        e[c] = 1.0L;
        fac.solve(e.data());
        for (size_t r = 0; r < L; ++r) {
            if (!std::isfinite(e[r])) return false;
            ainv[r * L + c] = static_cast<double>(e[r]);
        }
    }
    for (size_t i = 0; i < L * L; ++i) aj_out[i] = static_cast<double>(a[i]);
    return true;
}

namespace {

__global__ void maxabs_kernel(const double* __restrict__ x, long long n, unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) m = fmax(m, fabs(x[i]));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

__global__ void gather_rows_kernel(const double* __restrict__ X, const uint32_t* __restrict__ rows, int k, int d,
                                   double* __restrict__ out) {
    for (int e = blockIdx.x * 256 + threadIdx.x; e < k * d; e += 256 * gridDim.x)
        out[e] = X[static_cast<long long>(rows[e / d]) * d + e % d];
}

}  // namespace

namespace {
template <typename T>
__global__ void __launch_bounds__(256) dense_transpose_kernel(const double* __restrict__ in, long long rows,
                                                              long long cols, T* __restrict__ out, T* __restrict__ copy) {
    __shared__ double tile[32][33];
    const long long r0 = static_cast<long long>(blockIdx.y) * 32, c0 = static_cast<long long>(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) {
        const long long i = r0 + r, j = c0 + tx;
        const double v = (i < rows && j < cols) ? in[i * cols + j] : 0.0;
        tile[r][tx] = v;
        if (copy && i < rows && j < cols) copy[i * cols + j] = static_cast<T>(v);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const long long j = c0 + r, i = r0 + tx;
        if (j < cols && i < rows) out[j * rows + i] = static_cast<T>(tile[tx][r]);
    }
}
}  // namespace

namespace {
// build_kernel (geometry.cpp:132-144): logk = inf ? -inf : 0.0 - c * inv
__global__ void logk_from_cost_kernel(const double* __restrict__ c, unsigned long long n, double inv,
                                      double* __restrict__ out) {
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 256ull * gridDim.x) {
        const double v = c[i];
        out[i] = isinf(v) ? kNegInf : xsub(0.0, xmul(v, inv));
    }
}
}  // namespace

// Dense cost matrix (build_cost) into op.dc64, then log K for lambda via
// dense_logk_from_cost (multi-head solves share one cost matrix).
void build_dense_cost(Op& op) {
    Ctx& ctx = *op.ctx;
    const size_t n = op.n, m = op.m, d = op.d;
    const double* nrm = union_norms(op);
    DevBuf<int> bad(1);
    bad.zero(ctx.stream);
    op.dc64.resize(std::max<size_t>(n * m, 1));
    EpiDenseCost epi{op.dc64.get(), static_cast<long long>(m), op.cost, nrm, nrm ? nrm + n : nullptr, bad.get()};
    if (op.cost == 1 || op.cost == 2)
        launch_dense_tiles<1>(ctx, op.P(), n, op.Q(), m, static_cast<int>(d), epi);
    else
        launch_dense_tiles<0>(ctx, op.P(), n, op.Q(), m, static_cast<int>(d), epi);
    if (read_flag(ctx, bad)) throw Status(2, "cosine-derived cost undefined for zero vectors");
}

void dense_logk_from_cost(Op& op, double lambda) {
    Ctx& ctx = *op.ctx;
    if (!(lambda > 0.0)) throw Status(2, "build_kernel: lambda must be positive");
    op.lambda = lambda;
    const size_t n = op.n, m = op.m;
    op.dk64.resize(std::max<size_t>(n * m, 1));
    logk_from_cost_kernel<<<std::min<long long>(ceil_div(n * m, 256), 16 * ctx.num_sms), 256, 0, ctx.stream>>>(
        op.dc64.get(), static_cast<unsigned long long>(n * m), 1.0 / lambda, op.dk64.get());
    const dim3 grid(static_cast<unsigned>(ceil_div(m, 32)), static_cast<unsigned>(ceil_div(n, 32)));
    if (op.fp64) {
        op.dk64T.resize(std::max<size_t>(n * m, 1));
        dense_transpose_kernel<double><<<grid, 256, 0, ctx.stream>>>(op.dk64.get(), n, m, op.dk64T.get(), nullptr);
    } else {
        op.dk32.resize(std::max<size_t>(n * m, 1));
        op.dk32T.resize(std::max<size_t>(n * m, 1));
        dense_transpose_kernel<float><<<grid, 256, 0, ctx.stream>>>(op.dk64.get(), n, m, op.dk32T.get(), op.dk32.get());
    }
    LAUNCH_OK("dense log K from cost");
    op.nnz = n * m;
    ctx.sync();
}

// Dense operator (KernelOperator::dense, operator.cpp:55-64): exact fp64 log K
// of every pair by the tiled sequential-fold kernel, then the iteration copies
// (fp32 or fp64) in both orientations so both half-iterations stream rows.
void build_dense(Op& op) {
    Ctx& ctx = *op.ctx;
    PhaseTimer pt(ctx, "dense log K");
    const size_t n = op.n, m = op.m, d = op.d;
    if (!(op.lambda > 0.0)) throw Status(2, "build_kernel: lambda must be positive");
    const double* nrm = union_norms(op);
    DevBuf<int> bad(1);
    bad.zero(ctx.stream);
    op.dk64.resize(std::max<size_t>(n * m, 1));
    EpiDenseLogK epi{op.dk64.get(), static_cast<long long>(m), op.cost, 1.0 / op.lambda, nrm, nrm ? nrm + n : nullptr,
                     bad.get()};
    if (op.cost == 1 || op.cost == 2)
        launch_dense_tiles<1>(ctx, op.P(), n, op.Q(), m, static_cast<int>(d), epi);
    else
        launch_dense_tiles<0>(ctx, op.P(), n, op.Q(), m, static_cast<int>(d), epi);
    if (read_flag(ctx, bad)) throw Status(2, "cosine-derived cost undefined for zero vectors");
    dense_storage(op);
}

// Iteration copies of a dense log K (op.dk64, n x m): fp32 or fp64, in both
// orientations so both half-iterations stream rows.
void dense_storage(Op& op) {
    Ctx& ctx = *op.ctx;
    const size_t n = op.n, m = op.m;
    const dim3 grid(static_cast<unsigned>(ceil_div(m, 32)), static_cast<unsigned>(ceil_div(n, 32)));
    if (op.fp64) {
        op.dk64T.resize(std::max<size_t>(n * m, 1));
        dense_transpose_kernel<double><<<grid, 256, 0, ctx.stream>>>(op.dk64.get(), n, m, op.dk64T.get(), nullptr);
    } else {
        op.dk32.resize(std::max<size_t>(n * m, 1));
        op.dk32T.resize(std::max<size_t>(n * m, 1));
        dense_transpose_kernel<float><<<grid, 256, 0, ctx.stream>>>(op.dk64.get(), n, m, op.dk32T.get(), op.dk32.get());
    }
    LAUNCH_OK("dense log K");
    op.nnz = n * m;
    ctx.sync();
}

// select_landmarks (nystrom.cpp:28-48) into op.L, on the given context (the
// build runs it as a job concurrent with the LSH k-means).
void select_landmarks_device(Op& op, Ctx& ctx, int method, uint64_t seed) {
    cudaStream_t s = ctx.stream;
    const size_t d = op.d, l = op.l, N = op.n + op.m;
    if (l < 1 || l > N) throw Status(2, "select_landmarks: l out of range");
    PhaseTimer pt(ctx, "landmarks");
    op.L.resize(l * d);
    if (method == 0) {
        DevBuf<uint32_t> asg(N);
        // seeded with the LSH bands when the build batched it (landmark_init)
        const uint32_t* init = op.landmark_init.size() == l ? op.landmark_init.get() : nullptr;
        if (op.X32.size())
            lloyd_device<float>(ctx, op.X32.get(), N, static_cast<int>(d), static_cast<int>(l), 10, seed, op.L.get(),
                                asg.get(), init);
        else
            lloyd_device<double>(ctx, op.X.get(), N, static_cast<int>(d), static_cast<int>(l), 10, seed, op.L.get(),
                                 asg.get(), init);
        op.landmark_init = DevBuf<uint32_t>();  // consumed
    } else {
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<std::size_t> first(0, N - 1);
        uint64_t f = first(rng);
        std::vector<unsigned long long> raw(l > 1 ? l - 1 : 0);
        for (auto& r : raw) r = rng();
        DevBuf<uint32_t> rows(l);
        kmeans_pp_device<double>(ctx, op.X.get(), N, static_cast<int>(d), static_cast<int>(l), f, raw, rows.get(),
                                 nullptr);
        gather_rows_kernel<<<ceil_div(l * d, 256), 256, 0, s>>>(op.X.get(), rows.get(), static_cast<int>(l),
                                                                 static_cast<int>(d), op.L.get());
        LAUNCH_OK("landmark rows");
    }
    ctx.sync();
}

bool tc_build_part(const Op& op, int part) { return use_tc_build(op, part); }

void wgemm_resid(Ctx& ctx, const double* Vt, const double* Ainv, const double* Aj, size_t m, size_t l, double* Wt,
                 int* bad, unsigned long long* maxbits);
void uv_gemm_exp(Ctx& ctx, const double* X, size_t rows, const double* L, size_t l, size_t d, const double* xsq,
                 const double* lsq, int kind, double inv, double* out, int* bad);

void build_nystrom(Op& op, const double* h_landmarks, int method, uint64_t seed, Ctx* on) {
    if (op.factors_ready) return;  // built concurrently with the LSH (lcn_op_lcn_lsh's landmark job)
    Ctx& ctx = on ? *on : *op.ctx;
    cudaStream_t s = ctx.stream;
    const size_t n = op.n, m = op.m, d = op.d, l = op.l, N = n + m;
    if (!(op.lambda > 0.0)) throw Status(2, "build_factors: lambda must be positive");
    if (h_landmarks) {
        op.L.resize(l * d);
        op.L.upload(h_landmarks, l * d, s);
    } else if (!op.landmarks_ready) {
        select_landmarks_device(op, ctx, method, seed);
    }
    op.landmarks_ready = false;
    ctx.sync();
    PhaseTimer ptf(ctx, "nystrom factors U, V, A, W");
    std::optional<PhaseTimer> pt0;
    pt0.emplace(ctx, "  norms, U / V allocation");
    const double* nrm = union_norms(op, s);
    DevBuf<double> lnorm;
    if (op.cost == 2) {
        lnorm.resize(l);
        norms_kernel<<<ceil_div(l, 256), 256, 0, s>>>(op.L.get(), l, d, lnorm.get());
    }
    DevBuf<int> bad(1);
    bad.zero(s);
    const int mode_dot = (op.cost == 1 || op.cost == 2);
    auto exp_block = [&](double* out, const double* A, long long na, const double* nA, const double* B, long long nb,
                         const double* nB, bool divide) {
        EpiExp epi{out, nb, op.cost, divide ? op.lambda : 1.0 / op.lambda, divide, nA, nB, bad.get()};
        if (mode_dot)
            launch_dense_tiles<1>(ctx, A, na, B, nb, static_cast<int>(d), epi);
        else
            launch_dense_tiles<0>(ctx, A, na, B, nb, static_cast<int>(d), epi);
    };
    // U = k(X_p, L) (n x l), V^T = k(X_q, L) (m x l), A = k(L, L) with division.
    op.U64.resize(std::max<size_t>(n * l, 1));
    DevBuf<double> Vt(std::max<size_t>(m * l, 1)), A(l * l);
    pt0.reset();
    {
    PhaseTimer ptuv(ctx, "  U, V point x landmark blocks");
    if (use_tc_build(op, 2)) {  // point x landmark blocks on the tensor cores (3xTF32)
        const double* sq = union_sqnorms(op, s);
        DevBuf<double> lsq(l);
        norms_kernel<<<ceil_div(l, 256), 256, 0, s>>>(op.L.get(), l, d, lsq.get());
        auto tiles_of = [](size_t rows) {
            std::vector<tcb::PackTile> t;
            for (size_t r0 = 0; r0 < rows; r0 += tcb::kM)
                t.push_back({static_cast<uint32_t>(r0), static_cast<uint32_t>(std::min<size_t>(tcb::kM, rows - r0)), ~0u});
            return t;
        };
        DevBuf<unsigned char> pl, px;
        const std::vector<tcb::PackTile> tl = tiles_of(l);
        tc_pack<double>(ctx, op.L.get(), d, static_cast<int>(d), nullptr, tl, pl);
        for (int side = 0; side < 2; ++side) {
            const size_t rows = side ? m : n;
            const std::vector<tcb::PackTile> tx = tiles_of(rows);
            tc_pack_points(op, side == 1, nullptr, tx, px);
            std::vector<int4> items;
            for (size_t a = 0; a < tx.size(); ++a)
                for (size_t c = 0; c < tl.size(); ++c)
                    items.push_back(make_int4(static_cast<int>(a), static_cast<int>(c), 0, 0));
            TcEpiExp epi{side ? Vt.get() : op.U64.get(), static_cast<long long>(l), static_cast<long long>(rows),
                         static_cast<long long>(l), op.cost, 1.0 / op.lambda, sq + (side ? n : 0), lsq.get(), bad.get()};
            tc_run(ctx, px, pl, static_cast<int>(d), items, epi);
        }
    } else if (!op.fp64 && !ctx.exact_build && op.cost >= 0 && op.cost <= 3 && std::getenv("LCN_UV_TILES") == nullptr) {
        // fp32 storage: the point x landmark dots as fp64 GEMMs on cuBLAS
        // (FP64 tensor cores), the cost and exp in an elementwise pass. fp64
        // dots keep U / V ~1e-15 from the reference's sequential folds (the
        // 3xTF32 split loses ~1e-4 of the plan to the 2 x.l cancellation,
        // see use_tc_build); LCN_UV_TILES forces the exact fold tiles.
        const double* sq = union_sqnorms(op, s);
        DevBuf<double> lsq(l);
        norms_kernel<<<ceil_div(l, 256), 256, 0, s>>>(op.L.get(), l, d, lsq.get());
        uv_gemm_exp(ctx, op.P(), n, op.L.get(), l, d, sq, lsq.get(), op.cost, 1.0 / op.lambda, op.U64.get(), bad.get());
        uv_gemm_exp(ctx, op.Q(), m, op.L.get(), l, d, sq + n, lsq.get(), op.cost, 1.0 / op.lambda, Vt.get(), bad.get());
    } else {
        exp_block(op.U64.get(), op.P(), n, nrm, op.L.get(), l, lnorm.get(), false);
        exp_block(Vt.get(), op.Q(), m, nrm ? nrm + n : nullptr, op.L.get(), l, lnorm.get(), false);
    }
    }
    std::optional<PhaseTimer> pta;
    pta.emplace(ctx, "  A, max |V|, host copies");
    exp_block(A.get(), op.L.get(), l, lnorm.get(), op.L.get(), l, lnorm.get(), true);
    if (read_flag(ctx, bad)) throw Status(2, "cosine-derived cost undefined for zero vectors");

    std::vector<double> hA(l * l);
    A.download(hA.data(), l * l, s);
    DevBuf<unsigned long long> vmax(1);
    vmax.zero(s);
    maxabs_kernel<<<std::min<long long>(ceil_div(m * l, 256), 1024), 256, 0, s>>>(Vt.get(), m * l, vmax.get());
    unsigned long long vbits = 0;
    vmax.download(&vbits, 1, s);
    ctx.sync();
    double vmaxd;
    std::memcpy(&vmaxd, &vbits, 8);
    const LD v_scale = std::max<LD>(static_cast<LD>(vmaxd), 1e-300L);
    pta.reset();
    std::vector<LD> a(l * l);
    for (size_t i = 0; i < l * l; ++i) a[i] = static_cast<LD>(hA[i]);
    LD trace = 0.0L;
    for (size_t i = 0; i < l; ++i) trace += a[i * l + i];
    const LD jitter_unit = trace / static_cast<LD>(l);

    pt0.emplace(ctx, "  W allocation");
    op.Wt64.resize(std::max<size_t>(m * l, 1));
    DevBuf<double> dAinv(l * l), dAj(l * l);
    pt0.reset();
    DevBuf<unsigned long long> rbits(1);
    for (double rel = 0.0; rel <= 1.1e-4; rel = (rel == 0.0 ? 1e-10 : rel * 10.0)) {
        std::vector<LD> aj = a;
        for (size_t i = 0; i < l; ++i) aj[i * l + i] += rel * jitter_unit;
        std::optional<PhaseTimer> pt_sub;
        pt_sub.emplace(ctx, "  host LDLT + inverse (long double)");
        std::vector<LD> inv(l * l);
        bool finite = true, fok = true;
        auto factor = [&] {
            HostLdlt fac(aj, l);
            if (!fac.ok) {
                fok = false;
                return;
            }
            // on a concurrent build job the other jobs' host threads are busy:
            // leave them cores (an oversubscribed team stalls at its barriers)
            const int nthr = on ? std::max(1, omp_get_num_procs() / 2 - 2) : omp_get_max_threads();
            bool fin = true;
#pragma omp parallel for schedule(static) reduction(&& : fin) num_threads(nthr)
            for (long long cc = 0; cc < static_cast<long long>(l); ++cc) {
                std::vector<LD> e(l, 0.0L);
                e[cc] = 1.0L;
                fac.solve(e.data());
                for (size_t r = 0; r < l; ++r) {
                    inv[r * l + cc] = e[r];
                    if (!std::isfinite(e[r])) fin = false;
                }
            }
            finite = fin;
        };
        if (op.during_ldlt) {
            // the first factorisation on a host thread while this one drives
            // device work that does not need the factors (K_sp, the CSR
            // support): the GPU is otherwise idle during the LDL^T
            auto work = std::move(op.during_ldlt);
            op.during_ldlt = nullptr;
            std::exception_ptr err, ferr;
            std::thread th([&] {
                try {
                    factor();
                } catch (...) {
                    ferr = std::current_exception();
                }
            });
            try {
                work();
            } catch (...) {
                err = std::current_exception();
            }
            th.join();
            if (err) std::rethrow_exception(err);
            if (ferr) std::rethrow_exception(ferr);
        } else {
            factor();
        }
        if (!fok) continue;
        pt_sub.reset();
        pt_sub.emplace(ctx, "  W = V A^-T, residual (device GEMMs)");
        if (!finite) continue;
        std::vector<double> hinv(l * l), haj(l * l);
        for (size_t i = 0; i < l * l; ++i) {
            hinv[i] = static_cast<double>(inv[i]);
            haj[i] = static_cast<double>(aj[i]);
        }
        dAinv.upload(hinv.data(), l * l, s);
        dAj.upload(haj.data(), l * l, s);
        bad.zero(s);
        // W^T = V^T A^-T  (row j: sum_b Vt[j][b] Ainv[a][b]) and the residual
        // max |A_j W - V| (nystrom.cpp:104-124): plain fp64 GEMMs, cuBLAS
        rbits.zero(s);
        wgemm_resid(ctx, Vt.get(), dAinv.get(), dAj.get(), m, l, op.Wt64.get(), bad.get(), rbits.get());
        if (read_flag(ctx, bad)) continue;
        unsigned long long rb = 0;
        rbits.download(&rb, 1, s);
        ctx.sync();
        double resid;
        std::memcpy(&resid, &rb, 8);
        if (static_cast<LD>(resid) > 1e-6L * v_scale) continue;
        LD norm_a = 0.0L, norm_inv = 0.0L;
        for (size_t c = 0; c < l; ++c) {
            LD sa = 0.0L, si = 0.0L;
            for (size_t r = 0; r < l; ++r) {
                sa += std::fabs(aj[r * l + c]);
                si += std::fabs(inv[r * l + c]);
            }
            norm_a = std::max(norm_a, sa);
            norm_inv = std::max(norm_inv, si);
        }
        LD cond = norm_a * norm_inv;
        op.cond = std::isfinite(cond) && cond > 0 ? static_cast<double>(cond) : std::numeric_limits<double>::infinity();
        ctx.sync();
        op.factors_ready = true;
        return;
    }
    throw Status(5, "build_factors: landmark kernel matrix numerically singular beyond jitter budget");
}

// ---- W = V A^-T and the residual test on cuBLAS (fp64 GEMMs) ---------------
namespace {
__global__ void resid_max_kernel(const double* __restrict__ R, const double* __restrict__ Vt, long long cnt,
                                 unsigned long long* __restrict__ maxbits, int* __restrict__ bad,
                                 const double* __restrict__ W) {
    double mx = 0.0;
    int nf = 0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < cnt; i += 256LL * gridDim.x) {
        double e = fabs(R[i] - Vt[i]);
        if (!(e <= 1.79e308)) e = kPosInf;
        mx = fmax(mx, e);
        nf |= !isfinite(W[i]);
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) {
        if (mx > 0.0) atomicMax(maxbits, static_cast<unsigned long long>(__double_as_longlong(mx)));
        if (__any_sync(0xffffffffu, nf) || nf) atomicOr(bad, 1);
    }
}
}  // namespace

cublasHandle_t cublas_of(Ctx& ctx);

namespace {
// k(x, l) = exp(-c(x, l) * (1 / lambda)) from the fp64 dot (in place) and the
// points' / landmarks' |.|^2 (kernel_block, nystrom.cpp:53-64)
__global__ void uv_exp_kernel(double* __restrict__ D, long long rows, int l, const double* __restrict__ xsq,
                              const double* __restrict__ lsq, int kind, double inv, int* __restrict__ bad) {
    const long long total = rows * l;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < total; e += 256LL * gridDim.x) {
        const long long r = e / l;
        const int a = static_cast<int>(e - r * l);
        const double dot = D[e], nx = xsq[r], nl = lsq[a];
        double c;
        if (kind == 1) {
            c = -dot;
        } else if (kind == 2) {
            if (nx == 0.0 || nl == 0.0) {
                atomicOr(bad, 1);
                c = 0.0;
            } else {
                double cs = dot / sqrt(nx * nl);
                cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
                c = sqrt(1.0 - cs);
            }
        } else {
            const double sq = fmax(nx + nl - 2.0 * dot, 0.0);
            c = kind == 0 ? sqrt(sq) : sq;
        }
        D[e] = exp(-c * inv);
    }
}
}  // namespace

void uv_gemm_exp(Ctx& ctx, const double* X, size_t rows, const double* L, size_t l, size_t d, const double* xsq,
                 const double* lsq, int kind, double inv, double* out, int* bad) {
    if (!rows) return;
    cublasHandle_t h = cublas_of(ctx);
    const double one = 1.0, zero = 0.0;
    // out (rows x l, row-major) = X L^T: column-major out^T = L X^T
    if (cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(l), static_cast<int>(rows), static_cast<int>(d),
                    &one, L, static_cast<int>(d), X, static_cast<int>(d), &zero, out, static_cast<int>(l)) !=
        CUBLAS_STATUS_SUCCESS)
        throw Status(100, "cublasDgemm failed (point x landmark dots)");
    const long long total = static_cast<long long>(rows) * static_cast<long long>(l);
    uv_exp_kernel<<<static_cast<int>(std::min<long long>(ceil_div(total, 256), 16LL * ctx.num_sms)), 256, 0,
                    ctx.stream>>>(out, static_cast<long long>(rows), static_cast<int>(l), xsq, lsq, kind, inv, bad);
    LAUNCH_OK("U / V from fp64 GEMM");
}

// Build jobs (run_jobs) run on copies of the context without a handle; they
// take one from this process-wide pool and give it back when the job ends,
// so a build does not pay cublasCreate per job (~0.1-0.2 s each on a fresh
// box). Handles are per device; a handle serves one thread at a time.
namespace {
std::mutex g_cublas_mu;
std::vector<std::pair<int, cublasHandle_t>> g_cublas_free;
}  // namespace
void* cublas_pool_take(int device) {
    {
        std::lock_guard<std::mutex> lk(g_cublas_mu);
        for (size_t i = 0; i < g_cublas_free.size(); ++i)
            if (g_cublas_free[i].first == device) {
                cublasHandle_t h = g_cublas_free[i].second;
                g_cublas_free.erase(g_cublas_free.begin() + static_cast<long>(i));
                return h;
            }
    }
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw Status(100, "cublasCreate failed");
    return h;
}
void cublas_pool_give(int device, void* h) {
    if (!h) return;
    std::lock_guard<std::mutex> lk(g_cublas_mu);
    g_cublas_free.emplace_back(device, static_cast<cublasHandle_t>(h));
}

cublasHandle_t cublas_of(Ctx& ctx) {
    if (!ctx.cublas) ctx.cublas = cublas_pool_take(ctx.device);
    cublasHandle_t h = static_cast<cublasHandle_t>(ctx.cublas);
    cublasSetStream(h, ctx.stream);
    return h;
}

// Wt (m x l, row-major) = Vt Ainv^T; residual max |Wt Aj^T - Vt| into maxbits
// (as bits of a non-negative double), non-finite W flagged in bad. Row-major
// X (r x c) is column-major X^T, so each product is one DGEMM; the residual
// runs in row chunks (a bounded temporary).
void wgemm_resid(Ctx& ctx, const double* Vt, const double* Ainv, const double* Aj, size_t m, size_t l, double* Wt,
                 int* bad, unsigned long long* maxbits) {
    cublasHandle_t h = cublas_of(ctx);
    const double one = 1.0, zero = 0.0;
    const int L = static_cast<int>(l);
    const size_t chunk = std::max<size_t>(1, (size_t(64) << 20) / std::max<size_t>(l, 1));  // rows per 512 MB
    DevBuf<double> R(std::min(m, chunk) * l);
    for (size_t r0 = 0; r0 < m; r0 += chunk) {
        const int rows = static_cast<int>(std::min(chunk, m - r0));
        if (cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, L, rows, L, &one, Ainv, L, Vt + r0 * l, L, &zero, Wt + r0 * l,
                        L) != CUBLAS_STATUS_SUCCESS ||
            cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, L, rows, L, &one, Aj, L, Wt + r0 * l, L, &zero, R.get(), L) !=
                CUBLAS_STATUS_SUCCESS)
            throw Status(100, "cublasDgemm failed");
        const long long cnt = static_cast<long long>(rows) * L;
        resid_max_kernel<<<static_cast<int>(std::min<long long>(ceil_div(cnt, 256), 8LL * ctx.num_sms)), 256, 0,
                           ctx.stream>>>(R.get(), Vt + r0 * l, cnt, maxbits, bad, Wt + r0 * l);
    }
    LAUNCH_OK("W = V A^-T (cuBLAS)");
}

// build_correction (sparse_kernel.cpp:82-117) on every band block.
void build_correction(Op& op) {
    Ctx& ctx = *op.ctx;
    PhaseTimer pt(ctx, "LCN correction (incl. K_sp)");
    // log K^sp first (same values as build_sparse; already built when the
    // factor build overlapped it with its host LDL^T), then delta.
    if (op.logk64.size() != op.bands.size()) {
        build_sparse_values(op);
        op.logk64 = std::move(op.val64);
    }
    op.val64.clear();
    DevBuf<unsigned long long> maxbits(1);
    DevBuf<int> overflow(1);
    maxbits.zero(ctx.stream);
    overflow.zero(ctx.stream);
    for (size_t b = 0; b < op.bands.size(); ++b) {
        DevBuf<double> dlt(std::max<unsigned long long>(op.bands[b].entries, 1));
        fill_value(ctx, dlt.get(), op.bands[b].entries, 0.0);  // row padding: delta = 0
        if (use_tc_build(op, 4)) {  // SDDMM U_b W_b on the tensor cores (3xTF32)
            const Band& B = op.bands[b];
            TcBandTiles T;
            tc_band_tiles(ctx, B, T);
            DevBuf<unsigned char> pa, pb;
            tc_pack<double>(ctx, op.U64.get(), op.l, static_cast<int>(op.l), B.src_order.get(), T.a, pa);
            tc_pack<double>(ctx, op.Wt64.get(), op.l, static_cast<int>(op.l), B.tgt_order.get(), T.b, pb);
            TcEpiDelta epi{dlt.get(), op.logk64[b].get(), op.view(static_cast<int>(b)), T.d_a_first.get(),
                           T.d_b_first.get(), maxbits.get(), overflow.get()};
            tc_run(ctx, pa, pb, static_cast<int>(op.l), T.items, epi);
            op.val64.push_back(std::move(dlt));
            continue;
        }
        EpiDelta epi{dlt.get(), op.logk64[b].get(), maxbits.get(), overflow.get()};
        launch_band_tiles<1>(ctx, op.bands[b], op.view(static_cast<int>(b)), op.U64.get(), op.Wt64.get(),
                             static_cast<int>(op.l), epi);
        op.val64.push_back(std::move(dlt));
    }
    if (read_flag(ctx, overflow)) throw Status(3, "build_correction: kernel value overflows linear space");
    unsigned long long mb = 0;
    maxbits.download(&mb, 1, ctx.stream);
    ctx.sync();
    std::memcpy(&op.max_abs_delta, &mb, 8);
}

namespace {
__global__ void to_f32_kernel(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) out[i] = static_cast<float>(in[i]);
}
void to_f32(Ctx& ctx, const DevBuf<double>& in, DevBuf<float>& out, size_t n) {
    out.resize(std::max<size_t>(n, 1));
    if (n) to_f32_kernel<<<std::min<long long>(ceil_div(n, 256), 8 * ctx.num_sms), 256, 0, ctx.stream>>>(in.get(), out.get(), n);
    LAUNCH_OK("to_f32");
}
// rows x l -> rows x lp (zero padded), converted to T
template <typename T>
__global__ void pad_rows_kernel(const double* __restrict__ in, long long rows, int l, int lp, T* __restrict__ out) {
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < rows * lp; e += 256LL * gridDim.x) {
        long long r = e / lp;
        int a = static_cast<int>(e % lp);
        out[e] = a < l ? static_cast<T>(in[r * l + a]) : T(0);
    }
}
template <typename T>
void pad_rows(Ctx& ctx, const DevBuf<double>& in, size_t rows, size_t l, size_t lp, DevBuf<T>& out) {
    out.resize(std::max<size_t>(rows * lp, 1));
    if (rows)
        pad_rows_kernel<T><<<std::min<long long>(ceil_div(rows * lp, 256), 16 * ctx.num_sms), 256, 0, ctx.stream>>>(
            in.get(), rows, static_cast<int>(l), static_cast<int>(lp), out.get());
    LAUNCH_OK("pad_rows");
}
}  // namespace

namespace {
// Transposed copy of every bucket block: out block b is m_b rows x
// row_stride(n_b) (padding columns stay 0 from the memset). 32 x 32 tiles
// through shared memory; one CTA per bucket walks its tiles.
template <typename T>
__global__ void __launch_bounds__(256) transpose_blocks_kernel(const double* __restrict__ in,
                                                               const unsigned long long* __restrict__ blk_off,
                                                               const unsigned long long* __restrict__ blkT_off,
                                                               const uint32_t* __restrict__ src_start,
                                                               const uint32_t* __restrict__ tgt_start,
                                                               T* __restrict__ out) {
    __shared__ double tile[32][33];
    const uint32_t b = blockIdx.x;
    const uint32_t nb = src_start[b + 1] - src_start[b], mb = tgt_start[b + 1] - tgt_start[b];
    if (nb == 0 || mb == 0) return;
    const unsigned long long ms = row_stride(mb), ns = row_stride(nb);
    const double* A = in + blk_off[b];
    T* O = out + blkT_off[b];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (uint32_t i0 = 0; i0 < nb; i0 += 32)
        for (uint32_t j0 = 0; j0 < mb; j0 += 32) {
            __syncthreads();
            for (int r = ty; r < 32; r += 8) {
                const uint32_t i = i0 + r, j = j0 + tx;
                tile[r][tx] = (i < nb && j < mb) ? A[i * ms + j] : 0.0;
            }
            __syncthreads();
            for (int r = ty; r < 32; r += 8) {
                const uint32_t j = j0 + r, i = i0 + tx;
                if (j < mb && i < nb) O[j * ns + i] = static_cast<T>(tile[tx][r]);
            }
        }
}

// ---- iteration layout (BandPanel, op.cuh) ----
__global__ void iter_key_kernel(const uint32_t* __restrict__ b, const uint32_t* __restrict__ b0, long long n,
                                unsigned long long r0, unsigned long long* __restrict__ key) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x)
        key[i] = static_cast<unsigned long long>(b[i]) * r0 + b0[i];
}
__global__ void inv_perm_kernel(const uint32_t* __restrict__ order, long long n, uint32_t* __restrict__ pos) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x)
        pos[order[i]] = static_cast<uint32_t>(i);
}

// One CTA per panel: stored entry (r, c) <- the fp64 block master at the pair
// (stream point of row r, output point c); ROWS: stream = targets.
template <bool ROWS>
__global__ void __launch_bounds__(256) panel_gather_kernel(const double* __restrict__ master,
                                                           const BandPanel* __restrict__ panels,
                                                           const uint32_t* __restrict__ s_order,
                                                           const uint32_t* __restrict__ o_order,
                                                           const uint32_t* __restrict__ src_local,
                                                           const uint32_t* __restrict__ tgt_local,
                                                           const unsigned long long* __restrict__ blk_off,
                                                           const uint32_t* __restrict__ tgt_start,
                                                           float* __restrict__ out) {
    const BandPanel P = panels[blockIdx.x];
    const unsigned long long ms = row_stride(tgt_start[P.bucket + 1] - tgt_start[P.bucket]);
    const double* A = master + blk_off[P.bucket];
    const unsigned long long rs = row_stride(P.ow);
    float* O = out + P.val_off;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c0 = 0; c0 < P.ow; c0 += 32) {
        const uint32_t c = c0 + lane;
        const bool okc = c < P.ow;
        const uint32_t po = okc ? o_order[P.o_base + c] : 0u;
        const uint32_t lo = okc ? (ROWS ? src_local[po] : tgt_local[po]) : 0u;
        for (uint32_t r = warp; r < P.ns; r += 8) {
            const uint32_t sp = r < P.gap0 ? r : r + P.gapn;
            const uint32_t ps = s_order[P.s_base + sp];
            const uint32_t ls = ROWS ? tgt_local[ps] : src_local[ps];
            if (okc) {
                const double v = ROWS ? A[static_cast<unsigned long long>(lo) * ms + ls]
                                      : A[static_cast<unsigned long long>(ls) * ms + lo];
                O[r * rs + c] = static_cast<float>(v);
            }
        }
    }
}

struct Group {
    uint32_t b0, start, count;  // band-0 bucket, first local position, size
};

// runs of equal key in keys[lo, hi) (sorted), local positions relative to lo
void key_groups(const std::vector<unsigned long long>& keys, size_t lo, size_t hi, unsigned long long r0,
                std::vector<Group>& g) {
    g.clear();
    for (size_t i = lo; i < hi;) {
        size_t j = i + 1;
        while (j < hi && keys[j] == keys[i]) ++j;
        g.push_back({static_cast<uint32_t>(keys[i] % r0), static_cast<uint32_t>(i - lo), static_cast<uint32_t>(j - i)});
        i = j;
    }
}

// Panels of one pass over one bucket: outputs `og`, stream groups `sg` (both in
// band-0 order). An output group whose band-0 twin in the stream is big enough
// gets its own panel without those rows; the rest share plain panels.
void bucket_panels(uint32_t bucket, uint32_t s_base, uint32_t ns, uint32_t o_base, const std::vector<Group>& og,
                   const std::vector<Group>& sg, uint32_t min_w, uint32_t min_area, std::vector<BandPanel>& out) {
    size_t j = 0;
    uint32_t run0 = 0, runw = 0;
    auto flush = [&]() {
        if (runw) out.push_back({0ull, bucket, s_base, ns, ns, 0u, o_base + run0, runw, 0u});
        runw = 0;
    };
    for (const Group& g : og) {
        while (j < sg.size() && sg[j].b0 < g.b0) ++j;
        const bool twin = j < sg.size() && sg[j].b0 == g.b0;
        const uint32_t same = twin ? sg[j].count : 0u;
        if (twin && g.count >= min_w && static_cast<unsigned long long>(same) * g.count >= min_area) {
            flush();
            if (ns > same) out.push_back({0ull, bucket, s_base, ns - same, sg[j].start, same, o_base + g.start, g.count, 0u});
            // ns == same: every pair of the group is in band 0; its outputs stay 0
        } else {
            if (!runw) run0 = g.start;
            runw += g.count;
        }
    }
    flush();
}

unsigned env_uint(const char* name, unsigned dflt) {
    const char* v = std::getenv(name);
    return v && *v ? static_cast<unsigned>(std::strtoul(v, nullptr, 10)) : dflt;
}

void iter_order(Ctx& ctx, const uint32_t* d_b, const uint32_t* d_b0, size_t n, unsigned long long r0,
                unsigned long long range, DevBuf<uint32_t>& order, DevBuf<uint32_t>& pos,
                std::vector<unsigned long long>& h_keys) {
    cudaStream_t s = ctx.stream;
    order.resize(n + 16);
    order.zero(s);
    pos.resize(n + 16);
    pos.zero(s);
    h_keys.assign(n, 0ull);
    if (!n) return;
    DevBuf<unsigned long long> key(n), skey(n);
    DevBuf<uint32_t> iota(n);
    const int g = static_cast<int>(std::min<long long>(ceil_div(n, 256), 8 * ctx.num_sms));
    iter_key_kernel<<<g, 256, 0, s>>>(d_b, d_b0, n, r0, key.get());
    iota32_kernel<<<ceil_div(n, 256), 256, 0, s>>>(iota.get(), n);
    int end_bit = 1;
    while (end_bit < 64 && (1ull << end_bit) < range) ++end_bit;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), skey.get(), iota.get(), order.get(), static_cast<int>(n), 0,
                                    end_bit, s);
    DevBuf<unsigned char> t(tmp);
    cub::DeviceRadixSort::SortPairs(t.get(), tmp, key.get(), skey.get(), iota.get(), order.get(), static_cast<int>(n), 0,
                                    end_bit, s);
    inv_perm_kernel<<<g, 256, 0, s>>>(order.get(), n, pos.get());
    skey.download(h_keys.data(), n, s);
    LAUNCH_OK("iter_order");
    ctx.sync();
}
}  // namespace

// Iteration layout of every band (BandPanel, op.cuh). Compact bands (fp32
// storage, bands after the first, LCN_PANELS != 0) get their own orders and
// panel value arrays gathered from the fp64 master; everything else keeps the
// bucket blocks with one plain panel per bucket.
void build_iter_layout(Op& op) {
    Ctx& ctx = *op.ctx;
    PhaseTimer pt(ctx, "band iteration layout (panels)");
    cudaStream_t s = ctx.stream;
    const bool panels_on = env_uint("LCN_PANELS", 1) != 0;
    const uint32_t min_w = env_uint("LCN_PANEL_W", 64), min_area = env_uint("LCN_PANEL_A", 4096);
    op.iter.clear();
    op.iter.resize(op.bands.size());
    for (size_t b = 0; b < op.bands.size(); ++b) {
        const Band& B = op.bands[b];
        BandIter& I = op.iter[b];
        I.compact = panels_on && !op.fp64 && b > 0 && B.n_work > 0;
        if (!I.compact) {
            I.so = B.src_order.get();
            I.to = B.tgt_order.get();
            I.sp = B.src_pos.get();
            I.tp = B.tgt_pos.get();
            for (int pass = 0; pass < 2; ++pass) {
                const bool rows = pass == 0;
                std::vector<BandPanel>& P = I.h_panels[pass];
                P.clear();
                for (size_t k = 0; k < B.nb; ++k) {
                    const uint32_t nbk = B.h_src_start[k + 1] - B.h_src_start[k];
                    const uint32_t mbk = B.h_tgt_start[k + 1] - B.h_tgt_start[k];
                    if (!nbk || !mbk) continue;
                    const uint32_t sl = rows ? mbk : nbk, ol = rows ? nbk : mbk;
                    P.push_back({rows ? B.h_blkT_off[k] : B.h_blk_off[k], static_cast<uint32_t>(k),
                                 rows ? B.h_tgt_start[k] : B.h_src_start[k], sl, sl, 0u,
                                 rows ? B.h_src_start[k] : B.h_tgt_start[k], ol, 0u});
                    I.real[pass] += static_cast<unsigned long long>(sl) * ol;
                }
                I.entries[pass] = rows ? B.entriesT : B.entries;
                if (P.empty()) I.panels[pass].resize(1);  // a band without any two-sided bucket
                else I.panels[pass].upload(P.data(), P.size(), s);
            }
            continue;
        }
        const Band& B0 = op.bands[0];
        const unsigned long long r0 = std::max<size_t>(B0.nb, 1);
        std::vector<unsigned long long> ks, kt;
        iter_order(ctx, B.src_bucket.get(), B0.src_bucket.get(), op.n, r0, B.nb * r0, I.src_order, I.src_pos, ks);
        iter_order(ctx, B.tgt_bucket.get(), B0.tgt_bucket.get(), op.m, r0, B.nb * r0, I.tgt_order, I.tgt_pos, kt);
        I.so = I.src_order.get();
        I.to = I.tgt_order.get();
        I.sp = I.src_pos.get();
        I.tp = I.tgt_pos.get();
        std::vector<Group> sg, tg;
        I.h_panels[0].clear();
        I.h_panels[1].clear();
        for (size_t k = 0; k < B.nb; ++k) {
            const uint32_t s0 = B.h_src_start[k], s1 = B.h_src_start[k + 1];
            const uint32_t t0 = B.h_tgt_start[k], t1 = B.h_tgt_start[k + 1];
            if (s0 == s1 || t0 == t1) continue;
            key_groups(ks, s0, s1, r0, sg);
            key_groups(kt, t0, t1, r0, tg);
            bucket_panels(static_cast<uint32_t>(k), t0, t1 - t0, s0, sg, tg, min_w, min_area, I.h_panels[0]);
            bucket_panels(static_cast<uint32_t>(k), s0, s1 - s0, t0, tg, sg, min_w, min_area, I.h_panels[1]);
        }
        for (int pass = 0; pass < 2; ++pass) {
            unsigned long long off = 0;
            for (BandPanel& p : I.h_panels[pass]) {
                p.val_off = off;
                off = (off + static_cast<unsigned long long>(p.ns) * row_stride(p.ow) + 31ull) & ~31ull;
                I.real[pass] += static_cast<unsigned long long>(p.ns) * p.ow;
            }
            I.entries[pass] = off;
            const std::vector<BandPanel>& P = I.h_panels[pass];
            if (P.empty()) I.panels[pass].resize(1);
            else I.panels[pass].upload(P.data(), P.size(), s);
            DevBuf<float> v(std::max<unsigned long long>(off, 1));
            v.zero(s);
            if (!P.empty()) {
                if (pass == 0)
                    panel_gather_kernel<true><<<static_cast<unsigned>(P.size()), 256, 0, s>>>(
                        op.val64[b].get(), I.panels[0].get(), I.to, I.so, B.src_local.get(), B.tgt_local.get(),
                        B.blk_off.get(), B.tgt_start.get(), v.get());
                else
                    panel_gather_kernel<false><<<static_cast<unsigned>(P.size()), 256, 0, s>>>(
                        op.val64[b].get(), I.panels[1].get(), I.so, I.to, B.src_local.get(), B.tgt_local.get(),
                        B.blk_off.get(), B.tgt_start.get(), v.get());
                LAUNCH_OK("panel_gather");
            }
            if (pass == 0) op.val32T[b] = std::move(v);
            else op.val32[b] = std::move(v);
        }
    }
    ctx.sync();
}

// Iteration copies (fp32 storage, fp64 accumulation;
// fp64 storage in the exact mode). Low-rank factor rows are padded to
// lp = round_up(l, 4) entries so each row starts 16-byte aligned.
void finalize_storage(Op& op) {
    Ctx& ctx = *op.ctx;
    PhaseTimer pt(ctx, "iteration storage (fp32 copies, transposes)");
    op.lp = (op.l + 3) & ~size_t(3);
    // compact bands (build_iter_layout) get panel arrays instead of block copies
    auto compact = [&](size_t b) {
        return (op.kind == 3 || op.kind == 1) && !op.fp64 && b > 0 && op.bands[b].n_work > 0 &&
               env_uint("LCN_PANELS", 1) != 0;
    };
    if (!op.fp64) {
        op.val32.clear();
        for (size_t b = 0; b < op.bands.size(); ++b) {
            DevBuf<float> v;
            if (!compact(b)) to_f32(ctx, op.val64[b], v, op.bands[b].entries);
            op.val32.push_back(std::move(v));
        }
    }
    if (op.kind == 3 || op.kind == 1) {
        // LCN: delta also stored transposed (targets x sources) so the row
        // pass streams its blocks in the same output-stationary order as the
        // column pass (2 x the delta bytes in HBM, same bytes per iteration).
        // Sparse: log K transposed, so the column log-sum-exp reads rows too.
        op.val32T.clear();
        op.val64T.clear();
        for (size_t b = 0; b < op.bands.size(); ++b) {
            const Band& B = op.bands[b];
            if (op.fp64) {
                DevBuf<double> t(std::max<unsigned long long>(B.entriesT, 1));
                t.zero(ctx.stream);
                if (B.nb)
                    transpose_blocks_kernel<double><<<static_cast<unsigned>(B.nb), 256, 0, ctx.stream>>>(
                        op.val64[b].get(), B.blk_off.get(), B.blkT_off.get(), B.src_start.get(), B.tgt_start.get(),
                        t.get());
                op.val64T.push_back(std::move(t));
            } else if (compact(b)) {
                op.val32T.emplace_back();
                continue;
            } else {
                DevBuf<float> t(std::max<unsigned long long>(B.entriesT, 1));
                t.zero(ctx.stream);
                if (B.nb)
                    transpose_blocks_kernel<float><<<static_cast<unsigned>(B.nb), 256, 0, ctx.stream>>>(
                        op.val64[b].get(), B.blk_off.get(), B.blkT_off.get(), B.src_start.get(), B.tgt_start.get(),
                        t.get());
                op.val32T.push_back(std::move(t));
            }
            LAUNCH_OK("transpose_blocks");
        }
        // the LCN band passes and the sparse operator's log-sum-exp passes (fp32)
        if (op.kind == 3 || !op.fp64) build_iter_layout(op);
    }
    if (op.kind >= 2) {
        if (op.fp64) {
            pad_rows<double>(ctx, op.U64, op.n, op.l, op.lp, op.U64p);
            pad_rows<double>(ctx, op.Wt64, op.m, op.l, op.lp, op.Wt64p);
        } else {
            pad_rows<float>(ctx, op.U64, op.n, op.l, op.lp, op.U32);
            pad_rows<float>(ctx, op.Wt64, op.m, op.l, op.lp, op.Wt32);
        }
    }
    ctx.sync();
}

// ---------------------------------------------------------------------------
// CSR export in the reference order (rows ascending, columns ascending,
// unique; NeighborPairs::from_pairs, lsh.cpp:163-177).
// ---------------------------------------------------------------------------
namespace {

struct BandViews {
    BandView v[kMaxBands];
    int bands;
};

__device__ __forceinline__ bool masked_before(const BandSet& bs, int band, uint32_t i, uint32_t j) {
    for (int b = 0; b < band; ++b)
        if (bs.src_bucket[b][i] == bs.tgt_bucket[b][j]) return true;
    return false;
}

__global__ void csr_count_kernel(BandViews bvs, BandSet bs, long long n, uint32_t* __restrict__ counts) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i >= n) return;
    uint32_t cnt = 0;
    for (int b = 0; b < bvs.bands; ++b) {
        const BandView& v = bvs.v[b];
        uint32_t bk = v.src_bucket[i];
        for (uint32_t p = v.tgt_start[bk]; p < v.tgt_start[bk + 1]; ++p)
            if (!masked_before(bs, b, static_cast<uint32_t>(i), v.tgt_order[p])) ++cnt;
    }
    counts[i] = cnt;
}

// k-way merge of the per-band sorted target lists of row i.
__global__ void csr_fill_kernel(BandViews bvs, BandSet bs, long long n, const uint32_t* __restrict__ row_ptr,
                                uint32_t* __restrict__ col) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i >= n) return;
    uint32_t pos[kMaxBands], end[kMaxBands];
    for (int b = 0; b < bvs.bands; ++b) {
        uint32_t bk = bvs.v[b].src_bucket[i];
        pos[b] = bvs.v[b].tgt_start[bk];
        end[b] = bvs.v[b].tgt_start[bk + 1];
    }
    uint32_t out = row_ptr[i];
    while (true) {
        int best = -1;
        uint32_t bj = 0xffffffffu;
        for (int b = 0; b < bvs.bands; ++b) {
            while (pos[b] < end[b] && masked_before(bs, b, static_cast<uint32_t>(i), bvs.v[b].tgt_order[pos[b]])) ++pos[b];
            if (pos[b] < end[b] && bvs.v[b].tgt_order[pos[b]] < bj) { bj = bvs.v[b].tgt_order[pos[b]]; best = b; }
        }
        if (best < 0) break;
        col[out++] = bj;
        ++pos[best];
    }
}

}  // namespace

void build_csr(Op& op, Ctx* on) {
    if (op.csr_ready) return;
    Ctx& ctx = on ? *on : *op.ctx;
    PhaseTimer pt(ctx, "CSR support export");
    cudaStream_t s = ctx.stream;
    const long long n = op.n;
    BandViews bvs{};
    bvs.bands = static_cast<int>(op.bands.size());
    for (int b = 0; b < bvs.bands; ++b) bvs.v[b] = op.view(b);
    DevBuf<uint32_t> counts(std::max<long long>(n, 1));
    op.csr_row_ptr.resize(n + 1);
    op.csr_row_ptr.zero(s);
    if (n && bvs.bands) {
        csr_count_kernel<<<ceil_div(n, 256), 256, 0, s>>>(bvs, op.bandset(), n, counts.get());
        size_t tmp = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tmp, counts.get(), op.csr_row_ptr.get() + 1, n, s);
        DevBuf<unsigned char> t(tmp);
        cub::DeviceScan::InclusiveSum(t.get(), tmp, counts.get(), op.csr_row_ptr.get() + 1, n, s);
        LAUNCH_OK("csr count");
    }
    uint32_t nnz = 0;
    CUDA_OK(cudaMemcpyAsync(&nnz, op.csr_row_ptr.get() + n, 4, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    op.nnz = nnz;
    op.csr_col.resize(std::max<uint32_t>(nnz, 1));
    if (nnz) {
        csr_fill_kernel<<<ceil_div(n, 256), 256, 0, s>>>(bvs, op.bandset(), n, op.csr_row_ptr.get(), op.csr_col.get());
        LAUNCH_OK("csr fill");
    }
    ctx.sync();
    op.csr_ready = true;
}

namespace {
// Value of CSR entry (i, j): the first band sharing the bucket holds it.
__device__ __forceinline__ unsigned long long entry_index(const BandViews& bvs, uint32_t i, uint32_t j, int* band) {
    for (int b = 0; b < bvs.bands; ++b) {
        const BandView& v = bvs.v[b];
        uint32_t bk = v.src_bucket[i];
        if (bk == v.tgt_bucket[j]) {
            *band = b;
            uint32_t mb = v.tgt_start[bk + 1] - v.tgt_start[bk];
            return v.blk_off[bk] + static_cast<unsigned long long>(v.src_local[i]) * row_stride(mb) + v.tgt_local[j];
        }
    }
    *band = -1;
    return 0;
}

struct ValPtrs {
    const double* p[kMaxBands];
};

// which: 0/1/2 read a stored band array (log K, delta, log_sp); 3 recomputes
// (U W)_ij in the reference's sequential order.
__global__ void csr_values_kernel(BandViews bvs, ValPtrs vals, long long n, const uint32_t* __restrict__ row_ptr,
                                  const uint32_t* __restrict__ col, int which, const double* __restrict__ U,
                                  const double* __restrict__ Wt, int l, double* __restrict__ out) {
    long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i >= n) return;
    for (uint32_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        uint32_t j = col[e];
        if (which == 3) {
            double s = 0.0;
            for (int a = 0; a < l; ++a) s = xadd(s, xmul(U[i * l + a], Wt[static_cast<long long>(j) * l + a]));
            out[e] = s;
        } else {
            int b;
            unsigned long long idx = entry_index(bvs, static_cast<uint32_t>(i), j, &b);
            out[e] = vals.p[b][idx];
        }
    }
}
}  // namespace

// CSR-ordered values of the support into device memory (d_vals: nnz).
void csr_values_device(Op& op, int which, double* d_vals) {
    build_csr(op);
    Ctx& ctx = *op.ctx;
    cudaStream_t s = ctx.stream;
    if (op.gcsr && op.nnz && which != 3) {
        if (which == 1 && op.kind != 3) throw Status(2, "export_csr: delta needs an lcn operator");
        const double* src = op.kind == 3 ? (which == 1 ? op.gval.get() : op.glogsp.get()) : op.gval.get();
        CUDA_OK(cudaMemcpyAsync(d_vals, src, op.nnz * 8, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (op.nnz) {
        BandViews bvs{};
        bvs.bands = static_cast<int>(op.bands.size());
        ValPtrs vp{};
        for (int b = 0; b < bvs.bands; ++b) {
            bvs.v[b] = op.view(b);
            if (which == 0) vp.p[b] = op.kind == 1 ? op.val64[b].get() : op.logk64[b].get();
            if (which == 1) vp.p[b] = op.kind == 3 ? op.val64[b].get() : nullptr;
            if (which == 2) vp.p[b] = op.kind == 3 ? op.logk64[b].get() : op.val64[b].get();
        }
        if (which == 1 && op.kind != 3) throw Status(2, "export_csr: delta needs an lcn operator");
        if (which == 3 && op.kind != 3) throw Status(2, "export_csr: nys_vals needs an lcn operator");
        csr_values_kernel<<<ceil_div(op.n, 256), 256, 0, s>>>(bvs, vp, op.n, op.csr_row_ptr.get(), op.csr_col.get(),
                                                              which, op.U64.get(), op.Wt64.get(),
                                                              static_cast<int>(op.l), d_vals);
        LAUNCH_OK("csr values");
    }
}

// ---- general CSR patterns (the staged API from host structs) ----------------
namespace {
// log K at the pairs of a CSR pattern (build_sparse, sparse_kernel.cpp:70-77):
// 0 - c(p_i, q_j) * (1 / lambda), exact sequential fold of cost_value. One
// warp per row, lanes over its entries.
__global__ void sparse_pairs_kernel(const double* __restrict__ X, long long n, int d, int kind, double inv,
                                    const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                    double* __restrict__ out, int* __restrict__ bad) {
    const long long i = (blockIdx.x * 256LL + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const double* x = X + i * d;
    for (uint32_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
        const double* y = X + (n + col[e]) * static_cast<long long>(d);
        const double c = cost_exact(kind, x, y, d);
        if (kind == 2 && isnan(c)) atomicOr(bad, 1);
        out[e] = xsub(0.0, xmul(c, inv));
    }
}

// build_correction (sparse_kernel.cpp:96-109) at a CSR pattern: exact =
// exp(log_sp), nys = sum_a U[i,a] W[a,j] in the reference's sequential order
// (NystromFactors::entry, nystrom.cpp:127-132), delta = exact - nys.
__global__ void correction_pairs_kernel(long long n, int l, const uint32_t* __restrict__ rp,
                                        const uint32_t* __restrict__ col, const double* __restrict__ logsp,
                                        const double* __restrict__ U, const double* __restrict__ Wt,
                                        double* __restrict__ delta, double* __restrict__ nys,
                                        unsigned long long* __restrict__ maxbits, int* __restrict__ overflow) {
    const long long i = (blockIdx.x * 256LL + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    double mx = 0.0;
    for (uint32_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
        const double exact = exp(logsp[e]);
        if (isinf(exact)) {
            atomicOr(overflow, 1);
            continue;
        }
        const double* u = U + i * l;
        const double* w = Wt + static_cast<long long>(col[e]) * l;
        double s = 0.0;
        for (int a = 0; a < l; ++a) s = xadd(s, xmul(u[a], w[a]));
        nys[e] = s;
        delta[e] = xsub(exact, s);
        mx = fmax(mx, fabs(delta[e]));
    }
    mx = warp_max(mx);
    if (lane == 0 && mx > 0.0) atomicMax(maxbits, static_cast<unsigned long long>(__double_as_longlong(mx)));
}
}  // namespace

void build_sparse_pairs(Op& op, const uint32_t* d_rp, const uint32_t* d_col, size_t nnz, double* d_out) {
    Ctx& ctx = *op.ctx;
    if (!(op.lambda > 0.0)) throw Status(2, "build_sparse: lambda must be positive");
    DevBuf<int> bad(1);
    bad.zero(ctx.stream);
    if (op.n && nnz)
        sparse_pairs_kernel<<<static_cast<unsigned>(ceil_div(op.n * 32, 256)), 256, 0, ctx.stream>>>(
            op.X.get(), static_cast<long long>(op.n), static_cast<int>(op.d), op.cost, 1.0 / op.lambda, d_rp, d_col,
            d_out, bad.get());
    LAUNCH_OK("build_sparse pairs");
    if (read_flag(ctx, bad)) throw Status(2, "cosine-derived cost undefined for zero vectors");
}

void correction_pairs(Ctx& ctx, size_t n, size_t l, const uint32_t* d_rp, const uint32_t* d_col, size_t nnz,
                      const double* d_logsp, const double* d_U, const double* d_Wt, double* d_delta, double* d_nys,
                      double* max_abs) {
    DevBuf<unsigned long long> mb(1);
    DevBuf<int> of(1);
    mb.zero(ctx.stream);
    of.zero(ctx.stream);
    if (n && nnz)
        correction_pairs_kernel<<<static_cast<unsigned>(ceil_div(n * 32, 256)), 256, 0, ctx.stream>>>(
            static_cast<long long>(n), static_cast<int>(l), d_rp, d_col, d_logsp, d_U, d_Wt, d_delta, d_nys, mb.get(),
            of.get());
    LAUNCH_OK("build_correction pairs");
    unsigned long long h = 0;
    mb.download(&h, 1, ctx.stream);
    if (read_flag(ctx, of)) throw Status(3, "build_correction: kernel value overflows linear space");
    double v;
    std::memcpy(&v, &h, 8);
    *max_abs = v;
}

// A host CSR pattern as the operator's support (KernelOperator::sparse / lcn):
// the CSC view by the reference's counting sort (build_csc_arrays,
// sparse_kernel.cpp:17-35), values in both orders.
void set_general_csr(Op& op, const uint32_t* h_rp, const uint32_t* h_col, size_t nnz, const double* h_val,
                     const double* h_logsp) {
    Ctx& ctx = *op.ctx;
    cudaStream_t s = ctx.stream;
    const size_t n = op.n, m = op.m;
    if (h_rp[0] != 0 || h_rp[n] != nnz) throw Status(1, "operator: pattern row pointer does not match nnz");
    for (size_t i = 0; i < n; ++i)
        if (h_rp[i + 1] < h_rp[i]) throw Status(2, "operator: pattern row pointer is not monotone");
    std::vector<uint32_t> cp(m + 1, 0), ri(nnz), cur(m);
    std::vector<double> vt(nnz);
    for (size_t e = 0; e < nnz; ++e) {
        if (h_col[e] >= m) throw Status(2, "neighbor pair index out of range");
        ++cp[h_col[e] + 1];
    }
    for (size_t j = 0; j < m; ++j) cp[j + 1] += cp[j];
    std::copy(cp.begin(), cp.end() - 1, cur.begin());
    for (size_t i = 0; i < n; ++i)
        for (uint32_t e = h_rp[i]; e < h_rp[i + 1]; ++e) {
            const uint32_t pos = cur[h_col[e]]++;
            ri[pos] = static_cast<uint32_t>(i);
            vt[pos] = h_val[e];
        }
    op.gcsr = true;
    op.nnz = nnz;
    op.stored = nnz;
    op.csr_row_ptr.upload(h_rp, n + 1, s);
    op.csr_col.resize(std::max<size_t>(nnz, 1));
    op.gval.resize(std::max<size_t>(nnz, 1));
    op.gvalT.resize(std::max<size_t>(nnz, 1));
    op.gri.resize(std::max<size_t>(nnz, 1));
    if (nnz) {
        CUDA_OK(cudaMemcpyAsync(op.csr_col.get(), h_col, nnz * 4, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(op.gval.get(), h_val, nnz * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(op.gvalT.get(), vt.data(), nnz * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(op.gri.get(), ri.data(), nnz * 4, cudaMemcpyHostToDevice, s));
    }
    op.gcp.upload(cp.data(), m + 1, s);
    if (h_logsp) {
        op.glogsp.resize(std::max<size_t>(nnz, 1));
        if (nnz) CUDA_OK(cudaMemcpyAsync(op.glogsp.get(), h_logsp, nnz * 8, cudaMemcpyHostToDevice, s));
    }
    op.csr_ready = true;
    ctx.sync();
}

void export_csr(Op& op, int which, uint32_t* row_ptr, uint32_t* col, double* vals) {
    build_csr(op);
    Ctx& ctx = *op.ctx;
    cudaStream_t s = ctx.stream;
    if (row_ptr) op.csr_row_ptr.download(row_ptr, op.n + 1, s);
    if (col && op.nnz) op.csr_col.download(col, op.nnz, s);
    if (vals && op.nnz) {
        DevBuf<double> dv(op.nnz);
        csr_values_device(op, which, dv.get());
        dv.download(vals, op.nnz, s);
    }
    ctx.sync();
}

}  // namespace lcnb
