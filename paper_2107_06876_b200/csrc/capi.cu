// extern "C" boundary (include/lcn_b200.h). Never throws: every entry point
// converts lcnb::Status / std::exception into an lcn_status and stores the
// message (text identical to the reference exception's what()) on the context.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include <cublas_v2.h>
#include <thread>
#include <nccl.h>

#include "../../include/lcn_b200.h"
#include "kmeans.cuh"
#include "kmeans_tc.cuh"
#include "op.cuh"
#include "shard.h"

using namespace lcnb;

namespace lcnb {
size_t max_bipartite_matching(size_t n, size_t m, const uint32_t* row_ptr, const uint32_t* col);
}

struct lcn_ctx {
    Ctx c;
};
struct lcn_op {
    Op o;
};
struct lcn_pairs {  // NeighborPairs (lsh.hpp:51-60) as CSR
    size_t n = 0, m = 0;
    std::vector<uint32_t> row_ptr, col;
};
struct lcn_result {
    Result r;
    lcn_op* op = nullptr;
    int device = 0;  // the operator may be destroyed first
};

namespace {

thread_local std::string g_orphan_error;

LshParams lsh_params(const lcn_lsh_config* cfg) {
    if (!cfg) throw Status(2, "lsh: null config");
    LshParams p;
    p.scheme = cfg->scheme;
    p.bands = cfg->bands;
    p.rows = cfg->rows_per_band;
    p.buckets = cfg->buckets_per_fn;
    p.iters = cfg->kmeans_iters;
    p.branching = cfg->branching;
    p.seed = cfg->seed;
    return p;
}

template <class F>
int guard(lcn_ctx* ctx, F&& f) {
    std::string* sink = ctx ? &ctx->c.last_error : &g_orphan_error;
    // device temporaries of this call are allocated / freed on its stream
    struct StreamScope {
        cudaStream_t saved;
        explicit StreamScope(cudaStream_t s) : saved(alloc_stream()) { alloc_stream() = s; }
        ~StreamScope() { alloc_stream() = saved; }
    } scope(ctx ? ctx->c.stream : nullptr);
    try {
        if (ctx) ctx->c.activate();
        f();
        return LCN_OK;
    } catch (const Status& e) {
        *sink = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        *sink = "out of host memory";
        return LCN_E_ERROR;
    } catch (const std::exception& e) {
        *sink = e.what();
        return LCN_E_ERROR;
    }
}

// PointSet::validate (geometry.cpp): shape on the host; the finiteness scan of
// the coordinates runs on the device for sets that upload_union takes
// (check_points_shape + upload_union), on the host otherwise.
void check_points_shape(const double* x, size_t n, size_t d, const char* id) {
    if (n == 0 || d == 0) throw Status(2, std::string("point set '") + id + "' is empty");
    if (!x) throw Status(2, std::string("point set '") + id + "' is null");
}
void check_points(const double* x, size_t n, size_t d, const char* id) {
    check_points_shape(x, n, d, id);
    for (size_t i = 0; i < n * d; ++i)
        if (!std::isfinite(x[i])) throw Status(2, std::string("point set '") + id + "' has non-finite coordinates");
}

// fp32 copy of the union, whether the demotion is exact (flag bit 0), and the
// finiteness of each side's coordinates (bit 1: p, bit 2: q; split = n d)
__global__ void demote_check_kernel(const double* __restrict__ in, float* __restrict__ out, long long n,
                                    long long split, unsigned* __restrict__ inexact) {
    unsigned bad = 0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
        const double v = in[i];
        const float f = static_cast<float>(v);
        out[i] = f;
        if (static_cast<double>(f) != v) bad |= 1u;
        if (!isfinite(v)) bad |= i < split ? 2u : 4u;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(inexact, bad);
}

void upload_union(Op& op, const double* p, size_t n, const double* q, size_t m, size_t d) {
    op.n = n;
    op.m = m;
    op.d = d;
    op.X.resize((n + m) * d);
    CUDA_OK(cudaMemcpyAsync(op.X.get(), p, n * d * 8, cudaMemcpyHostToDevice, op.ctx->stream));
    CUDA_OK(cudaMemcpyAsync(op.X.get() + n * d, q, m * d * 8, cudaMemcpyHostToDevice, op.ctx->stream));
    // fp32 copy for the k-means reads when the promotion is exact, made and
    // checked on the device (no host pass over the points)
    const long long cnt = static_cast<long long>((n + m) * d);
    op.X32.resize(cnt);
    DevBuf<unsigned> inexact(1);
    inexact.zero(op.ctx->stream);
    demote_check_kernel<<<static_cast<int>(std::min<long long>(ceil_div(cnt, 256), 8LL * op.ctx->num_sms)), 256, 0,
                          op.ctx->stream>>>(op.X.get(), op.X32.get(), cnt, static_cast<long long>(n * d),
                                            inexact.get());
    LAUNCH_OK("demote_check");
    unsigned h = 0;
    inexact.download(&h, 1, op.ctx->stream);
    op.ctx->sync();
    if (h & 2u) throw Status(2, "point set 'p' has non-finite coordinates");
    if (h & 4u) throw Status(2, "point set 'q' has non-finite coordinates");
    if (h & 1u) op.X32 = DevBuf<float>();
}

__global__ void promote_kernel(const float* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) out[i] = static_cast<double>(in[i]);
}

void check_cost_lambda(int cost, double lambda, const char* who) {
    if (cost < 0 || cost > 3) throw Status(2, "unknown cost kind");
    if (!(lambda > 0.0)) throw Status(2, std::string(who) + ": lambda must be positive");
}

// Bands from device bucket ids of the union (ids[b]: n+m entries).
void bands_from_union_ids(Op& op, std::vector<DevBuf<uint32_t>>& ids, size_t range) {
    op.bands.clear();
    op.bands.resize(ids.size());
    for (size_t b = 0; b < ids.size(); ++b)
        build_band_layout(*op.ctx, op.bands[b], ids[b].get(), ids[b].get() + op.n, op.n, op.m, range);
}

// Host bucket ids (bands x n, bands x m) -> dense device ids.
void shard_lcn(Op& o, std::vector<DevBuf<uint32_t>>& ids, size_t range, const double* h_landmarks, int method,
               uint64_t seed);
void bands_from_host_ids(Op& op, const uint64_t* ids_p, const uint64_t* ids_q, int bands, uint64_t range,
                         bool shard = false, const double* h_landmarks = nullptr, int method = 0, uint64_t seed = 0) {
    if (bands < 0 || bands > kMaxBands) throw Status(2, "neighbor_pairs: band count out of range");
    std::vector<DevBuf<uint32_t>> ids;
    size_t dense_range = 0;
    for (int b = 0; b < bands; ++b) {
        const uint64_t* bp = ids_p + static_cast<size_t>(b) * op.n;
        const uint64_t* bq = ids_q + static_cast<size_t>(b) * op.m;
        // compress to dense bucket indices preserving order (sorted_by_bucket
        // groups equal ids, lsh.cpp:193-208; only equality matters for pairs)
        std::vector<uint64_t> all(bp, bp + op.n);
        all.insert(all.end(), bq, bq + op.m);
        std::vector<uint64_t> uniq = all;
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        if (range && !uniq.empty() && uniq.back() >= range) throw Status(2, "neighbor_pairs: bucket id out of range");
        std::vector<uint32_t> dense(all.size());
        for (size_t i = 0; i < all.size(); ++i)
            dense[i] = static_cast<uint32_t>(std::lower_bound(uniq.begin(), uniq.end(), all[i]) - uniq.begin());
        DevBuf<uint32_t> d(std::max<size_t>(dense.size(), 1));
        d.upload(dense.data(), dense.size(), op.ctx->stream);
        ids.push_back(std::move(d));
        dense_range = std::max(dense_range, uniq.size());
    }
    op.ctx->sync();
    if (shard && op.ctx->comm) {
        shard_lcn(op, ids, std::max<size_t>(dense_range, 1), h_landmarks, method, seed);
        return;
    }
    op.bands.clear();
    op.bands.resize(bands);
    for (int b = 0; b < bands; ++b)
        build_band_layout(*op.ctx, op.bands[b], ids[b].get(), ids[b].get() + op.n, op.n, op.m, std::max<size_t>(dense_range, 1));
}

// ---- bucket-sharded LCN build (plan in shard.cpp) --------
template <typename T>
__global__ void gather_points_kernel(const T* __restrict__ X, const uint32_t* __restrict__ idx, long long rows, int d,
                                     long long base, T* __restrict__ out) {
    const long long total = rows * d;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < total; e += 256LL * gridDim.x) {
        const long long r = e / d, k = e - r * d;
        out[e] = X[(base + idx[r]) * d + k];
    }
}

// local bucket ids of one band: ids of the global union gathered by the
// local -> global map; halo points (k >= own) go to halo_id when given
__global__ void gather_ids_kernel(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ idx, long long cnt,
                                  long long base, long long own, uint32_t halo_id, uint32_t* __restrict__ out) {
    for (long long k = blockIdx.x * 256LL + threadIdx.x; k < cnt; k += 256LL * gridDim.x)
        out[k] = (k >= own && halo_id != 0xffffffffu) ? halo_id : ids[base + idx[k]];
}

// Support size of the whole problem from the bucket ids (the local operators
// hold only their blocks): band b adds the pairs of its buckets that no
// earlier band holds, by inclusion-exclusion over the earlier bands.
unsigned long long global_support(const std::vector<uint32_t>& is, const std::vector<uint32_t>& it, size_t n, size_t m,
                                  int bands) {
    auto mixk = [](uint64_t x) {
        x += 0x9E3779B97F4A7C15ull;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        return x ^ (x >> 31);
    };
    // pairs sharing the buckets of every band in `mask`
    auto shared = [&](unsigned mask) {
        std::vector<uint64_t> ks(n), kt(m);
        auto key = [&](const std::vector<uint32_t>& ids, size_t cnt, size_t i) {
            uint64_t h = 0;
            for (int b = 0; b < bands; ++b)
                if (mask >> b & 1u) h = mixk(h ^ (uint64_t(b) << 40) ^ ids[b * cnt + i]);
            return h;
        };
        for (size_t i = 0; i < n; ++i) ks[i] = key(is, n, i);
        for (size_t j = 0; j < m; ++j) kt[j] = key(it, m, j);
        std::sort(ks.begin(), ks.end());
        std::sort(kt.begin(), kt.end());
        unsigned long long tot = 0;
        size_t a = 0, c = 0;
        while (a < n && c < m) {
            if (ks[a] < kt[c]) ++a;
            else if (kt[c] < ks[a]) ++c;
            else {
                size_t a2 = a, c2 = c;
                while (a2 < n && ks[a2] == ks[a]) ++a2;
                while (c2 < m && kt[c2] == kt[c]) ++c2;
                tot += static_cast<unsigned long long>(a2 - a) * (c2 - c);
                a = a2;
                c = c2;
            }
        }
        return tot;
    };
    long long nnz = 0;
    for (unsigned mask = 1; mask < (1u << bands); ++mask)
        nnz += (__builtin_popcount(mask) & 1 ? 1LL : -1LL) * static_cast<long long>(shared(mask));
    return static_cast<unsigned long long>(nnz);
}

// Replace the whole-problem op (union points uploaded, device bucket ids of
// every band computed on this rank, landmarks in o.L when landmarks_ready)
// by this rank's shard of it and build the shard's LCN operator.
void shard_lcn(Op& o, std::vector<DevBuf<uint32_t>>& ids, size_t range, const double* h_landmarks, int method,
               uint64_t seed) {
    Ctx& ctx = *o.ctx;
    cudaStream_t s = ctx.stream;
    const size_t n = o.n, m = o.m, d = o.d, N = n + m;
    const int bands = static_cast<int>(ids.size());
    if (bands < 1) throw Status(2, "sharded solve: the LCN operator needs at least one LSH band");
    if (range + 2 > 0xffffffffull) throw Status(2, "sharded solve: bucket range too large");
    if (h_landmarks) {
        o.L.resize(o.l * d);
        o.L.upload(h_landmarks, o.l * d, s);
        o.landmarks_ready = true;
    } else if (!o.landmarks_ready) {
        select_landmarks_device(o, ctx, method, seed);  // the whole problem's landmarks
        o.landmarks_ready = true;
    }
    PhaseTimer pt(ctx, "shard plan + local points");
    std::vector<uint32_t> hid(static_cast<size_t>(bands) * N);
    for (int b = 0; b < bands; ++b) ids[b].download(hid.data() + static_cast<size_t>(b) * N, N, s);
    ctx.sync();
    std::vector<uint32_t> is(static_cast<size_t>(bands) * n), it(static_cast<size_t>(bands) * m);
    for (int b = 0; b < bands; ++b) {
        std::copy(hid.begin() + static_cast<size_t>(b) * N, hid.begin() + static_cast<size_t>(b) * N + n,
                  is.begin() + static_cast<size_t>(b) * n);
        std::copy(hid.begin() + static_cast<size_t>(b) * N + n, hid.begin() + static_cast<size_t>(b + 1) * N,
                  it.begin() + static_cast<size_t>(b) * m);
    }
    std::vector<uint32_t> rng(bands, static_cast<uint32_t>(range));
    ShardPlan P = make_shard_plan(is.data(), n, it.data(), m, bands, rng.data(), o.l, ctx.world());
    const ShardRank& R = P.ranks[ctx.rank()];
    auto st = std::make_shared<ShardState>();
    st->comm = ctx.comm;
    st->rank = ctx.rank();
    st->world = ctx.world();
    st->n_glob = n;
    st->m_glob = m;
    st->n_own = R.n_own;
    st->m_own = R.m_own;
    st->bands = bands;
    st->ids_src = is;  // the support size is computed on first request (lcn_op_get_info)
    st->ids_tgt = it;
    st->src_glob = R.src;
    st->tgt_glob = R.tgt;
    st->n_halo = R.src.size() - R.n_own;
    st->m_halo = R.tgt.size() - R.m_own;
    // a rank with no local point on a side (more ranks than band-0 groups, or
    // one-sided groups) gets one phantom point there, after the halo, in no
    // shared bucket: the local operator is never empty, and the phantom is
    // neither owned nor imported, so nothing reads its values
    const bool ph_s = R.src.empty(), ph_t = R.tgt.empty();
    if (ph_s) st->src_glob.push_back(0u);
    if (ph_t) st->tgt_glob.push_back(0u);
    st->n_exp_s = R.exp_s.size();
    st->n_exp_t = R.exp_t.size();
    st->max_exp_s = P.max_exp_s;
    st->max_exp_t = P.max_exp_t;
    st->groups = P.groups;
    st->cost = R.cost;
    for (const ShardRank& Q : P.ranks) {
        st->own_src_all.emplace_back(Q.src.begin(), Q.src.begin() + Q.n_own);
        st->own_tgt_all.emplace_back(Q.tgt.begin(), Q.tgt.begin() + Q.m_own);
    }
    st->rows_need.assign(bands, std::vector<uint8_t>(range + 2, 0));
    st->cols_need.assign(bands, std::vector<uint8_t>(range + 2, 0));
    for (int b = 0; b < bands; ++b) {
        for (uint32_t k = 0; k < R.n_own; ++k) st->rows_need[b][is[static_cast<size_t>(b) * n + R.src[k]]] = 1;
        for (uint32_t k = 0; k < R.m_own; ++k) st->cols_need[b][it[static_cast<size_t>(b) * m + R.tgt[k]]] = 1;
    }
    auto up = [&](DevBuf<uint32_t>& dst, const std::vector<uint32_t>& v) {
        dst.resize(std::max<size_t>(v.size(), 1));
        if (!v.empty()) dst.upload(v.data(), v.size(), s);
    };
    up(st->d_src_glob, st->src_glob);
    up(st->d_tgt_glob, st->tgt_glob);
    up(st->exp_s, R.exp_s);
    up(st->exp_t, R.exp_t);
    up(st->imp_s_rank, R.imp_s_rank);
    up(st->imp_s_slot, R.imp_s_slot);
    up(st->imp_t_rank, R.imp_t_rank);
    up(st->imp_t_slot, R.imp_t_slot);
    // local points: sources then targets of the local union
    const long long nl = static_cast<long long>(st->src_glob.size()), ml = static_cast<long long>(st->tgt_glob.size());
    const int gb = static_cast<int>(std::min<long long>(ceil_div((nl + ml) * static_cast<long long>(d), 256), 8LL * ctx.num_sms)) + 1;
    DevBuf<double> X(std::max<size_t>((nl + ml) * d, 1));
    gather_points_kernel<double><<<gb, 256, 0, s>>>(o.X.get(), st->d_src_glob.get(), nl, static_cast<int>(d), 0, X.get());
    gather_points_kernel<double><<<gb, 256, 0, s>>>(o.X.get(), st->d_tgt_glob.get(), ml, static_cast<int>(d),
                                                    static_cast<long long>(n), X.get() + nl * d);
    DevBuf<float> X32;
    if (o.X32.size()) {
        X32.resize(std::max<size_t>((nl + ml) * d, 1));
        gather_points_kernel<float><<<gb, 256, 0, s>>>(o.X32.get(), st->d_src_glob.get(), nl, static_cast<int>(d), 0,
                                                       X32.get());
        gather_points_kernel<float><<<gb, 256, 0, s>>>(o.X32.get(), st->d_tgt_glob.get(), ml, static_cast<int>(d),
                                                       static_cast<long long>(n), X32.get() + nl * d);
    }
    std::vector<DevBuf<uint32_t>> lids(bands);
    for (int b = 0; b < bands; ++b) {
        lids[b].resize(std::max<long long>(nl + ml, 1));
        const uint32_t hs = b == 0 ? static_cast<uint32_t>(range) : 0xffffffffu;
        const uint32_t ht = b == 0 ? static_cast<uint32_t>(range + 1) : 0xffffffffu;
        gather_ids_kernel<<<gb, 256, 0, s>>>(ids[b].get(), st->d_src_glob.get(), nl, 0, R.n_own, hs, lids[b].get());
        gather_ids_kernel<<<gb, 256, 0, s>>>(ids[b].get(), st->d_tgt_glob.get(), ml, static_cast<long long>(n), R.m_own,
                                             ht, lids[b].get() + nl);
    }
    LAUNCH_OK("shard gather");
    // phantoms: their own bucket in every later band (range + 1; band 0 has
    // the one-sided halo buckets already)
    for (int b = 1; b < bands; ++b) {
        const uint32_t lone = static_cast<uint32_t>(range + 1);
        if (ph_s) CUDA_OK(cudaMemcpyAsync(lids[b].get() + nl - 1, &lone, 4, cudaMemcpyHostToDevice, s));
        if (ph_t) CUDA_OK(cudaMemcpyAsync(lids[b].get() + nl + ml - 1, &lone, 4, cudaMemcpyHostToDevice, s));
    }
    ctx.sync();
    ids.clear();
    o.X = std::move(X);
    o.X32 = std::move(X32);
    o.norms = DevBuf<double>();
    o.n = static_cast<size_t>(nl);
    o.m = static_cast<size_t>(ml);
    bands_from_union_ids(o, lids, range + 2);
    o.shard = st;
}

void finish_sparse(Op& op) {
    op.kind = LCN_OP_SPARSE;
    build_sparse_values(op);
    build_csr(op);
    finalize_storage(op);
}

void finish_lcn(Op& op, const double* landmarks, size_t l, int method, uint64_t seed) {
    op.l = l;
    op.kind = op.bands.empty() ? LCN_OP_NYSTROM : LCN_OP_LCN;
    if (op.kind == LCN_OP_LCN && !op.ctx->comm)
        op.during_ldlt = [&op] {  // overlapped with the host LDL^T
            build_sparse_values(op);
            op.logk64 = std::move(op.val64);
            op.val64.clear();
            build_csr(op);
        };
    build_nystrom(op, landmarks, method, seed);
    op.during_ldlt = nullptr;
    if (op.kind == LCN_OP_LCN) {
        if (!op.csr_ready && !op.ctx->comm) {
            // the CSR support needs only the bands: a host thread builds it on
            // its own stream while this one runs the correction (K_sp, delta)
            Ctx side = *op.ctx;
            side.own_stream = nullptr;
            side.comm.reset();
            side.cublas = nullptr;
            CUDA_OK(cudaStreamCreateWithFlags(&side.stream, cudaStreamNonBlocking));
            std::exception_ptr cerr, serr;
            std::thread th([&] {
                try {
                    CUDA_OK(cudaSetDevice(side.device));
                    alloc_stream() = side.stream;
                    build_csr(op, &side);
                    side.sync();
                } catch (...) {
                    serr = std::current_exception();
                }
            });
            try {
                build_correction(op);
            } catch (...) {
                cerr = std::current_exception();
            }
            th.join();
            cudaStreamDestroy(side.stream);
            if (cerr) std::rethrow_exception(cerr);
            if (serr) std::rethrow_exception(serr);
        } else {
            build_correction(op);
            build_csr(op);
        }
    }
    finalize_storage(op);
}

lcn_op* new_op(lcn_ctx* ctx, int cost, double lambda) {
    auto* h = new lcn_op();
    h->o.ctx = &ctx->c;
    h->o.cost = cost;
    h->o.lambda = lambda;
    h->o.fp64 = ctx->c.store_fp64 != 0;
    return h;
}

}  // namespace

extern "C" {

int lcn_abi_version(void) { return LCN_B200_ABI_VERSION; }

const char* lcn_status_name(int s) {
    switch (s) {
        case LCN_OK: return "ok";
        case LCN_E_DIMENSION: return "DimensionError";
        case LCN_E_INVALID_ARGUMENT: return "InvalidArgument";
        case LCN_E_STABILIZATION: return "StabilizationError";
        case LCN_E_NEGATIVE_KERNEL: return "NegativeKernelError";
        case LCN_E_FACTORIZATION: return "FactorizationError";
        case LCN_E_ERROR: return "Error";
        case LCN_E_CUDA: return "CudaError";
        case LCN_E_NO_DEVICE: return "NoDevice";
    }
    return "Unknown";
}

int lcn_ctx_create(int device, int flags, lcn_ctx** out) {
    return guard(nullptr, [&] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) throw Status(LCN_E_NO_DEVICE, "no CUDA device");
        if (device < 0 || device >= count) throw Status(LCN_E_NO_DEVICE, "device index out of range");
        cudaDeviceProp prop{};
        CUDA_OK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw Status(LCN_E_NO_DEVICE, "this build targets sm_100a (B200)");
        auto c = std::make_unique<lcn_ctx>();
        c->c.device = device;
        c->c.store_fp64 = (flags & LCN_STORE_FP64) ? 1 : 0;
        c->c.exact_build = (flags & LCN_EXACT_BUILD) || std::getenv("LCN_EXACT_BUILD") ? 1 : 0;
        c->c.dense_recompute = (flags & LCN_DENSE_RECOMPUTE) ? 1 : 0;
        c->c.num_sms = prop.multiProcessorCount;
        CUDA_OK(cudaSetDevice(device));
        // keep freed pool memory resident (stream-ordered DevBuf temporaries)
        cudaMemPool_t pool;
        CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = ~0ull;
        CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        CUDA_OK(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
        // LCN_POOL_RESERVE_GB: map that much into the pool up front (one
        // allocation, freed at once and kept). A build's multi-GB buffers
        // are then carved from resident memory instead of growing the pool
        // (mapping fresh memory mid-build cost 0.1-0.25 s per configs[3]
        // build whenever the job threads' allocation order fragmented it).
        if (const char* rv = std::getenv("LCN_POOL_RESERVE_GB")) {
            const double gb = std::atof(rv);
            uint64_t have = 0;
            CUDA_OK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have));
            const size_t want = gb > 0 ? static_cast<size_t>(gb * 1073741824.0) : 0;
            if (want > have) {
                void* p = nullptr;
                if (cudaMallocAsync(&p, want - have, c->c.stream) == cudaSuccess) {
                    CUDA_OK(cudaFreeAsync(p, c->c.stream));
                } else {
                    cudaGetLastError();  // not enough free memory: skip the reservation
                }
                CUDA_OK(cudaStreamSynchronize(c->c.stream));
            }
        }
        c->c.own_stream = c->c.stream;
        *out = c.release();
    });
}

int lcn_ctx_destroy(lcn_ctx* ctx) {
    if (!ctx) return LCN_OK;
    cudaSetDevice(ctx->c.device);
    cudaDeviceSynchronize();
    ctx->c.comm.reset();
    if (ctx->c.cublas) cublasDestroy(static_cast<cublasHandle_t>(ctx->c.cublas));
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.own_stream);
    delete ctx;
    return LCN_OK;
}

int lcn_ctx_set_stream(lcn_ctx* ctx, void* stream) {
    if (!ctx) return LCN_E_INVALID_ARGUMENT;
    ctx->c.stream = stream ? static_cast<cudaStream_t>(stream) : ctx->c.own_stream;
    return LCN_OK;
}

int lcn_nccl_unique_id(uint8_t* out128) {
    return guard(nullptr, [&] {
        if (!out128) throw Status(2, "null id buffer");
        ncclUniqueId id;
        if (ncclGetUniqueId(&id) != ncclSuccess) throw Status(LCN_E_CUDA, "ncclGetUniqueId failed");
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(out128, &id, 128);
    });
}

int lcn_ctx_set_comm(lcn_ctx* ctx, int world, int rank, const uint8_t* id128) {
    return guard(ctx, [&] {
        if (!ctx || !id128) throw Status(2, "null context or id");
        if (world < 1 || rank < 0 || rank >= world) throw Status(2, "rank / world out of range");
        ctx->c.comm.reset();
        ctx->c.comm = make_nccl_comm(world, rank, id128);
    });
}

int lcn_loopback_create(int world, lcn_loopback** out) {
    return guard(nullptr, [&] {
        if (!out) throw Status(2, "null output");
        if (world < 1 || world > 64) throw Status(2, "rank / world out of range");
        *out = reinterpret_cast<lcn_loopback*>(new std::shared_ptr<LoopbackGroup>(std::make_shared<LoopbackGroup>(world)));
    });
}

int lcn_loopback_abort(lcn_loopback* lb) {
    if (!lb) return LCN_E_INVALID_ARGUMENT;
    (*reinterpret_cast<std::shared_ptr<LoopbackGroup>*>(lb))->abort();
    return LCN_OK;
}

int lcn_loopback_destroy(lcn_loopback* lb) {
    delete reinterpret_cast<std::shared_ptr<LoopbackGroup>*>(lb);
    return LCN_OK;
}

int lcn_ctx_set_loopback(lcn_ctx* ctx, lcn_loopback* lb, int rank) {
    return guard(ctx, [&] {
        if (!ctx || !lb) throw Status(2, "null context or loopback group");
        auto& g = *reinterpret_cast<std::shared_ptr<LoopbackGroup>*>(lb);
        if (rank < 0 || rank >= g->world) throw Status(2, "rank / world out of range");
        ctx->c.comm = make_loopback_comm(g, rank);
    });
}

int lcn_ctx_set_profile(lcn_ctx* ctx, int on) {
    if (!ctx) return LCN_E_INVALID_ARGUMENT;
    ctx->c.profile = on ? 1 : 0;
    return LCN_OK;
}

const char* lcn_ctx_last_error(const lcn_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : g_orphan_error.c_str(); }

// fp32 copy of host points when every coordinate is fp32-representable (the
// k-means kernels then read 4-byte points; distances are the same fp64 folds)
static bool fp32_copy(const double* p, size_t count, std::vector<float>& f) {
    f.resize(count);
    for (size_t i = 0; i < count; ++i)
        if (static_cast<double>(f[i] = static_cast<float>(p[i])) != p[i]) return false;
    return true;
}

int lcn_kmeans_pp_indices(lcn_ctx* ctx, const double* points, size_t n, size_t d, size_t k, uint64_t first_index,
                          const uint64_t* raw_draws, size_t n_draws, uint32_t* out, size_t* draws_used) {
    return guard(ctx, [&] {
        if (k == 0 || k > n) throw Status(2, "kmeans++: k must be in [1, n]");
        if (first_index >= n) throw Status(2, "kmeans++: first index out of range");
        std::vector<unsigned long long> raw(raw_draws, raw_draws + n_draws);
        DevBuf<uint32_t> ch(k);
        int used = 0;
        std::vector<float> f;
        if (fp32_copy(points, n * d, f)) {
            DevBuf<float> X32;
            X32.upload(f.data(), f.size(), ctx->c.stream);
            kmeans_pp_device<float>(ctx->c, X32.get(), n, static_cast<int>(d), static_cast<int>(k), first_index, raw,
                                    ch.get(), &used);
        } else {
            DevBuf<double> X;
            X.upload(points, n * d, ctx->c.stream);
            kmeans_pp_device<double>(ctx->c, X.get(), n, static_cast<int>(d), static_cast<int>(k), first_index, raw,
                                     ch.get(), &used);
        }
        ch.download(out, k, ctx->c.stream);
        ctx->c.sync();
        if (draws_used) *draws_used = static_cast<size_t>(used);
    });
}

int lcn_assign_nearest(lcn_ctx* ctx, const double* points, size_t n, size_t d, const double* centroids, size_t k,
                       uint32_t* out) {
    return guard(ctx, [&] {
        DevBuf<double> X, C;
        DevBuf<uint32_t> a(std::max<size_t>(n, 1));
        C.upload(centroids, k * d, ctx->c.stream);
        std::vector<float> f;
        if (fp32_copy(points, n * d, f)) {
            DevBuf<float> X32;
            X32.upload(f.data(), f.size(), ctx->c.stream);
            assign_device<float>(ctx->c, X32.get(), n, static_cast<int>(d), C.get(), static_cast<int>(k), a.get());
            a.download(out, n, ctx->c.stream);
            ctx->c.sync();
            return;
        }
        X.upload(points, n * d, ctx->c.stream);
        assign_device<double>(ctx->c, X.get(), n, static_cast<int>(d), C.get(), static_cast<int>(k), a.get());
        a.download(out, n, ctx->c.stream);
        ctx->c.sync();
    });
}

// Test hook (not part of the solver API): raw tensor-core accumulators of the
// first centroid tile (64 centroids) for the first 128 points of an fp32
// point set; hh_only = 1 issues only the x_hi . c_hi products.
extern "C" int lcn_debug_tc_scores(lcn_ctx* ctx, const float* points, size_t n, size_t d, const double* centroids,
                                   size_t k, int hh_only, float* acc_out) {
    return guard(ctx, [&] {
        DevBuf<float> X;
        DevBuf<double> C;
        X.upload(points, n * d, ctx->c.stream);
        C.upload(centroids, k * d, ctx->c.stream);
        DevBuf<uint32_t> out(std::max<size_t>(n, 1)), amb(std::max<size_t>(n, 1));
        DevBuf<unsigned> namb(1);
        DevBuf<float> dbg(128 * 64);
        namb.zero(ctx->c.stream);
        dbg.zero(ctx->c.stream);
        if (!assign_filter_tc(ctx->c, X.get(), n, static_cast<int>(d), C.get(), static_cast<int>(k), out.get(),
                              amb.get(), namb.get(), dbg.get(), hh_only))
            throw Status(2, "shape not handled by the tensor-core filter");
        dbg.download(acc_out, 128 * 64, ctx->c.stream);
        ctx->c.sync();
    });
}

int lcn_ctx_tc_work(lcn_ctx* ctx, int reset, unsigned long long* point_tiles) {
    return guard(ctx, [&] {
        if (!point_tiles) throw Status(2, "lcn_ctx_tc_work: null output");
        CUDA_OK(cudaSetDevice(ctx->c.device));
        *point_tiles = tc_point_tiles(reset != 0);
    });
}

int lcn_lloyd(lcn_ctx* ctx, const double* points, size_t n, size_t d, size_t k, int iters, uint64_t seed,
              double* centroids_out, uint32_t* assign_out) {
    return guard(ctx, [&] {
        if (n == 0) throw Status(2, "k-means on empty input");
        if (k == 0 || k > n) throw Status(2, "k-means: more buckets than points");
        DevBuf<double> X, C(k * d);
        DevBuf<float> X32;
        DevBuf<uint32_t> a(n);
        std::vector<float> f;
        if (fp32_copy(points, n * d, f)) {
            X32.upload(f.data(), f.size(), ctx->c.stream);
            lloyd_device<float>(ctx->c, X32.get(), n, static_cast<int>(d), static_cast<int>(k), iters, seed, C.get(),
                                a.get());
        } else {
            X.upload(points, n * d, ctx->c.stream);
            lloyd_device<double>(ctx->c, X.get(), n, static_cast<int>(d), static_cast<int>(k), iters, seed, C.get(),
                                 a.get());
        }
        C.download(centroids_out, k * d, ctx->c.stream);
        a.download(assign_out, n, ctx->c.stream);
        ctx->c.sync();
    });
}

int lcn_cross_polytope_buckets(lcn_ctx* ctx, const double* points, size_t n, size_t d, const double* proj,
                               size_t half, uint32_t* out) {
    return guard(ctx, [&] {
        if (!proj || half == 0) throw Status(2, "cross_polytope_bucket: empty projection");
        check_points(points, n, d, "points");
        if (n == 0) return;
        DevBuf<double> X(n * d);
        X.upload(points, n * d, ctx->c.stream);
        DevBuf<uint32_t> o(n);
        cross_polytope_buckets_device(ctx->c, X.get(), static_cast<long long>(n), static_cast<int>(d), proj,
                                      static_cast<int>(half), o.get());
        o.download(out, n, ctx->c.stream);
        ctx->c.sync();
    });
}

int lcn_lsh_kmeans_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                           const lcn_lsh_config* cfg, uint64_t* ids_out) {
    return lcn_lsh_buckets(ctx, p, n, q, m, d, cfg, ids_out);
}

int lcn_lsh_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                    const lcn_lsh_config* cfg, uint64_t* ids_out) {
    return guard(ctx, [&] {
        if (!cfg) throw Status(2, "lsh: null config");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        Op tmp;
        tmp.ctx = &ctx->c;
        upload_union(tmp, p, n, q, m, d);
        std::vector<DevBuf<uint32_t>> ids;
        size_t range = 0;
        lsh_bucket_ids(ctx->c, tmp.X.get(), tmp.X32.size() ? tmp.X32.get() : nullptr, n, m, d, lsh_params(cfg), ids, range);
        std::vector<uint32_t> h(n + m);
        for (size_t b = 0; b < ids.size(); ++b) {
            ids[b].download(h.data(), n + m, ctx->c.stream);
            ctx->c.sync();
            for (size_t i = 0; i < n + m; ++i) ids_out[b * (n + m) + i] = h[i];
        }
    });
}

int lcn_op_sparse_lsh(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                      double lambda, const lcn_lsh_config* cfg, lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_sparse");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        upload_union(h->o, p, n, q, m, d);
        std::vector<DevBuf<uint32_t>> ids;
        size_t range = 0;
        lsh_bucket_ids(ctx->c, h->o.X.get(), h->o.X32.size() ? h->o.X32.get() : nullptr, n, m, d, lsh_params(cfg), ids, range);
        if (static_cast<int>(ids.size()) > kMaxBands) throw Status(2, "lsh: at most 8 bands on this path");
        bands_from_union_ids(h->o, ids, range);
        finish_sparse(h->o);
        *out = h.release();
    });
}

// ---- staged build from host structs (runner.cpp:258-271) -------------------
int lcn_lsh_neighbor_pairs(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                           const lcn_lsh_config* cfg, lcn_pairs** out) {
    return guard(ctx, [&] {
        if (!out) throw Status(2, "null output");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, 0, 1.0));
        upload_union(h->o, p, n, q, m, d);
        std::vector<DevBuf<uint32_t>> ids;
        size_t range = 0;
        lsh_bucket_ids(ctx->c, h->o.X.get(), h->o.X32.size() ? h->o.X32.get() : nullptr, n, m, d, lsh_params(cfg), ids,
                       range);
        if (static_cast<int>(ids.size()) > kMaxBands) throw Status(2, "lsh: at most 8 bands on this path");
        bands_from_union_ids(h->o, ids, range);
        build_csr(h->o);
        auto pr = std::make_unique<lcn_pairs>();
        pr->n = n;
        pr->m = m;
        pr->row_ptr.resize(n + 1);
        pr->col.resize(h->o.nnz);
        export_csr(h->o, 0, pr->row_ptr.data(), pr->col.data(), nullptr);
        *out = pr.release();
    });
}

int lcn_pairs_info(const lcn_pairs* pr, size_t* n, size_t* m, size_t* nnz) {
    if (!pr) return LCN_E_INVALID_ARGUMENT;
    if (n) *n = pr->n;
    if (m) *m = pr->m;
    if (nnz) *nnz = pr->col.size();
    return LCN_OK;
}

int lcn_pairs_copy(const lcn_pairs* pr, uint32_t* row_ptr, uint32_t* col) {
    if (!pr) return LCN_E_INVALID_ARGUMENT;
    if (row_ptr) std::memcpy(row_ptr, pr->row_ptr.data(), pr->row_ptr.size() * 4);
    if (col && !pr->col.empty()) std::memcpy(col, pr->col.data(), pr->col.size() * 4);
    return LCN_OK;
}

int lcn_pairs_destroy(lcn_pairs* pr) {
    delete pr;
    return LCN_OK;
}

int lcn_build_sparse(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                     const uint32_t* row_ptr, const uint32_t* col, size_t nnz, int cost, double lambda,
                     double* logvals) {
    return guard(ctx, [&] {
        if (!(lambda > 0.0)) throw Status(2, "build_sparse: lambda must be positive");
        if (cost < 0 || cost > 3) throw Status(2, "unknown cost kind");
        if (!row_ptr || (nnz && (!col || !logvals))) throw Status(2, "null pattern");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        if (row_ptr[n] != nnz) throw Status(1, "build_sparse: pattern shape mismatch");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        upload_union(h->o, p, n, q, m, d);
        cudaStream_t s = ctx->c.stream;
        for (size_t e = 0; e < nnz; ++e)
            if (col[e] >= m) throw Status(2, "neighbor pair index out of range");
        DevBuf<uint32_t> rp, cl(std::max<size_t>(nnz, 1));
        DevBuf<double> out(std::max<size_t>(nnz, 1));
        rp.upload(row_ptr, n + 1, s);
        if (nnz) CUDA_OK(cudaMemcpyAsync(cl.get(), col, nnz * 4, cudaMemcpyHostToDevice, s));
        build_sparse_pairs(h->o, rp.get(), cl.get(), nnz, out.get());
        out.download(logvals, nnz, s);
        ctx->c.sync();
    });
}

int lcn_select_landmarks(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, size_t l,
                         int method, uint64_t seed, double* out) {
    return guard(ctx, [&] {
        if (!out) throw Status(2, "null output");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        if (l < 1 || l > n + m) throw Status(2, "select_landmarks: l out of range");
        std::unique_ptr<lcn_op> h(new_op(ctx, 0, 1.0));
        upload_union(h->o, p, n, q, m, d);
        h->o.l = l;
        select_landmarks_device(h->o, ctx->c, method, seed);
        h->o.L.download(out, l * d, ctx->c.stream);
        ctx->c.sync();
    });
}

int lcn_build_factors(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                      const double* landmarks, size_t l, int cost, double lambda, double* U, double* W, double* cond) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_factors");
        if (!landmarks || !U || !W) throw Status(2, "null argument");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        h->o.fp64 = true;  // exact fp64 blocks (the reference's values, not the 3xTF32 iteration build)
        upload_union(h->o, p, n, q, m, d);
        h->o.l = l;
        build_nystrom(h->o, landmarks, 0, 0);
        h->o.U64.download(U, n * l, ctx->c.stream);
        std::vector<double> wt(m * l);
        h->o.Wt64.download(wt.data(), m * l, ctx->c.stream);
        ctx->c.sync();
        for (size_t a = 0; a < l; ++a)
            for (size_t j = 0; j < m; ++j) W[a * m + j] = wt[j * l + a];
        if (cond) *cond = h->o.cond;
    });
}

int lcn_build_correction(lcn_ctx* ctx, size_t n, size_t m, size_t l, const uint32_t* row_ptr, const uint32_t* col,
                         size_t nnz, const double* log_sp, const double* U, const double* W, double* delta,
                         double* nys_vals, double* max_abs_delta) {
    return guard(ctx, [&] {
        if (!row_ptr || !U || !W || (nnz && (!col || !log_sp || !delta))) throw Status(2, "null argument");
        if (row_ptr[n] != nnz) throw Status(1, "build_correction: shape mismatch");
        for (size_t e = 0; e < nnz; ++e)
            if (col[e] >= m) throw Status(1, "build_correction: shape mismatch");
        cudaStream_t s = ctx->c.stream;
        std::vector<double> wt(m * l);
        for (size_t a = 0; a < l; ++a)
            for (size_t j = 0; j < m; ++j) wt[j * l + a] = W[a * m + j];
        DevBuf<uint32_t> rp, cl(std::max<size_t>(nnz, 1));
        DevBuf<double> ls(std::max<size_t>(nnz, 1)), du, dw, dd(std::max<size_t>(nnz, 1)), dn(std::max<size_t>(nnz, 1));
        rp.upload(row_ptr, n + 1, s);
        du.upload(U, std::max<size_t>(n * l, 1), s);
        dw.upload(wt.data(), std::max<size_t>(m * l, 1), s);
        if (nnz) {
            CUDA_OK(cudaMemcpyAsync(cl.get(), col, nnz * 4, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(ls.get(), log_sp, nnz * 8, cudaMemcpyHostToDevice, s));
        }
        double mx = 0.0;
        correction_pairs(ctx->c, n, l, rp.get(), cl.get(), nnz, ls.get(), du.get(), dw.get(), dd.get(), dn.get(), &mx);
        if (nnz) {
            dd.download(delta, nnz, s);
            if (nys_vals) dn.download(nys_vals, nnz, s);
        }
        ctx->c.sync();
        if (max_abs_delta) *max_abs_delta = mx;
    });
}

int lcn_op_from_dense(lcn_ctx* ctx, size_t n, size_t m, const double* logk, double lambda, lcn_op** out) {
    return guard(ctx, [&] {
        if (!(lambda > 0.0)) throw Status(2, "dense operator: lambda must be positive");
        if (!logk || !out) throw Status(2, "null argument");
        std::unique_ptr<lcn_op> h(new_op(ctx, 0, lambda));
        Op& o = h->o;
        o.kind = LCN_OP_DENSE;
        o.n = n;
        o.m = m;
        o.dk64.upload(logk, std::max<size_t>(n * m, 1), ctx->c.stream);
        dense_storage(o);
        *out = h.release();
    });
}

int lcn_op_from_sparse(lcn_ctx* ctx, size_t n, size_t m, const uint32_t* row_ptr, const uint32_t* col, size_t nnz,
                       const double* logvals, double lambda, lcn_op** out) {
    return guard(ctx, [&] {
        if (!(lambda > 0.0)) throw Status(2, "sparse operator: lambda must be positive");
        if (!row_ptr || !out || (nnz && (!col || !logvals))) throw Status(2, "null argument");
        std::unique_ptr<lcn_op> h(new_op(ctx, 0, lambda));
        Op& o = h->o;
        o.kind = LCN_OP_SPARSE;
        o.n = n;
        o.m = m;
        set_general_csr(o, row_ptr, col, nnz, logvals, nullptr);
        *out = h.release();
    });
}

// NystromFactors (nystrom.hpp:33-44) onto the device: U, W^T and their
// iteration copies.
void factors_from_host(Op& o, size_t l, const double* U, const double* W) {
    cudaStream_t s = o.ctx->stream;
    o.l = l;
    std::vector<double> wt(o.m * l);
    for (size_t a = 0; a < l; ++a)
        for (size_t j = 0; j < o.m; ++j) wt[j * l + a] = W[a * o.m + j];
    o.U64.upload(U, std::max<size_t>(o.n * l, 1), s);
    o.Wt64.upload(wt.data(), std::max<size_t>(o.m * l, 1), s);
    o.ctx->sync();
}

int lcn_op_from_nystrom(lcn_ctx* ctx, size_t n, size_t m, size_t l, const double* U, const double* W, double lambda,
                        lcn_op** out) {
    return guard(ctx, [&] {
        if (!U || !W || !out) throw Status(2, "null argument");
        if (l < 1 || l > 4096) throw Status(2, "nystrom operator: landmark count out of range");
        std::unique_ptr<lcn_op> h(new_op(ctx, 0, lambda));
        Op& o = h->o;
        o.kind = LCN_OP_NYSTROM;
        o.n = n;
        o.m = m;
        factors_from_host(o, l, U, W);
        finalize_storage(o);
        *out = h.release();
    });
}

int lcn_op_from_lcn(lcn_ctx* ctx, size_t n, size_t m, size_t l, const double* U, const double* W, double lambda,
                    const uint32_t* row_ptr, const uint32_t* col, size_t nnz, const double* delta,
                    const double* log_sp, double max_abs_delta, lcn_op** out) {
    return guard(ctx, [&] {
        if (!U || !W || !out || !row_ptr || (nnz && (!col || !delta || !log_sp))) throw Status(2, "null argument");
        if (l < 1 || l > 4096) throw Status(2, "lcn operator: landmark count out of range");
        std::unique_ptr<lcn_op> h(new_op(ctx, 0, lambda));
        Op& o = h->o;
        o.kind = LCN_OP_LCN;
        o.n = n;
        o.m = m;
        factors_from_host(o, l, U, W);
        set_general_csr(o, row_ptr, col, nnz, delta, log_sp);
        o.max_abs_delta = max_abs_delta;
        finalize_storage(o);
        *out = h.release();
    });
}

int lcn_op_sparse_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                          double lambda, const uint64_t* ids_p, const uint64_t* ids_q, int bands, uint64_t range,
                          lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_sparse");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        upload_union(h->o, p, n, q, m, d);
        bands_from_host_ids(h->o, ids_p, ids_q, bands, range);
        finish_sparse(h->o);
        *out = h.release();
    });
}

int lcn_op_lcn_lsh(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                   double lambda, const lcn_lsh_config* cfg, size_t l, int landmark_method, uint64_t landmark_seed,
                   lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_factors");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        upload_union(h->o, p, n, q, m, d);
        std::vector<DevBuf<uint32_t>> ids;
        size_t range = 0;
        Op& o = h->o;
        o.l = l;
        // (building the Nystrom factors on this job too, concurrently with the
        // LSH k-means, measured slower: 1.32 s vs 1.28 s per build at
        // configs[3] -- the factor GEMMs and the host LDL^T contend with the
        // seeding chains)
        // the landmark k-means and the Nystrom factors (they need no LSH
        // ids) run on their own job from the start, beside the bands'
        // seeding chain (LCN_EARLY_FACTORS=0: landmarks seeded with the
        // bands in one batched chain, factors after the LSH)
        const char* efenv = std::getenv("LCN_EARLY_FACTORS");
        const bool early = !ctx->c.comm && !(efenv && efenv[0] == '0') && l >= 1 && l <= n + m;
        auto landmarks_job = [&](Ctx& jc) {
            select_landmarks_device(o, jc, landmark_method, landmark_seed);
            o.landmarks_ready = true;
            if (early) build_nystrom(o, nullptr, landmark_method, landmark_seed, &jc);
        };
        ExtraSeeding es;
        if (!early && landmark_method == 0 && l >= 1 && l <= n + m) {  // k-means landmarks: seeded with the bands
            o.landmark_init.resize(l);
            es = ExtraSeeding{static_cast<int>(l), landmark_seed, o.landmark_init.get()};
        }
        lsh_bucket_ids(ctx->c, o.X.get(), o.X32.size() ? o.X32.get() : nullptr, n, m, d, lsh_params(cfg), ids, range,
                              landmarks_job, &es, early);
        if (ctx->c.comm) shard_lcn(o, ids, range, nullptr, landmark_method, landmark_seed);
        else bands_from_union_ids(o, ids, range);
        finish_lcn(o, nullptr, l, landmark_method, landmark_seed);
        *out = h.release();
    });
}

int lcn_op_lcn_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                       double lambda, const uint64_t* ids_p, const uint64_t* ids_q, int bands, uint64_t range,
                       const double* landmarks, size_t l, int landmark_method, uint64_t landmark_seed, lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_factors");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        upload_union(h->o, p, n, q, m, d);
        h->o.l = l;
        bands_from_host_ids(h->o, ids_p, ids_q, bands, range, true, landmarks, landmark_method, landmark_seed);
        finish_lcn(h->o, h->o.shard ? nullptr : landmarks, l, landmark_method, landmark_seed);
        *out = h.release();
    });
}

int lcn_op_dense(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                 double lambda, lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_cost");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        upload_union(h->o, p, n, q, m, d);
        h->o.kind = LCN_OP_DENSE;
        if (ctx->c.dense_recompute && !h->o.fp64) dense_tc_prepare(h->o);
        else build_dense(h->o);
        *out = h.release();
    });
}

int lcn_op_dense_device(lcn_ctx* ctx, const float* d_p, size_t n, const float* d_q, size_t m, size_t d, int cost,
                        double lambda, lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, "build_cost");
        if (n == 0 || m == 0 || d == 0) throw Status(2, "point set is empty");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        Op& op = h->o;
        op.n = n;
        op.m = m;
        op.d = d;
        op.X.resize((n + m) * d);
        promote_kernel<<<std::min<long long>(ceil_div(n * d, 256), 8 * ctx->c.num_sms), 256, 0, ctx->c.stream>>>(
            d_p, op.X.get(), n * d);
        promote_kernel<<<std::min<long long>(ceil_div(m * d, 256), 8 * ctx->c.num_sms), 256, 0, ctx->c.stream>>>(
            d_q, op.X.get() + n * d, m * d);
        LAUNCH_OK("promote");
        op.kind = LCN_OP_DENSE;
        if (ctx->c.dense_recompute && !op.fp64) dense_tc_prepare(op);
        else build_dense(op);
        *out = h.release();
    });
}

int lcn_multihead(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                  double lambda, int heads, const double* pmarg, const double* qmarg,
                  const lcn_sinkhorn_options* opts, double* lambdas_out, double* dist_out, int* iters_out,
                  int* converged_out, int* status_out) {
    return guard(ctx, [&] {
        // multihead_lambdas (sinkhorn.cpp:322-331)
        if (heads < 1) throw Status(2, "multihead: heads must be >= 1");
        if (!(lambda > 0.0)) throw Status(2, "multihead: lambda must be positive");
        check_cost_lambda(cost, lambda, "build_cost");
        check_points_shape(p, n, d, "p");
        check_points_shape(q, m, d, "q");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        Op& op = h->o;
        upload_union(op, p, n, q, m, d);
        op.kind = LCN_OP_DENSE;
        build_dense_cost(op);
        SolveOptions so;
        if (opts) {
            so.tol = opts->tol;
            so.max_iters = opts->max_iters;
            so.check_support = false;
            so.want_plan = false;
        }
        std::string last_err;
        // multihead (sinkhorn.cpp:333-353): independent solves, per-head errors
        for (int k = 1; k <= heads; ++k) {
            const double lam_k = std::exp2(static_cast<double>(k) - static_cast<double>(heads) / 2.0) * lambda;
            const int i = k - 1;
            lambdas_out[i] = lam_k;
            dist_out[i] = 0.0;
            iters_out[i] = 0;
            converged_out[i] = 0;
            status_out[i] = LCN_OK;
            try {
                dense_logk_from_cost(op, lam_k);
                Result r;
                sinkhorn_solve(op, pmarg, qmarg, false, so, r);
                dist_out[i] = r.distance;
                iters_out[i] = r.iters;
                converged_out[i] = r.converged ? 1 : 0;
            } catch (const Status& e) {
                status_out[i] = e.code;
                last_err = e.what();
            }
        }
        if (!last_err.empty()) ctx->c.last_error = last_err;
    });
}

int lcn_op_export_dense(lcn_op* op, double* out) {
    lcn_ctx* ctx = op ? reinterpret_cast<lcn_ctx*>(op->o.ctx) : nullptr;
    return guard(ctx, [&] {
        if (!op || !out) throw Status(2, "null operator or buffer");
        if (op->o.kind != LCN_OP_DENSE) throw Status(2, "export_dense: not a dense operator");
        if (op->o.dense_tc) {  // recomputed operator: the exact log K on demand
            build_dense(op->o);
            op->o.dk64.download(out, op->o.n * op->o.m, op->o.ctx->stream);
            op->o.ctx->sync();
            op->o.dk64 = DevBuf<double>();
            op->o.dk32 = DevBuf<float>();
            op->o.dk32T = DevBuf<float>();
            op->o.dk64T = DevBuf<double>();
            return;
        }
        op->o.dk64.download(out, op->o.n * op->o.m, op->o.ctx->stream);
        op->o.ctx->sync();
    });
}

int lcn_op_create_device(lcn_ctx* ctx, const float* d_p, size_t n, const float* d_q, size_t m, size_t d, int cost,
                         double lambda, const lcn_lsh_config* cfg, size_t l, int landmark_method,
                         uint64_t landmark_seed, lcn_op** out) {
    return guard(ctx, [&] {
        check_cost_lambda(cost, lambda, l ? "build_factors" : "build_sparse");
        std::unique_ptr<lcn_op> h(new_op(ctx, cost, lambda));
        Op& op = h->o;
        op.n = n;
        op.m = m;
        op.d = d;
        op.X.resize((n + m) * d);
        op.X32.resize((n + m) * d);
        CUDA_OK(cudaMemcpyAsync(op.X32.get(), d_p, n * d * 4, cudaMemcpyDeviceToDevice, ctx->c.stream));
        CUDA_OK(cudaMemcpyAsync(op.X32.get() + n * d, d_q, m * d * 4, cudaMemcpyDeviceToDevice, ctx->c.stream));
        promote_kernel<<<std::min<long long>(ceil_div(n * d, 256), 8 * ctx->c.num_sms), 256, 0, ctx->c.stream>>>(
            d_p, op.X.get(), n * d);
        promote_kernel<<<std::min<long long>(ceil_div(m * d, 256), 8 * ctx->c.num_sms), 256, 0, ctx->c.stream>>>(
            d_q, op.X.get() + n * d, m * d);
        LAUNCH_OK("promote");
        std::vector<DevBuf<uint32_t>> ids;
        size_t range = 0;
        op.l = l;
        const char* efenv = std::getenv("LCN_EARLY_FACTORS");
        const bool early = l && !ctx->c.comm && !(efenv && efenv[0] == '0') && l <= n + m;  // see lcn_op_lcn_lsh
        std::function<void(Ctx&)> landmarks_job;
        if (l)
            landmarks_job = [&](Ctx& jc) {
                select_landmarks_device(op, jc, landmark_method, landmark_seed);
                op.landmarks_ready = true;
                if (early) build_nystrom(op, nullptr, landmark_method, landmark_seed, &jc);
            };
        ExtraSeeding es;
        if (l && !early && landmark_method == 0 && l <= n + m) {  // k-means landmarks: seeded with the bands
            op.landmark_init.resize(l);
            es = ExtraSeeding{static_cast<int>(l), landmark_seed, op.landmark_init.get()};
        }
        lsh_bucket_ids(ctx->c, op.X.get(), op.X32.size() ? op.X32.get() : nullptr, n, m, d, lsh_params(cfg), ids, range,
                              landmarks_job, &es, early);
        if (ctx->c.comm && l) shard_lcn(op, ids, range, nullptr, landmark_method, landmark_seed);
        else bands_from_union_ids(op, ids, range);
        if (l) finish_lcn(op, nullptr, l, landmark_method, landmark_seed);
        else finish_sparse(op);
        *out = h.release();
    });
}

int lcn_batched_lcn(lcn_ctx* ctx, const double* X, size_t rows, size_t d, int nprob, const int* n, const int* m,
                    int cost, double lambda, int buckets, int kmeans_iters, const uint64_t* lsh_seeds, size_t l,
                    const uint64_t* landmark_seeds, int iters, double* distance_out, int* status_out,
                    int* iters_out) {
    return guard(ctx, [&] {
        if (nprob < 0 || (nprob > 0 && (!X || !n || !m || !lsh_seeds || !landmark_seeds || !distance_out || !status_out)))
            throw Status(2, "batched LCN: null argument");
        if (iters < 1) throw Status(2, "sinkhorn: max_iters must be >= 1");
        if (nprob == 0) return;
        bool finite = true;
#pragma omp parallel for schedule(static) reduction(&& : finite)
        for (long long i = 0; i < static_cast<long long>(rows * d); ++i) finite = finite && std::isfinite(X[i]);
        if (!finite) throw Status(2, "point set has a non-finite coordinate");
        batched_lcn(ctx->c, X, rows, static_cast<int>(d), nprob, n, m, cost, lambda, buckets, kmeans_iters, lsh_seeds,
                    static_cast<int>(l), landmark_seeds, iters, distance_out, status_out, iters_out);
    });
}

int lcn_op_destroy(lcn_op* op) {
    if (!op) return LCN_OK;
    cudaSetDevice(op->o.ctx->device);
    cudaDeviceSynchronize();  // any stream may still read the operator
    // free on the context's stream: the pool hands the blocks straight back to
    // the next build on that stream (frees on another stream are only reused
    // opportunistically, and the pool grows instead)
    cudaStream_t saved = alloc_stream();
    alloc_stream() = op->o.ctx->stream;
    delete op;
    alloc_stream() = saved;
    return LCN_OK;
}

int lcn_op_set_bp(lcn_op* op, const double* del_p, const double* del_q) {
    lcn_ctx* ctx = op ? reinterpret_cast<lcn_ctx*>(op->o.ctx) : nullptr;
    return guard(ctx, [&] {
        if (!op) throw Status(2, "null operator");
        Op& o = op->o;
        if (!del_p && !del_q) {
            o.bp = false;
            return;
        }
        if (!del_p || !del_q) throw Status(1, "with_bp: deletion vector length mismatch");
        if (o.shard) throw Status(2, "with_bp: the BP extension is not available on a sharded operator");
        std::vector<double> lp(o.n), lq(o.m);
        for (size_t i = 0; i < o.n; ++i) {
            if (!(del_p[i] >= 0.0) || !std::isfinite(del_p[i]))
                throw Status(2, "with_bp: deletion kernels must be finite and nonnegative");
            lp[i] = std::log(del_p[i]);
        }
        for (size_t j = 0; j < o.m; ++j) {
            if (!(del_q[j] >= 0.0) || !std::isfinite(del_q[j]))
                throw Status(2, "with_bp: deletion kernels must be finite and nonnegative");
            lq[j] = std::log(del_q[j]);
        }
        o.bp_ldp.upload(lp.data(), o.n, o.ctx->stream);
        o.bp_ldq.upload(lq.data(), o.m, o.ctx->stream);
        o.ctx->sync();
        o.bp = true;
    });
}

int lcn_op_get_info(const lcn_op* op, lcn_op_info_t* info) {
    if (!op || !info) return LCN_E_INVALID_ARGUMENT;
    const Op& o = op->o;
    info->kind = o.kind;
    info->n = o.n_glob();
    info->m = o.m_glob();
    info->l = o.l;
    info->d = o.d;
    info->bands = static_cast<int>(o.bands.size());
    info->nnz = o.nnz;
    info->stored = o.stored;
    info->lambda = o.lambda;
    info->max_abs_delta = o.max_abs_delta;
    info->cond_estimate = o.cond;
    info->store_fp64 = o.fp64 ? 1 : 0;
    info->streamed = o.stored;
    if (o.kind == 3 && o.iter.size() == o.bands.size()) {
        info->streamed = 0;
        for (const auto& I : o.iter) info->streamed += I.real[1];
    }
    if (o.shard) {  // stored / streamed stay this rank's
        ShardState& sh = *const_cast<Op&>(o).shard;
        if (!sh.ids_src.empty()) {
            sh.nnz_glob = global_support(sh.ids_src, sh.ids_tgt, sh.n_glob, sh.m_glob, sh.bands);
            sh.ids_src.clear();
            sh.ids_src.shrink_to_fit();
            sh.ids_tgt.clear();
            sh.ids_tgt.shrink_to_fit();
        }
        info->nnz = sh.nnz_glob;
    }
    return LCN_OK;
}

int lcn_op_export_csr(lcn_op* op, int which, uint32_t* row_ptr, uint32_t* col, double* vals) {
    lcn_ctx* ctx = reinterpret_cast<lcn_ctx*>(op->o.ctx);  // Ctx is the first member of lcn_ctx
    return guard(ctx, [&] {
        if (op->o.shard) throw Status(2, "export_csr: a sharded operator holds only its rank's blocks");
        export_csr(op->o, which, row_ptr, col, vals);
    });
}

int lcn_op_export_factor(lcn_op* op, int which, double* out) {
    lcn_ctx* ctx = reinterpret_cast<lcn_ctx*>(op->o.ctx);
    return guard(ctx, [&] {
        Op& o = op->o;
        if (o.kind < 2 && which != 2) throw Status(2, "export_factor: operator has no low-rank factors");
        if (o.shard && which != 2) throw Status(2, "export_factor: a sharded operator holds only its rank's factor rows");
        cudaStream_t s = o.ctx->stream;
        if (which == 0) {
            o.U64.download(out, o.n * o.l, s);
        } else if (which == 1) {
            std::vector<double> wt(o.m * o.l);
            o.Wt64.download(wt.data(), o.m * o.l, s);
            o.ctx->sync();
            for (size_t a = 0; a < o.l; ++a)
                for (size_t j = 0; j < o.m; ++j) out[a * o.m + j] = wt[j * o.l + a];
        } else if (which == 2) {
            o.L.download(out, o.l * o.d, s);
        } else {
            throw Status(2, "export_factor: unknown factor");
        }
        o.ctx->sync();
    });
}

int lcn_op_log_matvec(lcn_op* op, const double* in, int transposed, double* out) {
    lcn_ctx* ctx = reinterpret_cast<lcn_ctx*>(op->o.ctx);
    return guard(ctx, [&] { op_log_matvec(op->o, in, transposed != 0, out); });
}

int lcn_sinkhorn(lcn_op* op, const double* p, const double* q, const lcn_sinkhorn_options* opts, lcn_result** out) {
    lcn_ctx* ctx = reinterpret_cast<lcn_ctx*>(op->o.ctx);
    return guard(ctx, [&] {
        Op& o = op->o;
        // Marginals::validate(balanced) (geometry.cpp:97-111)
        if (!p || !q || o.n == 0 || o.m == 0) throw Status(2, "marginals must be non-empty");
        double sp = 0.0, sq = 0.0;
        for (size_t i = 0; i < o.n_glob(); ++i) {
            if (!(p[i] > 0.0) || !std::isfinite(p[i])) throw Status(2, "marginal p has a non-positive or non-finite entry");
            sp += p[i];
        }
        for (size_t j = 0; j < o.m_glob(); ++j) {
            if (!(q[j] > 0.0) || !std::isfinite(q[j])) throw Status(2, "marginal q has a non-positive or non-finite entry");
            sq += q[j];
        }
        if (!o.bp && std::abs(sp - sq) > 1e-12 * std::max(sp, sq))  // validate(balanced = !has_bp)
            throw Status(2, "marginals are unbalanced; balanced OT requires equal mass");
        SolveOptions so;
        if (opts) {
            so.tol = opts->tol;
            so.max_iters = opts->max_iters;
            so.check_support = opts->check_support != 0;
            so.want_plan = opts->want_plan != 0;
        }
        if (o.shard && so.want_plan)
            throw Status(2, "extract_plan: the plan of a sharded operator is distributed over the ranks; "
                            "pass want_plan = 0");
        auto res = std::make_unique<lcn_result>();
        res->op = op;
        res->device = op->o.ctx->device;
        if (o.kind == LCN_OP_SPARSE && so.check_support && !o.bp) {  // sinkhorn.cpp:122 (!op.has_bp())
            // sinkhorn.cpp:122-128: warn when the pattern has no support
            // (maximum bipartite matching < min(n, m), sparse_kernel.cpp:189-196).
            // Band 1's pattern is a disjoint union of complete bipartite
            // blocks, whose maximum matching is sum_b min(n_b, m_b): exact for
            // one band, a lower bound of the union otherwise. Only a union
            // whose band-1 bound falls short needs the general matching.
            const size_t small = std::min(o.n, o.m);
            bool support = o.nnz > 0;
            if (support && !o.bands.empty()) {
                const Band& B0 = o.bands[0];
                unsigned long long mb = 0;
                for (size_t b = 0; b + 1 < B0.h_src_start.size(); ++b)
                    mb += std::min(B0.h_src_start[b + 1] - B0.h_src_start[b], B0.h_tgt_start[b + 1] - B0.h_tgt_start[b]);
                if (mb >= small) support = true;
                else if (o.bands.size() == 1) support = false;
                else support = [&] {
                    build_csr(o);
                    std::vector<uint32_t> rp(o.n + 1), col(std::max<unsigned long long>(o.nnz, 1));
                    export_csr(o, 0, rp.data(), col.data(), nullptr);
                    return max_bipartite_matching(o.n, o.m, rp.data(), col.data()) >= small;
                }();
            } else if (support) {
                build_csr(o);
                std::vector<uint32_t> rp(o.n + 1), col(std::max<unsigned long long>(o.nnz, 1));
                export_csr(o, 0, rp.data(), col.data(), nullptr);
                support = max_bipartite_matching(o.n, o.m, rp.data(), col.data()) >= small;
            }
            if (!support) {
                res->r.warnings.push_back("sparse kernel pattern has no support; Sinkhorn may not converge");
                std::fprintf(stderr, "lcn: warning: %s\n", res->r.warnings.back().c_str());
            }
        }
        if (o.bp) sinkhorn_solve_bp(o, p, q, so, res->r);
        else sinkhorn_solve(o, p, q, false, so, res->r);
        if (so.want_plan) extract_plan_device(o, res->r);  // sinkhorn.cpp:23-100 (base block under BP)
        *out = res.release();
    });
}

int lcn_sinkhorn_device(lcn_op* op, const double* d_p, const double* d_q, const lcn_sinkhorn_options* opts,
                        lcn_result** out) {
    lcn_ctx* ctx = reinterpret_cast<lcn_ctx*>(op->o.ctx);
    return guard(ctx, [&] {
        SolveOptions so;
        if (opts) {
            so.tol = opts->tol;
            so.max_iters = opts->max_iters;
            so.check_support = opts->check_support != 0;
            so.want_plan = false;
        }
        if (op->o.bp)  // the device entry solves the balanced base problem only
            throw Status(2, "lcn_sinkhorn_device: BP-extended operators need lcn_sinkhorn (host marginals)");
        auto res = std::make_unique<lcn_result>();
        res->op = op;
        res->device = op->o.ctx->device;
        sinkhorn_solve(op->o, d_p, d_q, true, so, res->r);
        *out = res.release();
    });
}

int lcn_result_phase_ms(const lcn_result* res, double* out4, int* iters) {
    if (!res || !out4) return LCN_E_INVALID_ARGUMENT;
    for (int k = 0; k < 4; ++k) out4[k] = k < static_cast<int>(res->r.phase_ms.size()) ? res->r.phase_ms[k] : 0.0;
    if (iters) *iters = res->r.phase_iters;
    return LCN_OK;
}

int lcn_result_destroy(lcn_result* res) {
    if (!res) return LCN_OK;
    cudaSetDevice(res->device);
    cudaDeviceSynchronize();
    delete res;
    return LCN_OK;
}

int lcn_result_get_info(const lcn_result* res, lcn_result_info_t* info) {
    if (!res || !info) return LCN_E_INVALID_ARGUMENT;
    info->distance = res->r.distance;
    info->iters = res->r.iters;
    info->converged = res->r.converged ? 1 : 0;
    info->marginal_err_final = res->r.marginal_err_final;
    info->n_warnings = static_cast<int>(res->r.warnings.size());
    info->device_ms = res->r.device_ms;
    return LCN_OK;
}

int lcn_result_copy(const lcn_result* res, int which, double* out, size_t* len) {
    if (!res) return LCN_E_INVALID_ARGUMENT;
    const Result& r = res->r;
    const std::vector<double>* v = nullptr;
    switch (which) {
        case 0: v = &r.log_s; break;
        case 1: v = &r.log_t; break;
        case 2: v = &r.row_marg; break;
        case 3: v = &r.err_trace; break;
        case 4: v = &r.plan_vals; break;
        case 5: v = &r.sp_vals; break;
        case 6: v = &r.sp_nys_vals; break;
        case 7: v = &r.del_p_mass; break;
        case 8: v = &r.del_q_mass; break;
        case 9:
            if (len) *len = 1;
            if (out) *out = r.eps_mass;
            return LCN_OK;
        default: return LCN_E_INVALID_ARGUMENT;
    }
    if (len) *len = v->size();
    if (out && !v->empty()) std::memcpy(out, v->data(), v->size() * sizeof(double));
    return LCN_OK;
}

int lcn_distance_lcn(const lcn_result* res, const lcn_op* op, double* out) {
    lcn_ctx* ctx = reinterpret_cast<lcn_ctx*>(op->o.ctx);
    return guard(ctx, [&] {
        if (op->o.kind < 2) throw Status(2, "distance_lcn: operator has no low-rank factors");
        if (op->o.shard) throw Status(2, "distance_lcn: not available on a sharded operator");
        *out = distance_lcn_device(const_cast<lcn_op*>(op)->o, res->r);
    });
}

// ---- grad_cost (sinkhorn.cpp:263-320) -----------------------------------
namespace {
// v[a] = sum_r F[r][a] x_r (F rows x l, fp64), one thread per column a, rows
// split over gridDim.y blocks; each block writes its partial to
// part[blockIdx.y * l + a] and colsum_combine_kernel adds them in block
// order, so the gradients are bit-identical run to run (as distance_lcn)
__global__ void colsum_kernel(const double* __restrict__ F, long long rows, int l, const double* __restrict__ x,
                              double* __restrict__ part) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= l) return;
    const long long per = (rows + gridDim.y - 1) / gridDim.y;
    const long long r0 = static_cast<long long>(blockIdx.y) * per, r1 = r0 + per < rows ? r0 + per : rows;
    double acc = 0.0;
    for (long long r = r0; r < r1; ++r) acc += F[r * l + a] * x[r];
    part[static_cast<long long>(blockIdx.y) * l + a] = acc;
}
__global__ void colsum_combine_kernel(const double* __restrict__ part, int blocks, int l, double* __restrict__ v) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= l) return;
    double acc = 0.0;
    for (int b = 0; b < blocks; ++b) acc += part[static_cast<long long>(b) * l + a];
    v[a] = acc;
}
// out[r][a] = scale * x_r * y_a (rows x l)
__global__ void outer_kernel(const double* __restrict__ x, long long rows, const double* __restrict__ y, int l,
                             double scale, double* __restrict__ out) {
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < rows * l; e += 256LL * gridDim.x)
        out[e] = scale * x[e / l] * y[e % l];
}
}  // namespace

namespace {
__global__ void exp_inplace_kernel(double* __restrict__ x, long long n) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < n) x[i] = exp(x[i]);
}
}  // namespace

int lcn_grad_cost(const lcn_result* res, const lcn_op* op, int which, double* out, size_t* len, int* stale) {
    lcn_ctx* ctx = op ? reinterpret_cast<lcn_ctx*>(op->o.ctx) : nullptr;
    return guard(ctx, [&] {
        if (!res || !op || !len) throw Status(2, "null argument");
        if (op->o.shard) throw Status(2, "grad_cost: not available on a sharded operator");
        const Result& r = res->r;
        const Op& o = op->o;
        if (stale) *stale = r.converged ? 0 : 1;
        if (!r.converged) std::fprintf(stderr, "lcn: warning: gradient requested before convergence (stale)\n");
        if (o.bp) throw Status(2, "grad_cost: gradients are defined for the unextended operators");  // sinkhorn.cpp:269-270
        const double lam = o.lambda;
        auto put = [&](const std::vector<double>& v, double scale) {
            if (out)
                for (size_t i = 0; i < v.size(); ++i) out[i] = scale * v[i];
            *len = v.size();
        };
        if (which == 0) {  // dense / sparse: d d / d C = plan
            if (o.kind >= 2) throw Status(2, "grad_cost: d/dC is defined for the dense and sparse operators");
            if (r.plan_vals.empty()) throw Status(2, "grad_cost: the solve kept no plan (want_plan = false)");
            put(r.plan_vals, 1.0);
            return;
        }
        if (which == 3 || which == 4) {  // lcn: -lambda P^sp, +lambda P^sp_Nys
            if (o.kind != 3) throw Status(2, "grad_cost: log-sparse gradients are defined for the LCN operator");
            if (r.sp_vals.empty()) throw Status(2, "grad_cost: the solve kept no plan (want_plan = false)");
            put(which == 3 ? r.sp_vals : r.sp_nys_vals, which == 3 ? -lam : lam);
            return;
        }
        if (which != 1 && which != 2) throw Status(2, "grad_cost: which out of range");
        if (o.kind < 2) throw Status(2, "grad_cost: operator has no low-rank factors");
        const size_t n = o.n, m = o.m, l = o.l;
        const size_t count = which == 1 ? n * l : l * m;
        *len = count;
        if (!out) return;
        cudaStream_t s = o.ctx->stream;
        // s_i = exp(log s_i), t_j = exp(log t_j) on the device; wt = W t, su = U^T s
        constexpr int kParts = 64;
        DevBuf<double> ds, dt, wt(l), su(l), g(count), part(kParts * l);
        ds.upload(r.log_s.data(), n, s);
        dt.upload(r.log_t.data(), m, s);
        exp_inplace_kernel<<<ceil_div(n, 256), 256, 0, s>>>(ds.get(), static_cast<long long>(n));
        exp_inplace_kernel<<<ceil_div(m, 256), 256, 0, s>>>(dt.get(), static_cast<long long>(m));
        const dim3 gs(static_cast<unsigned>(ceil_div(l, 128)), kParts);
        const unsigned gc = static_cast<unsigned>(ceil_div(l, 128));
        colsum_kernel<<<gs, 128, 0, s>>>(o.Wt64.get(), m, static_cast<int>(l), dt.get(), part.get());
        colsum_combine_kernel<<<gc, 128, 0, s>>>(part.get(), kParts, static_cast<int>(l), wt.get());
        colsum_kernel<<<gs, 128, 0, s>>>(o.U64.get(), n, static_cast<int>(l), ds.get(), part.get());
        colsum_combine_kernel<<<gc, 128, 0, s>>>(part.get(), kParts, static_cast<int>(l), su.get());
        const int grid = static_cast<int>(std::min<long long>(ceil_div(count, 256), 16 * o.ctx->num_sms));
        if (which == 1) {
            // du(i, a) = -lambda s_i wt_a (n x l)
            outer_kernel<<<grid, 256, 0, s>>>(ds.get(), n, wt.get(), static_cast<int>(l), -lam, g.get());
            LAUNCH_OK("grad_cost du");
            g.download(out, count, s);
        } else {
            // dw(a, j) = -lambda su_a t_j (l x m): rows of the transpose, then transposed on the host
            outer_kernel<<<grid, 256, 0, s>>>(dt.get(), m, su.get(), static_cast<int>(l), -lam, g.get());
            LAUNCH_OK("grad_cost dw");
            std::vector<double> tmp(count);
            g.download(tmp.data(), count, s);
            o.ctx->sync();
            for (size_t j = 0; j < m; ++j)
                for (size_t a = 0; a < l; ++a) out[a * m + j] = tmp[j * l + a];
        }
        o.ctx->sync();
    });
}

const char* lcn_result_warning(const lcn_result* res, int i) {
    if (!res || i < 0 || i >= static_cast<int>(res->r.warnings.size())) return nullptr;
    return res->r.warnings[static_cast<size_t>(i)].c_str();
}

}  // extern "C"
