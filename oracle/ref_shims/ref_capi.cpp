// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// extern "C" wrappers over the *compiled reference* (/root/reference/proj/src,
// built unmodified by oracle/Makefile into oracle/_ref/libref_lcn.so) so that
// tests/ and bench.py's reference arm can drive it through ctypes. Every
// wrapper forwards to the reference function named in its comment; no
// algorithmic code lives here except mix64/fn_seed, which restate the
// file-local helpers at lsh.cpp:17-27 so bucket ids per band can be exported
// (lsh_neighbor_pairs itself only returns pairs).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "lcn/error.hpp"
#include "lcn/generators.hpp"
#include "lcn/geometry.hpp"
#include "lcn/io.hpp"
#include "lcn/runner.hpp"
#include "lcn/kmeans.hpp"
#include "lcn/lsh.hpp"
#include "lcn/nystrom.hpp"
#include "lcn/operator.hpp"
#include "lcn/reference.hpp"
#include "lcn/sinkhorn.hpp"
#include "lcn/sparse_kernel.hpp"

namespace lcn {
// ref_shims/correction_blocked.cpp: build_correction with the reference's
// per-entry arithmetic, visited bucket block by bucket block
LcnCorrection build_correction_blocked(const SparseKernel& sparse, const NystromFactors& factors,
                                       const std::uint64_t* ids_p, const std::uint64_t* ids_q, int bands,
                                       std::uint64_t range);
}  // namespace lcn

using namespace lcn;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const DimensionError*>(&e)) return 1;
    if (dynamic_cast<const InvalidArgument*>(&e)) return 2;
    if (dynamic_cast<const StabilizationError*>(&e)) return 3;
    if (dynamic_cast<const NegativeKernelError*>(&e)) return 4;
    if (dynamic_cast<const FactorizationError*>(&e)) return 5;
    if (dynamic_cast<const Error*>(&e)) return 6;
    return 9;
}

#define GUARD(...)                           \
    try {                                    \
        __VA_ARGS__;                         \
        return 0;                            \
    } catch (const std::exception& e) {      \
        return fail(e);                      \
    }

PointSet make_points(const double* x, std::size_t n, std::size_t d, const char* id) {
    PointSet ps(n, d, id);
    if (n * d) std::memcpy(ps.coords.data(), x, n * d * sizeof(double));
    return ps;
}

// lsh.cpp:17-27 (file-local in the reference).
std::uint64_t mix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
std::uint64_t fn_seed(std::uint64_t seed, int band, int fn) {
    return mix64(seed ^ mix64(static_cast<std::uint64_t>(band) * 0x100000001b3ull +
                              static_cast<std::uint64_t>(fn)));
}

LshConfig kmeans_cfg(int bands, int buckets, int iters, std::uint64_t seed) {
    LshConfig cfg;
    cfg.scheme = LshScheme::KMeans;
    cfg.bands = bands;
    cfg.rows_per_band = 1;
    cfg.buckets_per_fn = buckets;
    cfg.kmeans_iters = iters;
    cfg.seed = seed;
    return cfg;
}

LshConfig full_cfg(int scheme, int bands, int rows, int buckets, int iters, int branching, std::uint64_t seed) {
    LshConfig cfg;
    cfg.scheme = static_cast<LshScheme>(scheme);
    cfg.bands = bands;
    cfg.rows_per_band = rows;
    cfg.buckets_per_fn = buckets;
    cfg.kmeans_iters = iters;
    cfg.branching = branching;
    cfg.seed = seed;
    return cfg;
}

struct RefOp {
    KernelOperator op;
    std::shared_ptr<SparseKernel> sparse;
    std::shared_ptr<NystromFactors> factors;
    std::shared_ptr<LcnCorrection> corr;
    std::vector<double> landmarks;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// generators.cpp:28-42
int ref_sample_uniform_ball(std::size_t n, std::size_t d, std::uint64_t seed, double* out) {
    GUARD({
        PointSet ps = sample_uniform_ball(n, d, seed, "ball");
        std::memcpy(out, ps.coords.data(), n * d * sizeof(double));
    })
}

// kmeans.cpp:23-65 with a fresh mt19937_64(seed)
int ref_kmeans_pp(const double* pts, std::size_t n, std::size_t d, std::size_t k, std::uint64_t seed,
                  std::uint32_t* out) {
    GUARD({
        std::mt19937_64 rng(seed);
        auto idx = kmeans_pp_indices(pts, n, d, k, rng);
        std::memcpy(out, idx.data(), k * sizeof(std::uint32_t));
    })
}

// kmeans.cpp:67-85
int ref_assign_nearest(const double* pts, std::size_t n, std::size_t d, const double* ctr, std::size_t k,
                       std::uint32_t* out) {
    GUARD({
        DenseMatrix c(k, d);
        std::memcpy(c.data.data(), ctr, k * d * sizeof(double));
        assign_nearest(pts, n, d, c, out);
    })
}

// kmeans.cpp:87-143
int ref_lloyd(const double* pts, std::size_t n, std::size_t d, std::size_t k, int iters, std::uint64_t seed,
              double* centroids, std::uint32_t* assign) {
    GUARD({
        KmeansResult r = lloyd(pts, n, d, k, iters, seed);
        std::memcpy(centroids, r.centroids.data.data(), k * d * sizeof(double));
        std::memcpy(assign, r.assign.data(), n * sizeof(std::uint32_t));
    })
}

// Bucket ids per band of the k-means LSH on X_p ∪ X_q, exactly as
// lsh_neighbor_pairs computes them (lsh.cpp:245-283): band b clusters the
// union with hash_kmeans(seed = fn_seed(cfg.seed, b, 0)). ids: bands x (n+m).
int ref_lsh_kmeans_buckets(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d,
                           int bands, int buckets, int iters, std::uint64_t seed, std::uint64_t* ids) {
    GUARD({
        PointSet all = union_points(make_points(p, n, d, "p"), make_points(q, m, d, "q"));
        for (int b = 0; b < bands; ++b) {
            LshConfig sub = kmeans_cfg(bands, buckets, iters, fn_seed(seed, b, 0));
            auto a = hash_kmeans(all, sub);
            for (std::size_t i = 0; i < n + m; ++i) ids[static_cast<std::size_t>(b) * (n + m) + i] = a[i];
        }
    })
}

// Composite bucket ids per band for any scheme, as lsh_neighbor_pairs
// computes them before neighbor_pairs (lsh.cpp:245-283): cross-polytope =
// hash_cross_polytope of p and of q; k-means schemes = the union loop over
// hash_kmeans with fn_seed(seed, band, fn). ids: bands x (n+m), p first.
int ref_lsh_buckets(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int scheme,
                    int bands, int rows, int buckets, int iters, int branching, std::uint64_t seed, std::uint64_t* ids) {
    GUARD({
        LshConfig cfg = full_cfg(scheme, bands, rows, buckets, iters, branching, seed);
        const std::size_t N = n + m;
        if (cfg.scheme == LshScheme::CrossPolytope) {
            BandBuckets bp = hash_cross_polytope(make_points(p, n, d, "p"), cfg);
            BandBuckets bq = hash_cross_polytope(make_points(q, m, d, "q"), cfg);
            for (int b = 0; b < bands; ++b) {
                std::copy(bp.bucket[b].begin(), bp.bucket[b].end(), ids + static_cast<std::size_t>(b) * N);
                std::copy(bq.bucket[b].begin(), bq.bucket[b].end(), ids + static_cast<std::size_t>(b) * N + n);
            }
        } else {
            PointSet all = union_points(make_points(p, n, d, "p"), make_points(q, m, d, "q"));
            for (int b = 0; b < bands; ++b) {
                std::uint64_t* row = ids + static_cast<std::size_t>(b) * N;
                std::fill(row, row + N, 0);
                for (int fn = 0; fn < rows; ++fn) {
                    LshConfig sub = cfg;
                    sub.seed = fn_seed(seed, b, fn);
                    auto a = hash_kmeans(all, sub);
                    for (std::size_t i = 0; i < N; ++i) row[i] = row[i] * static_cast<std::uint64_t>(buckets) + a[i];
                }
            }
        }
    })
}

// cross_polytope_bucket (lsh.cpp:55-71) per point; proj is d x half row-major.
int ref_cross_polytope_bucket(const double* x, std::size_t n, std::size_t d, const double* proj, std::size_t half,
                              std::uint32_t* out) {
    GUARD({
        DenseMatrix R(d, half);
        std::memcpy(R.data.data(), proj, d * half * sizeof(double));
        for (std::size_t i = 0; i < n; ++i) out[i] = cross_polytope_bucket(x + i * d, d, R);
    })
}

// std::normal_distribution<double>(0, 1) over mt19937_64(seed), as
// hash_cross_polytope draws its projections (lsh.cpp:85-89).
int ref_normal_draws(std::uint64_t seed, std::size_t count, double* out) {
    GUARD({
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (std::size_t i = 0; i < count; ++i) out[i] = gauss(rng);
    })
}

// lsh_neighbor_pairs (lsh.cpp:245-283) for any scheme; returns a NeighborPairs*.
int ref_lsh_pairs_cfg(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int scheme,
                      int bands, int rows, int buckets, int iters, int branching, std::uint64_t seed, void** out) {
    GUARD({
        auto np = std::make_unique<NeighborPairs>(
            lsh_neighbor_pairs(make_points(p, n, d, "p"), make_points(q, m, d, "q"),
                               full_cfg(scheme, bands, rows, buckets, iters, branching, seed)));
        *out = np.release();
    })
}

// lsh.cpp:245-283 end to end; returns a NeighborPairs*.
int ref_lsh_pairs(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int bands,
                  int buckets, int iters, std::uint64_t seed, void** out) {
    GUARD({
        auto np = std::make_unique<NeighborPairs>(lsh_neighbor_pairs(
            make_points(p, n, d, "p"), make_points(q, m, d, "q"), kmeans_cfg(bands, buckets, iters, seed)));
        *out = np.release();
    })
}

// lsh.cpp:212-243 from external bucket ids (ids_p: bands x n, ids_q: bands x m).
int ref_pairs_from_buckets(const std::uint64_t* ids_p, std::size_t n, const std::uint64_t* ids_q, std::size_t m,
                           int bands, std::uint64_t range, void** out) {
    GUARD({
        BandBuckets bp, bq;
        bp.composite_range = bq.composite_range = range;
        for (int b = 0; b < bands; ++b) {
            bp.bucket.emplace_back(ids_p + static_cast<std::size_t>(b) * n, ids_p + (static_cast<std::size_t>(b) + 1) * n);
            bq.bucket.emplace_back(ids_q + static_cast<std::size_t>(b) * m, ids_q + (static_cast<std::size_t>(b) + 1) * m);
        }
        *out = new NeighborPairs(neighbor_pairs(bp, bq, LshConfig{}));
    })
}

// NeighborPairs::from_pairs (lsh.cpp:163-177)
int ref_pairs_from_arrays(std::size_t n, std::size_t m, const std::uint32_t* rows, const std::uint32_t* cols,
                          std::size_t count, void** out) {
    GUARD({
        std::vector<std::pair<std::uint32_t, std::uint32_t>> raw(count);
        for (std::size_t e = 0; e < count; ++e) raw[e] = {rows[e], cols[e]};
        *out = new NeighborPairs(NeighborPairs::from_pairs(n, m, std::move(raw)));
    })
}

std::size_t ref_pairs_nnz(void* h) { return static_cast<NeighborPairs*>(h)->pairs.size(); }
void ref_pairs_copy(void* h, std::uint32_t* rows, std::uint32_t* cols) {
    auto* np = static_cast<NeighborPairs*>(h);
    for (std::size_t e = 0; e < np->pairs.size(); ++e) {
        rows[e] = np->pairs[e].first;
        cols[e] = np->pairs[e].second;
    }
}
void ref_pairs_free(void* h) { delete static_cast<NeighborPairs*>(h); }

// sparse_kernel.cpp:51-80 + operator.cpp:67-78
int ref_op_sparse(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int kind,
                  double lambda, void* pairs, void** out) {
    GUARD({
        auto* r = new RefOp{KernelOperator::sparse(
            build_sparse(make_points(p, n, d, "p"), make_points(q, m, d, "q"),
                         *static_cast<NeighborPairs*>(pairs), static_cast<CostKind>(kind), lambda),
            lambda)};
        *out = r;
    })
}

// nystrom.cpp:28-125 (restated, oracle/ref_shims/nystrom_restated.cpp) +
// sparse_kernel.cpp:82-117 + operator.cpp:90-101. landmarks == nullptr selects
// them with select_landmarks(l, method, lm_seed); otherwise uses the given l x d rows.
int ref_op_lcn(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int kind,
               double lambda, void* pairs, std::size_t l, int method, std::uint64_t lm_seed,
               const double* landmarks, int nystrom_only, void** out, double* phase_ms) {
    GUARD({
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        PointSet P = make_points(p, n, d, "p"), Q = make_points(q, m, d, "q");
        LandmarkSet lm;
        auto t0 = now();
        if (landmarks) {
            lm.points = make_points(landmarks, l, d, "landmarks");
        } else {
            lm = select_landmarks(P, Q, l, static_cast<LandmarkMethod>(method), lm_seed);
        }
        auto t1 = now();
        NystromFactors f = build_factors(P, Q, lm, static_cast<CostKind>(kind), lambda);
        auto t2 = now();
        auto* r = new RefOp{KernelOperator::nystrom(f)};
        r->landmarks = lm.points.coords;
        auto t3 = t2, t4 = t2;
        if (!nystrom_only) {
            SparseKernel sk = build_sparse(P, Q, *static_cast<NeighborPairs*>(pairs), static_cast<CostKind>(kind), lambda);
            t3 = now();
            LcnCorrection c = build_correction(sk, f);
            t4 = now();
            r->op = KernelOperator::lcn(f, c);
        }
        if (phase_ms) {
            phase_ms[0] = ms(t0, t1);  // select_landmarks
            phase_ms[1] = ms(t1, t2);  // build_factors (restated)
            phase_ms[2] = ms(t2, t3);  // build_sparse
            phase_ms[3] = ms(t3, t4);  // build_correction
        }
        *out = r;
    })
}

// geometry.cpp:113-144 + operator.cpp:55-65
int ref_op_dense(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int kind,
                 double lambda, void** out) {
    GUARD({
        *out = new RefOp{KernelOperator::dense(
            build_kernel(build_cost(make_points(p, n, d, "p"), make_points(q, m, d, "q"),
                                    static_cast<CostKind>(kind), lambda)),
            lambda)};
    })
}

void ref_op_free(void* h) { delete static_cast<RefOp*>(h); }

// multihead (sinkhorn.cpp:333-353) over build_cost; per head: lambda,
// distance, iterations, converged, error flag (1 = the head threw)
int ref_multihead(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int kind,
                  double lambda, int heads, const double* pm, const double* qm, double tol, int max_iters,
                  double* lam_out, double* dist_out, int* iters_out, int* conv_out, int* err_out) {
    GUARD({
        DenseCost cost = build_cost(make_points(p, n, d, "p"), make_points(q, m, d, "q"),
                                    static_cast<CostKind>(kind), lambda);
        Marginals marg;
        marg.p.assign(pm, pm + n);
        marg.q.assign(qm, qm + m);
        SinkhornOptions o;
        o.tol = tol;
        o.max_iters = max_iters;
        o.want_plan = false;
        MultiHeadConfig cfg;
        cfg.heads = heads;
        cfg.lambda = lambda;
        std::vector<HeadOutcome> out = multihead(cost, marg, cfg, o);
        for (std::size_t k = 0; k < out.size(); ++k) {
            lam_out[k] = out[k].lambda;
            dist_out[k] = out[k].distance;
            iters_out[k] = out[k].iters;
            conv_out[k] = out[k].converged ? 1 : 0;
            err_out[k] = out[k].error.empty() ? 0 : 1;
        }
    })
}

// Accessors. which: 0 sparse CSR (row_ptr n+1, col nnz, vals = logvals nnz);
// 1 lcn correction (row_ptr, col, vals = delta); 2 U (n x l); 3 W (l x m);
// 4 landmarks (l x d); 5 lcn nys_vals; 6 lcn log_sp.
std::size_t ref_op_nnz(void* h) {
    auto* r = static_cast<RefOp*>(h);
    if (r->op.sparse_kernel()) return r->op.sparse_kernel()->nnz();
    if (r->op.correction()) return r->op.correction()->col.size();
    return 0;
}
std::size_t ref_op_rank(void* h) {
    auto* r = static_cast<RefOp*>(h);
    return r->op.factors() ? r->op.factors()->l : 0;
}
double ref_op_scalar(void* h, int which) {
    auto* r = static_cast<RefOp*>(h);
    if (which == 0) return r->op.correction() ? r->op.correction()->max_abs_delta : 0.0;
    if (which == 1) return r->op.factors() ? r->op.factors()->cond_estimate : 0.0;
    return 0.0;
}
int ref_op_copy(void* h, int which, std::uint32_t* row_ptr, std::uint32_t* col, double* vals) {
    auto* r = static_cast<RefOp*>(h);
    if (which == 0 && r->op.sparse_kernel()) {
        const SparseKernel& s = *r->op.sparse_kernel();
        if (row_ptr) std::memcpy(row_ptr, s.row_ptr.data(), s.row_ptr.size() * 4);
        if (col) std::memcpy(col, s.col.data(), s.col.size() * 4);
        if (vals) std::memcpy(vals, s.logvals.data(), s.logvals.size() * 8);
        return 0;
    }
    if ((which == 0 || which == 1 || which == 5 || which == 6) && r->op.correction()) {
        const LcnCorrection& c = *r->op.correction();  // which 0 on an lcn operator: log K^sp = log_sp
        if (row_ptr) std::memcpy(row_ptr, c.row_ptr.data(), c.row_ptr.size() * 4);
        if (col) std::memcpy(col, c.col.data(), c.col.size() * 4);
        const std::vector<double>& src = which == 1 ? c.delta : which == 5 ? c.nys_vals : c.log_sp;  // 0, 6: log_sp
        if (vals) std::memcpy(vals, src.data(), src.size() * 8);
        return 0;
    }
    if (which == 2 && r->op.factors()) {
        std::memcpy(vals, r->op.factors()->u.data.data(), r->op.factors()->u.data.size() * 8);
        return 0;
    }
    if (which == 3 && r->op.factors()) {
        std::memcpy(vals, r->op.factors()->w.data.data(), r->op.factors()->w.data.size() * 8);
        return 0;
    }
    if (which == 4) {
        std::memcpy(vals, r->landmarks.data(), r->landmarks.size() * 8);
        return 0;
    }
    if (which == 7 && r->op.dense_kernel()) {  // DenseKernel::logk, n x m row-major
        std::memcpy(vals, r->op.dense_kernel()->logk.data.data(), r->op.dense_kernel()->logk.data.size() * 8);
        return 0;
    }
    g_err = "ref_op_copy: nothing to copy";
    return 2;
}

// operator.cpp:226-252
int ref_op_log_matvec(void* h, const double* in, std::size_t len, int transposed, double* out) {
    GUARD({
        auto* r = static_cast<RefOp*>(h);
        std::span<const double> v(in, len);
        std::vector<double> y = transposed ? r->op.log_matvec_t(v) : r->op.log_matvec(v);
        std::memcpy(out, y.data(), y.size() * 8);
    })
}

// sinkhorn.cpp:104-188; returns a SinkhornResult*.
int ref_sinkhorn(void* h, const double* pm, std::size_t n, const double* qm, std::size_t m, double tol,
                 int max_iters, int check_support, int want_plan, void** out) {
    GUARD({
        auto* r = static_cast<RefOp*>(h);
        Marginals marg;
        marg.p.assign(pm, pm + n);
        marg.q.assign(qm, qm + m);
        SinkhornOptions o;
        o.tol = tol;
        o.max_iters = max_iters;
        o.check_support = check_support != 0;
        o.want_plan = want_plan != 0;
        *out = new SinkhornResult(sinkhorn(r->op, marg, o));
    })
}

// One small LCN problem end to end (the configs[4] unit):
// lsh_neighbor_pairs (k-means, 1 band) -> build_sparse -> select_landmarks
// (KMeans) -> build_factors -> build_correction -> KernelOperator::lcn ->
// sinkhorn(tol 0, iters). Returns the distance; errors as status codes.
int ref_lcn_problem(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int kind,
                    double lambda, int buckets, int kmeans_iters, std::uint64_t lsh_seed, std::size_t l,
                    std::uint64_t lm_seed, int iters, double* distance) {
    GUARD({
        PointSet P = make_points(p, n, d, "p"), Q = make_points(q, m, d, "q");
        NeighborPairs pairs = lsh_neighbor_pairs(P, Q, kmeans_cfg(1, buckets, kmeans_iters, lsh_seed));
        SparseKernel sk = build_sparse(P, Q, pairs, static_cast<CostKind>(kind), lambda);
        LandmarkSet lm = select_landmarks(P, Q, l, LandmarkMethod::KMeans, lm_seed);
        NystromFactors f = build_factors(P, Q, lm, static_cast<CostKind>(kind), lambda);
        LcnCorrection c = build_correction(sk, f);
        KernelOperator op = KernelOperator::lcn(f, c);
        Marginals marg;
        marg.p.assign(n, 1.0 / static_cast<double>(n));
        marg.q.assign(m, 1.0 / static_cast<double>(m));
        SinkhornOptions o;
        o.tol = 0.0;
        o.max_iters = iters;
        o.check_support = false;
        o.want_plan = false;
        *distance = sinkhorn(op, marg, o).distance;
    })
}

void ref_result_free(void* h) { delete static_cast<SinkhornResult*>(h); }

// 0 distance, 1 iters, 2 converged, 3 marginal_err_final, 4 #warnings, 5 #err trace
double ref_result_scalar(void* h, int which) {
    auto* s = static_cast<SinkhornResult*>(h);
    switch (which) {
        case 0: return s->distance;
        case 1: return s->iters;
        case 2: return s->converged ? 1.0 : 0.0;
        case 3: return s->marginal_err_final;
        case 4: return static_cast<double>(s->warnings.size());
        case 5: return static_cast<double>(s->state.marginal_err.size());
        case 6: return s->plan.eps_mass;
    }
    return 0.0;
}

// 0 log_s, 1 log_t, 2 row_marginal, 3 marginal_err trace, 4 sparse plan vals,
// 5 lcn sp_vals, 6 lcn sp_nys_vals, 7 P_U (n x l), 8 P_W (l x m), 9 dense plan (n x m)
std::size_t ref_result_copy(void* h, int which, double* out) {
    auto* s = static_cast<SinkhornResult*>(h);
    const std::vector<double>* v = nullptr;
    switch (which) {
        case 0: v = &s->state.log_s; break;
        case 1: v = &s->state.log_t; break;
        case 2: v = &s->row_marginal; break;
        case 3: v = &s->state.marginal_err; break;
        case 4: v = &s->plan.sparse_vals; break;
        case 5: v = &s->plan.sp_vals; break;
        case 6: v = &s->plan.sp_nys_vals; break;
        case 7: if (s->plan.p_u) v = &s->plan.p_u->data; break;
        case 8: if (s->plan.p_w) v = &s->plan.p_w->data; break;
        case 9: if (s->plan.dense) v = &s->plan.dense->data; break;
        case 10: v = &s->plan.del_p_mass; break;
        case 11: v = &s->plan.del_q_mass; break;
    }
    if (!v) return 0;
    if (out) std::memcpy(out, v->data(), v->size() * 8);
    return v->size();
}

// grad_cost (sinkhorn.cpp:263-320). which: 0 dense cost grad (n x m) or
// sparse cost grad, 1 du (n x l), 2 dw (l x m), 3 log_sparse, 4 log_sparse_nys.
// Returns the length (0 when absent); *stale as Gradients::stale.
std::size_t ref_grad_cost(void* op, void* res, int which, double* out, int* stale) {
    try {
        auto* r = static_cast<RefOp*>(op);
        auto* s = static_cast<SinkhornResult*>(res);
        Gradients g = grad_cost(*s, r->op);
        if (stale) *stale = g.stale ? 1 : 0;
        const std::vector<double>* v = nullptr;
        switch (which) {
            case 0: v = g.cost ? &g.cost->data : &g.cost_sparse; break;
            case 1: if (g.u) v = &g.u->data; break;
            case 2: if (g.w) v = &g.w->data; break;
            case 3: v = &g.log_sparse; break;
            case 4: v = &g.log_sparse_nys; break;
        }
        if (!v) return 0;
        if (out) std::memcpy(out, v->data(), v->size() * 8);
        return v->size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
}

// sinkhorn.cpp:222-261
int ref_distance_lcn(void* res, void* op, double* out) {
    GUARD({
        auto* s = static_cast<SinkhornResult*>(res);
        auto* r = static_cast<RefOp*>(op);
        *out = distance_lcn(s->state, *r->op.factors(), *r->op.correction());
    })
}

// reference.cpp:41-105 (independent serial linear-space solver)
int ref_dense_reference(const double* cost, std::size_t n, std::size_t m, const double* p, const double* q,
                        double lambda, double tol, int max_iters, double* plan, double* distance, int* iters) {
    GUARD({
        ref::Solution sol = ref::solve(std::vector<double>(cost, cost + n * m), n, m,
                                       std::vector<double>(p, p + n), std::vector<double>(q, q + m), lambda,
                                       tol, max_iters);
        if (plan) std::memcpy(plan, sol.plan.data(), n * m * 8);
        *distance = sol.distance;
        *iters = sol.iters;
    })
}

// sample_clustered (generators.cpp:42-106)
int ref_sample_clustered(std::size_t n, std::size_t d, std::size_t c, double D, double r, std::uint64_t seed,
                         double* p_out, double* q_out, double* centers_out) {
    GUARD({
        ClusteredProblem cp = sample_clustered(n, d, c, D, r, seed);
        std::memcpy(p_out, cp.p.coords.data(), n * d * sizeof(double));
        std::memcpy(q_out, cp.q.coords.data(), n * d * sizeof(double));
        if (centers_out) std::memcpy(centers_out, cp.centers.data.data(), c * d * sizeof(double));
    })
}

// read_points_file (io.cpp:105-116); out == nullptr: shape only
int ref_points_read(const char* path, double* out, std::size_t* n, std::size_t* d) {
    GUARD({
        PointSet ps = read_points_file(path);
        if (out) std::memcpy(out, ps.coords.data(), ps.coords.size() * sizeof(double));
        *n = ps.n;
        *d = ps.dim;
    })
}

// write_points_file (io.cpp:118-126)
int ref_points_write(const char* path, const double* pts, std::size_t n, std::size_t d, int binary) {
    GUARD(write_points_file(path, make_points(pts, n, d, "p"), binary != 0))
}

// run_all (runner.cpp:344-418) on a JSON config (config_from_json,
// runner.cpp:92-141); *out = {"records": [record_to_json ...]} (free with
// ref_free_string). Timing fields are dropped by strict-deterministic configs.
int ref_run_all_json(const char* config_json, char** out) {
    GUARD({
        RunConfig cfg = config_from_json(nlohmann::json::parse(config_json));
        nlohmann::json j;
        j["records"] = nlohmann::json::array();
        for (const RunRecord& r : run_all(cfg)) j["records"].push_back(record_to_json(r));
        const std::string s = j.dump();
        *out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*out, s.c_str(), s.size() + 1);
    })
}

void ref_free_string(char* p) { std::free(p); }

// ---- full-size parity (configs[3] at n = m = 1e6, tests/ and oracle/parity_c3.py) ----

// One band of the k-means LSH on the union (lsh.cpp:267-281): hash_kmeans
// with fn_seed(seed, band, 0). Separate entry so the bands can run on
// separate host threads (the reference loops them; ids do not depend on it).
int ref_hash_kmeans_band(const double* all, std::size_t N, std::size_t d, int buckets, int iters, std::uint64_t seed,
                         int band, std::uint64_t* ids) {
    GUARD({
        PointSet ps = make_points(all, N, d, "union");
        LshConfig sub = kmeans_cfg(1, buckets, iters, fn_seed(seed, band, 0));
        auto a = hash_kmeans(ps, sub);
        for (std::size_t i = 0; i < N; ++i) ids[i] = a[i];
    })
}

// select_landmarks (nystrom.cpp:28-48); out: l x d.
int ref_select_landmarks(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d,
                         std::size_t l, int method, std::uint64_t seed, double* out) {
    GUARD({
        LandmarkSet lm = select_landmarks(make_points(p, n, d, "p"), make_points(q, m, d, "q"), l,
                                          static_cast<LandmarkMethod>(method), seed);
        std::memcpy(out, lm.points.coords.data(), l * d * sizeof(double));
    })
}

// The reference's staged LCN build from external bucket ids and explicit
// landmarks, as run_one does it (runner.cpp:258-271) but with
// neighbor_pairs(BandBuckets...) (lsh.cpp:212-243) in place of the LSH:
// neighbor_pairs -> build_sparse -> build_factors -> build_correction ->
// KernelOperator::lcn. Intermediates are released as soon as the next stage
// has consumed them (the configs[3] operator is ~27 GB of host memory).
// phase_ms: pairs, build_sparse, build_factors, build_correction.
int ref_lcn_pipeline(const double* p, std::size_t n, const double* q, std::size_t m, std::size_t d, int kind,
                     double lambda, const std::uint64_t* ids_p, const std::uint64_t* ids_q, int bands,
                     std::uint64_t range, const double* landmarks, std::size_t l, double* phase_ms, void** out) {
    GUARD({
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        PointSet P = make_points(p, n, d, "p"), Q = make_points(q, m, d, "q");
        auto t0 = now();
        auto np = std::make_unique<NeighborPairs>();
        {
            BandBuckets bp, bq;
            bp.composite_range = bq.composite_range = range;
            for (int b = 0; b < bands; ++b) {
                bp.bucket.emplace_back(ids_p + static_cast<std::size_t>(b) * n,
                                       ids_p + (static_cast<std::size_t>(b) + 1) * n);
                bq.bucket.emplace_back(ids_q + static_cast<std::size_t>(b) * m,
                                       ids_q + (static_cast<std::size_t>(b) + 1) * m);
            }
            *np = neighbor_pairs(bp, bq, LshConfig{});
        }
        auto t1 = now();
        auto sk = std::make_unique<SparseKernel>(build_sparse(P, Q, *np, static_cast<CostKind>(kind), lambda));
        np.reset();
        auto t2 = now();
        LandmarkSet lm;
        lm.points = make_points(landmarks, l, d, "landmarks");
        NystromFactors f = build_factors(P, Q, lm, static_cast<CostKind>(kind), lambda);
        auto t3 = now();
        // LCN_REF_BLOCKED_CORRECTION=1: same values, bucket-blocked traversal
        // (the row walk of sparse_kernel.cpp:96-109 is days at configs[3])
        const char* blk = std::getenv("LCN_REF_BLOCKED_CORRECTION");
        LcnCorrection c = (blk && *blk == '1') ? build_correction_blocked(*sk, f, ids_p, ids_q, bands, range)
                                               : build_correction(*sk, f);
        sk.reset();
        auto t4 = now();
        auto* r = new RefOp{KernelOperator::lcn(std::move(f), std::move(c))};
        r->landmarks = lm.points.coords;
        if (phase_ms) {
            phase_ms[0] = ms(t0, t1);
            phase_ms[1] = ms(t1, t2);
            phase_ms[2] = ms(t2, t3);
            phase_ms[3] = ms(t3, t4);
        }
        *out = r;
    })
}

// Per-row digest of the operator's support (CSR of the LCN correction or the
// sparse kernel): count and two 64-bit folds of mix64(col) (wrapping sum and
// xor). Columns are sorted within a row (sparse_kernel.hpp:19-21), so equal
// digests mean equal rows with overwhelming probability.
int ref_op_row_digest(void* h, std::uint32_t* cnt, std::uint64_t* hsum, std::uint64_t* hxor) {
    try {
        auto* r = static_cast<RefOp*>(h);
        const std::vector<std::uint32_t>* rp = nullptr;
        const std::vector<std::uint32_t>* col = nullptr;
        if (r->op.correction()) {
            rp = &r->op.correction()->row_ptr;
            col = &r->op.correction()->col;
        } else if (r->op.sparse_kernel()) {
            rp = &r->op.sparse_kernel()->row_ptr;
            col = &r->op.sparse_kernel()->col;
        } else {
            throw InvalidArgument("ref_op_row_digest: operator has no support");
        }
        const std::size_t rows = rp->size() - 1;
#pragma omp parallel for schedule(static)
        for (std::ptrdiff_t ii = 0; ii < static_cast<std::ptrdiff_t>(rows); ++ii) {
            const std::size_t i = static_cast<std::size_t>(ii);
            std::uint64_t s = 0, x = 0;
            for (std::uint32_t e = (*rp)[i]; e < (*rp)[i + 1]; ++e) {
                std::uint64_t hcol = mix64((*col)[e]);
                s += hcol;
                x ^= hcol;
            }
            cnt[i] = (*rp)[i + 1] - (*rp)[i];
            hsum[i] = s;
            hxor[i] = x;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// extract_plan (sinkhorn.cpp:365-369) of a solved LCN operator, copied out
// only for the listed rows (ascending): per entry the column, log K^sp,
// delta, sp_vals and sp_nys_vals (Plan, sinkhorn.hpp:34-52). cnt[k] = row
// length; the flat outputs hold sum(cnt) entries (size them with
// ref_op_row_digest's counts).
int ref_plan_rows(void* op, void* res, const std::uint32_t* rows, std::size_t nrows, std::uint32_t* cnt,
                  std::uint32_t* cols, double* log_sp, double* delta, double* sp_vals, double* sp_nys_vals) {
    GUARD({
        auto* r = static_cast<RefOp*>(op);
        auto* s = static_cast<SinkhornResult*>(res);
        const LcnCorrection& c = *r->op.correction();
        Plan plan = extract_plan(r->op, s->state);
        std::size_t o = 0;
        for (std::size_t k = 0; k < nrows; ++k) {
            const std::uint32_t i = rows[k];
            cnt[k] = c.row_ptr[i + 1] - c.row_ptr[i];
            for (std::uint32_t e = c.row_ptr[i]; e < c.row_ptr[i + 1]; ++e, ++o) {
                cols[o] = c.col[e];
                log_sp[o] = c.log_sp[e];
                delta[o] = c.delta[e];
                sp_vals[o] = plan.sp_vals[e];
                sp_nys_vals[o] = plan.sp_nys_vals[e];
            }
        }
    })
}

// KernelOperator::with_bp (operator.cpp:103-115) with
// BpExtension::from_costs (operator.cpp:33-43), replacing the handle's operator
int ref_op_with_bp(void* h, const double* cost_p, std::size_t n, const double* cost_q, std::size_t m, double lambda) {
    GUARD({
        auto* r = static_cast<RefOp*>(h);
        r->op = r->op.with_bp(BpExtension::from_costs(std::span<const double>(cost_p, n),
                                                      std::span<const double>(cost_q, m), lambda));
    })
}

}  // extern "C"
