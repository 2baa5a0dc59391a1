// Drop-in shim: the reference's lcn:: hot-path functions implemented over the
// B200 C-ABI (include/lcn_b200.h). Compiled against the reference's own
// headers; linked in place of the reference's definitions of the same
// functions (integration/Makefile weakens those definitions), every
// caller of the reference's API -- runner.cpp's run_one, the reference's unit
// tests -- runs its staged build and its Sinkhorn solves on the GPU with no
// source change:
//
//   lsh_neighbor_pairs  lsh.hpp:67-68         -> lcn_lsh_neighbor_pairs
//   build_sparse        sparse_kernel.hpp:32  -> lcn_build_sparse
//   build_correction    sparse_kernel.hpp:54  -> lcn_build_correction
//   select_landmarks    nystrom.hpp:26        -> lcn_select_landmarks
//   build_factors       nystrom.hpp:46        -> lcn_build_factors
//   sinkhorn            sinkhorn.hpp:68-69    -> lcn_op_from_{dense,sparse,nystrom,lcn}
//                                                (+ lcn_op_set_bp) and lcn_sinkhorn
//
// The reference keeps its host-side types and the rest of its API (operator
// matvecs, plan extraction from the returned scalings, distances, gradients,
// metrics). C-ABI statuses are rethrown as the lcn::Error subtype they map to,
// with the library's message (the reference's text).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "lcn/error.hpp"
#include "lcn/lsh.hpp"
#include "lcn/nystrom.hpp"
#include "lcn/operator.hpp"
#include "lcn/sinkhorn.hpp"
#include "lcn/sparse_kernel.hpp"
#include "lcn_b200.h"

namespace lcn {

namespace {

// One process-wide context, fp64 storage: the reference's API promises fp64
// results (its unit tests hold 1e-12 tolerances).
lcn_ctx* ctx() {
    static std::once_flag once;
    static lcn_ctx* c = nullptr;
    static int rc = 0;
    std::call_once(once, [] {
        int dev = 0;
        if (const char* e = std::getenv("LCN_SHIM_DEVICE")) dev = std::atoi(e);
        rc = lcn_ctx_create(dev, LCN_STORE_FP64, &c);
        if (rc == LCN_OK) std::fprintf(stderr, "lcn shim: B200 context on device %d (liblcn_b200 ABI %d)\n", dev,
                                       lcn_abi_version());
    });
    if (rc != LCN_OK) throw Error(std::string("lcn shim: no B200 context: ") + lcn_ctx_last_error(nullptr));
    return c;
}

[[noreturn]] void rethrow(int rc) {
    const std::string msg = lcn_ctx_last_error(ctx());
    switch (rc) {
        case LCN_E_DIMENSION: throw DimensionError(msg);
        case LCN_E_INVALID_ARGUMENT: throw InvalidArgument(msg);
        case LCN_E_STABILIZATION: throw StabilizationError(msg);
        case LCN_E_NEGATIVE_KERNEL: throw NegativeKernelError(msg);
        case LCN_E_FACTORIZATION: throw FactorizationError(msg);
        default: throw Error(msg);
    }
}

void ok(int rc) {
    if (rc != LCN_OK) rethrow(rc);
}

int cost_code(CostKind k) { return static_cast<int>(k); }

void check_same_dim(const PointSet& p, const PointSet& q) {
    if (p.dim != q.dim) throw DimensionError("point sets have different dimensions");
}

struct OpDeleter {
    void operator()(lcn_op* o) const { lcn_op_destroy(o); }
};
struct ResDeleter {
    void operator()(lcn_result* r) const { lcn_result_destroy(r); }
};

// The device operator of a KernelOperator, from its host structs.
std::unique_ptr<lcn_op, OpDeleter> device_op(const KernelOperator& op) {
    lcn_op* h = nullptr;
    const std::size_t n = op.base_rows(), m = op.base_cols();
    switch (op.kind()) {
        case KernelOperator::Kind::Dense:
            ok(lcn_op_from_dense(ctx(), n, m, op.dense_kernel()->logk.data.data(), op.lambda(), &h));
            break;
        case KernelOperator::Kind::Sparse: {
            const SparseKernel& s = *op.sparse_kernel();
            ok(lcn_op_from_sparse(ctx(), n, m, s.row_ptr.data(), s.col.data(), s.nnz(), s.logvals.data(), op.lambda(),
                                  &h));
            break;
        }
        case KernelOperator::Kind::Nystrom: {
            const NystromFactors& f = *op.factors();
            ok(lcn_op_from_nystrom(ctx(), n, m, f.l, f.u.data.data(), f.w.data.data(), op.lambda(), &h));
            break;
        }
        case KernelOperator::Kind::Lcn: {
            const NystromFactors& f = *op.factors();
            const LcnCorrection& c = *op.correction();
            std::vector<std::uint32_t> rp = c.row_ptr;
            if (rp.size() != n + 1) rp.assign(n + 1, 0);  // an empty correction may leave row_ptr short
            ok(lcn_op_from_lcn(ctx(), n, m, f.l, f.u.data.data(), f.w.data.data(), op.lambda(), rp.data(),
                               c.col.data(), c.col.size(), c.delta.data(), c.log_sp.data(), c.max_abs_delta, &h));
            break;
        }
    }
    std::unique_ptr<lcn_op, OpDeleter> d(h);
    if (op.has_bp()) ok(lcn_op_set_bp(d.get(), op.bp()->del_p.data(), op.bp()->del_q.data()));
    return d;
}

std::vector<double> copy_vec(const lcn_result* r, int which) {
    std::size_t len = 0;
    ok(lcn_result_copy(r, which, nullptr, &len));
    std::vector<double> v(len);
    if (len) ok(lcn_result_copy(r, which, v.data(), &len));
    return v;
}

}  // namespace

NeighborPairs lsh_neighbor_pairs(const PointSet& p, const PointSet& q, const LshConfig& cfg) {
    p.validate();
    q.validate();
    check_same_dim(p, q);
    lcn_lsh_config c{};
    c.bands = cfg.bands;
    c.rows_per_band = cfg.rows_per_band;
    c.buckets_per_fn = cfg.buckets_per_fn;
    c.kmeans_iters = cfg.kmeans_iters;
    c.seed = cfg.seed;
    c.scheme = static_cast<int>(cfg.scheme);
    c.branching = cfg.branching;
    lcn_pairs* h = nullptr;
    ok(lcn_lsh_neighbor_pairs(ctx(), p.coords.data(), p.n, q.coords.data(), q.n, p.dim, &c, &h));
    std::size_t nnz = 0;
    lcn_pairs_info(h, nullptr, nullptr, &nnz);
    std::vector<std::uint32_t> rp(p.n + 1), col(nnz);
    lcn_pairs_copy(h, rp.data(), col.data());
    lcn_pairs_destroy(h);
    NeighborPairs out;
    out.n = p.n;
    out.m = q.n;
    out.pairs.reserve(nnz);
    out.row_counts.assign(p.n, 0);
    for (std::size_t i = 0; i < p.n; ++i) {
        out.row_counts[i] = rp[i + 1] - rp[i];
        for (std::uint32_t e = rp[i]; e < rp[i + 1]; ++e) out.pairs.emplace_back(static_cast<std::uint32_t>(i), col[e]);
    }
    return out;
}

SparseKernel build_sparse(const PointSet& p, const PointSet& q, const NeighborPairs& pairs, CostKind kind,
                          double lambda) {
    if (!(lambda > 0.0)) throw InvalidArgument("build_sparse: lambda must be positive");
    if (pairs.n != p.n || pairs.m != q.n) throw DimensionError("build_sparse: pattern shape mismatch");
    check_same_dim(p, q);
    SparseKernel s;
    s.n = p.n;
    s.m = q.n;
    s.row_ptr.assign(s.n + 1, 0);
    for (const auto& pr : pairs.pairs) ++s.row_ptr[pr.first + 1];
    for (std::size_t i = 0; i < s.n; ++i) s.row_ptr[i + 1] += s.row_ptr[i];
    s.col.resize(pairs.pairs.size());
    for (std::size_t e = 0; e < pairs.pairs.size(); ++e) s.col[e] = pairs.pairs[e].second;
    s.logvals.assign(s.col.size(), 0.0);
    ok(lcn_build_sparse(ctx(), p.coords.data(), p.n, q.coords.data(), q.n, p.dim, s.row_ptr.data(), s.col.data(),
                        s.col.size(), cost_code(kind), lambda, s.logvals.data()));
    s.build_csc();
    return s;
}

LcnCorrection build_correction(const SparseKernel& sparse, const NystromFactors& factors) {
    if (sparse.n != factors.n || sparse.m != factors.m) throw DimensionError("build_correction: shape mismatch");
    LcnCorrection c;
    c.n = sparse.n;
    c.m = sparse.m;
    c.row_ptr = sparse.row_ptr;
    if (c.row_ptr.size() != c.n + 1) c.row_ptr.assign(c.n + 1, 0);
    c.col = sparse.col;
    c.log_sp = sparse.logvals;
    c.delta.assign(sparse.nnz(), 0.0);
    c.nys_vals.assign(sparse.nnz(), 0.0);
    ok(lcn_build_correction(ctx(), c.n, c.m, factors.l, c.row_ptr.data(), c.col.data(), c.col.size(),
                            c.log_sp.data(), factors.u.data.data(), factors.w.data.data(), c.delta.data(),
                            c.nys_vals.data(), &c.max_abs_delta));
    c.build_csc();
    return c;
}

LandmarkSet select_landmarks(const PointSet& p, const PointSet& q, std::size_t l, LandmarkMethod method,
                             std::uint64_t seed) {
    check_same_dim(p, q);
    if (l < 1 || l > p.n + q.n) throw InvalidArgument("select_landmarks: l out of range");
    LandmarkSet out;
    out.method = method;
    out.seed = seed;
    out.points = PointSet(l, p.dim, "landmarks");
    ok(lcn_select_landmarks(ctx(), p.coords.data(), p.n, q.coords.data(), q.n, p.dim, l, static_cast<int>(method),
                            seed, out.points.coords.data()));
    return out;
}

NystromFactors build_factors(const PointSet& p, const PointSet& q, const LandmarkSet& landmarks, CostKind kind,
                             double lambda) {
    if (!(lambda > 0.0)) throw InvalidArgument("build_factors: lambda must be positive");
    check_same_dim(p, q);
    if (landmarks.points.dim != p.dim) throw DimensionError("build_factors: landmark dimension mismatch");
    NystromFactors f;
    f.n = p.n;
    f.m = q.n;
    f.l = landmarks.points.n;
    f.lambda = lambda;
    f.kind = kind;
    f.u = DenseMatrix(f.n, f.l);
    f.w = DenseMatrix(f.l, f.m);
    ok(lcn_build_factors(ctx(), p.coords.data(), p.n, q.coords.data(), q.n, p.dim, landmarks.points.coords.data(),
                         f.l, cost_code(kind), lambda, f.u.data.data(), f.w.data.data(), &f.cond_estimate));
    return f;
}

SinkhornResult sinkhorn(const KernelOperator& op, const Marginals& marg, const SinkhornOptions& opts) {
    marg.validate(/*balanced=*/!op.has_bp());
    if (marg.p.size() != op.base_rows() || marg.q.size() != op.base_cols())
        throw DimensionError("sinkhorn: marginal length does not match operator shape");
    if (opts.max_iters < 1) throw InvalidArgument("sinkhorn: max_iters must be >= 1");
    auto d = device_op(op);
    lcn_sinkhorn_options o{opts.tol, opts.max_iters, opts.check_support ? 1 : 0, 0};
    lcn_result* rh = nullptr;
    ok(lcn_sinkhorn(d.get(), marg.p.data(), marg.q.data(), &o, &rh));
    std::unique_ptr<lcn_result, ResDeleter> r(rh);
    lcn_result_info_t info{};
    ok(lcn_result_get_info(r.get(), &info));
    SinkhornResult res;
    res.distance = info.distance;
    res.iters = info.iters;
    res.converged = info.converged != 0;
    res.marginal_err_final = info.marginal_err_final;
    res.row_marginal = copy_vec(r.get(), 2);
    res.state.log_s = copy_vec(r.get(), 0);
    res.state.log_t = copy_vec(r.get(), 1);
    res.state.marginal_err = copy_vec(r.get(), 3);
    res.state.iters = info.iters;
    for (int i = 0; i < info.n_warnings; ++i) res.warnings.emplace_back(lcn_result_warning(r.get(), i));
    // the decomposed plan of the GPU's scalings, by the reference's own
    // extract_plan (sinkhorn.hpp:118-120)
    if (opts.want_plan) res.plan = extract_plan(op, res.state);
    return res;
}

}  // namespace lcn
