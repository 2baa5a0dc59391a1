// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// Stand-in for /root/reference/proj/src/nystrom.cpp inside the oracle/_ref
// build. The reference file includes <Eigen/Cholesky> (nystrom.cpp:3-4),
// which is absent from this image, so that single translation unit cannot be
// compiled; every other reference source is compiled unmodified. This file
// restates nystrom.cpp:28-196 behaviour-for-behaviour:
//   * select_landmarks            nystrom.cpp:28-48   (Lloyd, 10 iterations, or k-means++ rows)
//   * kernel_block                nystrom.cpp:53-64   (exp(-c * (1/lambda)))
//   * build_factors               nystrom.cpp:68-125  (A in long double, jitter schedule
//                                                      rel in {0,1e-10,...,1e-4} * tr(A)/l,
//                                                      accept iff finite and
//                                                      max|A W - V| <= 1e-6 max|V|)
//   * NystromFactors::entry       nystrom.cpp:127-132
//   * nys_matvec / nys_matvec_t   nystrom.cpp:134-194
// Eigen::LDLT<long double> (diagonal pivoting, zero pivots zeroed in the
// solve) is restated as a hand-written pivoted LDL^T in long double. The
// condition estimate (a diagnostic) is computed exactly as ||A||_1 ||A^-1||_1.
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <vector>

#include "lcn/error.hpp"
#include "lcn/kmeans.hpp"
#include "lcn/nystrom.hpp"

namespace lcn {

const char* landmark_method_name(LandmarkMethod method) {
    switch (method) {
        case LandmarkMethod::KMeans: return "kmeans";
        case LandmarkMethod::KMeansPPSampling: return "kmeans++-sampling";
    }
    return "?";
}

LandmarkMethod landmark_method_from_name(const std::string& name) {
    if (name == "kmeans") return LandmarkMethod::KMeans;
    if (name == "kmeans++-sampling" || name == "kmeanspp") return LandmarkMethod::KMeansPPSampling;
    throw InvalidArgument("unknown landmark method '" + name + "'");
}

LandmarkSet select_landmarks(const PointSet& p, const PointSet& q, std::size_t l,
                             LandmarkMethod method, std::uint64_t seed) {
    PointSet all = union_points(p, q);
    if (l < 1 || l > all.n) throw InvalidArgument("select_landmarks: l out of range");
    LandmarkSet res;
    res.method = method;
    res.seed = seed;
    res.points = PointSet(l, all.dim, "landmarks");
    if (method == LandmarkMethod::KMeans) {
        KmeansResult km = lloyd(all.coords.data(), all.n, all.dim, l, 10, seed);
        res.points.coords = std::move(km.centroids.data);
    } else {
        std::mt19937_64 rng(seed);
        std::vector<std::uint32_t> rows = kmeans_pp_indices(all.coords.data(), all.n, all.dim, l, rng);
        for (std::size_t a = 0; a < l; ++a)
            std::copy(all.point(rows[a]), all.point(rows[a]) + all.dim, res.points.point(a));
    }
    return res;
}

namespace {

using LD = long double;

// k(X, Z) = exp(-c(x, z) * (1/lambda)) in linear space.
DenseMatrix linear_kernel(const PointSet& x, const PointSet& z, CostKind kind, double lambda) {
    DenseMatrix k(x.n, z.n);
    const double inv_lambda = 1.0 / lambda;
#pragma omp parallel for schedule(static) if (x.n > 32)
    for (std::ptrdiff_t r = 0; r < static_cast<std::ptrdiff_t>(x.n); ++r)
        for (std::size_t c = 0; c < z.n; ++c)
            k(static_cast<std::size_t>(r), c) =
                std::exp(-cost_value(kind, x.point(static_cast<std::size_t>(r)), z.point(c), x.dim) *
                         inv_lambda);
    return k;
}

// Symmetric diagonal-pivoted LDL^T of an l x l long-double matrix (column
// major storage is irrelevant: the matrix is symmetric). Returns false when a
// zero pivot leaves a nonzero column below it (Eigen's NumericalIssue).
struct PivotedLdlt {
    std::size_t l = 0;
    std::vector<LD> f;               // packed L (strict lower) + D (diagonal), row-major
    std::vector<std::size_t> perm;   // perm[k] = original index at position k
    bool ok = true;

    explicit PivotedLdlt(const std::vector<LD>& a, std::size_t n) : l(n), f(a), perm(n) {
        for (std::size_t i = 0; i < l; ++i) perm[i] = i;
        std::vector<LD> scratch(l);
        for (std::size_t k = 0; k < l; ++k) {
            std::size_t piv = k;
            LD best = std::fabs(f[k * l + k]);
            for (std::size_t i = k + 1; i < l; ++i)
                if (std::fabs(f[i * l + i]) > best) { best = std::fabs(f[i * l + i]); piv = i; }
            if (piv != k) {
                for (std::size_t c = 0; c < l; ++c) std::swap(f[k * l + c], f[piv * l + c]);
                for (std::size_t r = 0; r < l; ++r) std::swap(f[r * l + k], f[r * l + piv]);
                std::swap(perm[k], perm[piv]);
            }
            // d_k = a_kk - sum_j L_kj^2 d_j; column below uses the same update.
            for (std::size_t j = 0; j < k; ++j) scratch[j] = f[j * l + j] * f[k * l + j];
            LD dk = f[k * l + k];
            for (std::size_t j = 0; j < k; ++j) dk -= f[k * l + j] * scratch[j];
            f[k * l + k] = dk;
            for (std::size_t i = k + 1; i < l; ++i) {
                LD v = f[i * l + k];
                for (std::size_t j = 0; j < k; ++j) v -= f[i * l + j] * scratch[j];
                f[i * l + k] = v;
            }
            if (std::fabs(dk) > 0) {
                for (std::size_t i = k + 1; i < l; ++i) f[i * l + k] /= dk;
            } else {
                for (std::size_t i = k + 1; i < l; ++i)
                    if (f[i * l + k] != 0) ok = false;
            }
        }
    }

    // Solve A x = b in place for one column; pivots at or below LDBL_MIN are
    // treated as zero (their component is dropped), as the restated solver does.
    void solve(LD* b) const {
        std::vector<LD> y(l);
        for (std::size_t k = 0; k < l; ++k) y[k] = b[perm[k]];
        for (std::size_t i = 0; i < l; ++i)
            for (std::size_t j = 0; j < i; ++j) y[i] -= f[i * l + j] * y[j];
        for (std::size_t i = 0; i < l; ++i) {
            LD d = f[i * l + i];
            y[i] = std::fabs(d) > std::numeric_limits<LD>::min() ? y[i] / d : 0;
        }
        for (std::size_t ii = l; ii-- > 0;)
            for (std::size_t j = ii + 1; j < l; ++j) y[ii] -= f[j * l + ii] * y[j];
        for (std::size_t k = 0; k < l; ++k) b[perm[k]] = y[k];
    }
};

}  // namespace

NystromFactors build_factors(const PointSet& p, const PointSet& q, const LandmarkSet& landmarks,
                             CostKind kind, double lambda) {
    if (!(lambda > 0.0)) throw InvalidArgument("build_factors: lambda must be positive");
    const PointSet& lm = landmarks.points;
    if (p.dim != q.dim || p.dim != lm.dim) throw DimensionError("build_factors: dimension mismatch");

    NystromFactors f;
    f.n = p.n;
    f.m = q.n;
    f.l = lm.n;
    f.lambda = lambda;
    f.kind = kind;
    f.u = linear_kernel(p, lm, kind, lambda);
    DenseMatrix v = linear_kernel(lm, q, kind, lambda);

    const std::size_t l = f.l, m = f.m;
    std::vector<LD> a(l * l);
    for (std::size_t r = 0; r < l; ++r)
        for (std::size_t c = 0; c < l; ++c)
            a[r * l + c] = static_cast<LD>(std::exp(-cost_value(kind, lm.point(r), lm.point(c), lm.dim) / lambda));
    LD trace = 0.0L;
    for (std::size_t r = 0; r < l; ++r) trace += a[r * l + r];
    const LD jitter_unit = trace / static_cast<LD>(l);
    LD v_scale = 0.0L;
    for (double x : v.data) v_scale = std::max<LD>(v_scale, std::fabs(static_cast<LD>(x)));
    v_scale = std::max<LD>(v_scale, 1e-300L);

    for (double rel = 0.0; rel <= 1.1e-4; rel = (rel == 0.0 ? 1e-10 : rel * 10.0)) {
        std::vector<LD> aj = a;
        for (std::size_t r = 0; r < l; ++r) aj[r * l + r] += rel * jitter_unit;
        PivotedLdlt fac(aj, l);
        if (!fac.ok) continue;
        // W column by column (columns of V are independent right-hand sides).
        std::vector<LD> w(l * m);
        bool finite = true;
#pragma omp parallel for schedule(static) reduction(&& : finite) if (m > 64)
        for (std::ptrdiff_t jj = 0; jj < static_cast<std::ptrdiff_t>(m); ++jj) {
            const std::size_t j = static_cast<std::size_t>(jj);
            std::vector<LD> col(l);
            for (std::size_t r = 0; r < l; ++r) col[r] = static_cast<LD>(v(r, j));
            fac.solve(col.data());
            for (std::size_t r = 0; r < l; ++r) {
                w[r * m + j] = col[r];
                if (!std::isfinite(col[r])) finite = false;
            }
        }
        if (!finite) continue;
        LD resid = 0.0L;
#pragma omp parallel for schedule(static) reduction(max : resid) if (m > 64)
        for (std::ptrdiff_t jj = 0; jj < static_cast<std::ptrdiff_t>(m); ++jj) {
            const std::size_t j = static_cast<std::size_t>(jj);
            for (std::size_t r = 0; r < l; ++r) {
                LD acc = 0.0L;
                for (std::size_t c = 0; c < l; ++c) acc += aj[r * l + c] * w[c * m + j];
                resid = std::max(resid, std::fabs(acc - static_cast<LD>(v(r, j))));
            }
        }
        if (resid > 1e-6L * v_scale) continue;

        f.w = DenseMatrix(l, m);
        for (std::size_t idx = 0; idx < l * m; ++idx) f.w.data[idx] = static_cast<double>(w[idx]);
        // cond_1(A_j) = ||A_j||_1 ||A_j^-1||_1, exact (diagnostic only).
        LD norm_a = 0.0L, norm_inv = 0.0L;
        for (std::size_t c = 0; c < l; ++c) {
            LD s = 0.0L;
            for (std::size_t r = 0; r < l; ++r) s += std::fabs(aj[r * l + c]);
            norm_a = std::max(norm_a, s);
        }
        std::vector<LD> e(l);
        for (std::size_t c = 0; c < l; ++c) {
            std::fill(e.begin(), e.end(), 0.0L);
            e[c] = 1.0L;
            fac.solve(e.data());
            LD s = 0.0L;
            for (LD x : e) s += std::fabs(x);
            norm_inv = std::max(norm_inv, s);
        }
        LD cond = norm_a * norm_inv;
        f.cond_estimate = std::isfinite(cond) && cond > 0 ? static_cast<double>(cond)
                                                          : std::numeric_limits<double>::infinity();
        return f;
    }
    throw FactorizationError(
        "build_factors: landmark kernel matrix numerically singular beyond jitter budget");
}

double NystromFactors::entry(std::size_t i, std::size_t j) const {
    double s = 0.0;
    for (std::size_t a = 0; a < l; ++a) s += u(i, a) * w(a, j);
    return s;
}

namespace {
bool strictly_positive(std::span<const double> x) {
    for (double v : x)
        if (!(v > 0.0)) return false;
    return true;
}
}  // namespace

std::vector<double> nys_matvec(const NystromFactors& f, std::span<const double> t) {
    if (t.size() != f.m) throw DimensionError("nys_matvec: vector length mismatch");
    const bool check = strictly_positive(t);
    std::vector<double> mid(f.l, 0.0), out(f.n, 0.0);
#pragma omp parallel for schedule(static) if (f.l > 16)
    for (std::ptrdiff_t a = 0; a < static_cast<std::ptrdiff_t>(f.l); ++a) {
        double s = 0.0;
        for (std::size_t j = 0; j < f.m; ++j) s += f.w(static_cast<std::size_t>(a), j) * t[j];
        mid[static_cast<std::size_t>(a)] = s;
    }
#pragma omp parallel for schedule(static) if (f.n > 64)
    for (std::ptrdiff_t i = 0; i < static_cast<std::ptrdiff_t>(f.n); ++i) {
        double s = 0.0;
        for (std::size_t a = 0; a < f.l; ++a) s += f.u(static_cast<std::size_t>(i), a) * mid[a];
        out[static_cast<std::size_t>(i)] = s;
    }
    if (check)
        for (double v : out)
            if (!(v > 0.0)) throw NegativeKernelError("nystrom matvec produced a nonpositive entry");
    return out;
}

std::vector<double> nys_matvec_t(const NystromFactors& f, std::span<const double> s) {
    if (s.size() != f.n) throw DimensionError("nys_matvec_t: vector length mismatch");
    const bool check = strictly_positive(s);
    std::vector<double> mid(f.l, 0.0), out(f.m, 0.0);
#pragma omp parallel for schedule(static) if (f.l > 16)
    for (std::ptrdiff_t a = 0; a < static_cast<std::ptrdiff_t>(f.l); ++a) {
        double acc = 0.0;
        for (std::size_t i = 0; i < f.n; ++i) acc += f.u(i, static_cast<std::size_t>(a)) * s[i];
        mid[static_cast<std::size_t>(a)] = acc;
    }
#pragma omp parallel for schedule(static) if (f.m > 64)
    for (std::ptrdiff_t j = 0; j < static_cast<std::ptrdiff_t>(f.m); ++j) {
        double acc = 0.0;
        for (std::size_t a = 0; a < f.l; ++a) acc += f.w(a, static_cast<std::size_t>(j)) * mid[a];
        out[static_cast<std::size_t>(j)] = acc;
    }
    if (check)
        for (double v : out)
            if (!(v > 0.0))
                throw NegativeKernelError("nystrom transposed matvec produced a nonpositive entry");
    return out;
}

}  // namespace lcn
