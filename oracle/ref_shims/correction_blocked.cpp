// ORACLE TEST INFRASTRUCTURE (not product code).
//
// build_correction (sparse_kernel.cpp:82-117) restated for full-size parity
// runs. Per stored pair the arithmetic is exactly the reference's:
//   exact = std::exp(log_sp[e])                       (sparse_kernel.cpp:101)
//   nys   = sum_a u(i, a) * w(a, j), left to right,    (nystrom.cpp:127-132)
//           each product rounded, then each sum rounded (-ffp-contract=off,
//           no FMA: this file is built with -mavx2 but never -mfma)
//   delta = exact - nys, max_abs = max |delta|          (sparse_kernel.cpp:105-108)
// so every value is bit-identical to the reference's (pinned by
// tests/test_oracle_cpu.py::test_blocked_correction_bit_exact). Only the
// traversal differs: the reference walks rows, and entry(i, j) reads column j
// of the row-major l x m W with stride m, 512 cache misses per entry, which at
// configs[3] (5.2e8 entries) is days of CPU time. Here the entries are
// visited bucket block by bucket block (the support of neighbor_pairs is the
// union of the bands' bucket blocks, lsh.cpp:212-243), each block's W columns
// packed once, and 4 x 8 entries computed together in SIMD lanes (each lane
// its own sequential chain).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "lcn/error.hpp"
#include "lcn/nystrom.hpp"
#include "lcn/sparse_kernel.hpp"

namespace lcn {

typedef double v4d __attribute__((vector_size(32)));

namespace {

struct Groups {
    std::vector<std::uint32_t> start;  // per bucket, into idx
    std::vector<std::uint32_t> idx;    // point indices, ascending within a bucket
};

Groups group_by(const std::uint64_t* ids, std::size_t n, std::uint64_t range) {
    Groups g;
    g.start.assign(range + 1, 0);
    for (std::size_t i = 0; i < n; ++i) {
        if (ids[i] >= range) throw InvalidArgument("build_correction_blocked: bucket id out of range");
        ++g.start[ids[i] + 1];
    }
    for (std::uint64_t b = 0; b < range; ++b) g.start[b + 1] += g.start[b];
    g.idx.resize(n);
    std::vector<std::uint32_t> cur(g.start.begin(), g.start.end() - 1);
    for (std::size_t i = 0; i < n; ++i) g.idx[cur[ids[i]]++] = static_cast<std::uint32_t>(i);
    return g;
}

}  // namespace

LcnCorrection build_correction_blocked(const SparseKernel& sparse, const NystromFactors& factors,
                                       const std::uint64_t* ids_p, const std::uint64_t* ids_q, int bands,
                                       std::uint64_t range) {
    if (sparse.n != factors.n || sparse.m != factors.m) throw DimensionError("build_correction: shape mismatch");
    LcnCorrection c;
    c.n = sparse.n;
    c.m = sparse.m;
    c.row_ptr = sparse.row_ptr;
    c.col = sparse.col;
    c.log_sp = sparse.logvals;
    c.delta.assign(sparse.nnz(), 0.0);
    c.nys_vals.assign(sparse.nnz(), 0.0);
    const std::size_t n = c.n, m = c.m, l = factors.l;
    const double* U = factors.u.data.data();  // n x l row-major
    const double* W = factors.w.data.data();  // l x m row-major

    double max_abs = 0.0;
    bool overflow = false;
    unsigned long long visited = 0;
    for (int band = 0; band < bands; ++band) {
        const Groups gp = group_by(ids_p + static_cast<std::size_t>(band) * n, n, range);
        const Groups gq = group_by(ids_q + static_cast<std::size_t>(band) * m, m, range);
#pragma omp parallel reduction(max : max_abs) reduction(|| : overflow) reduction(+ : visited)
        {
            std::vector<double> wp;   // l x mbp: the block's W columns, padded to 8
            std::vector<std::uint32_t> pos;
            std::vector<double> acc;
#pragma omp for schedule(dynamic, 1)
            for (std::int64_t bb = 0; bb < static_cast<std::int64_t>(range); ++bb) {
                const std::uint32_t* S = gp.idx.data() + gp.start[bb];
                const std::uint32_t* T = gq.idx.data() + gq.start[bb];
                const std::size_t ns = gp.start[bb + 1] - gp.start[bb], mt = gq.start[bb + 1] - gq.start[bb];
                if (!ns || !mt) continue;
                const std::size_t mbp = (mt + 7) / 8 * 8;
                wp.assign(l * mbp, 0.0);
                for (std::size_t a = 0; a < l; ++a)
                    for (std::size_t y = 0; y < mt; ++y) wp[a * mbp + y] = W[a * m + T[y]];
                for (std::size_t x0 = 0; x0 < ns; x0 += 4) {
                    const std::size_t nx = std::min<std::size_t>(4, ns - x0);
                    const double* u[4];
                    for (std::size_t r = 0; r < 4; ++r) u[r] = U + static_cast<std::size_t>(S[x0 + std::min(r, nx - 1)]) * l;
                    for (std::size_t y0 = 0; y0 < mbp; y0 += 8) {
                        v4d s[4][2];
                        for (int r = 0; r < 4; ++r) s[r][0] = s[r][1] = v4d{0.0, 0.0, 0.0, 0.0};
                        const double* wc = wp.data() + y0;
                        for (std::size_t a = 0; a < l; ++a) {
                            v4d w0, w1;
                            std::memcpy(&w0, wc + a * mbp, 32);
                            std::memcpy(&w1, wc + a * mbp + 4, 32);
                            for (int r = 0; r < 4; ++r) {
                                const double ua = u[r][a];
                                const v4d uv = {ua, ua, ua, ua};
                                s[r][0] = s[r][0] + uv * w0;
                                s[r][1] = s[r][1] + uv * w1;
                            }
                        }
                        for (std::size_t r = 0; r < nx; ++r) {
                            const std::uint32_t i = S[x0 + r];
                            const std::uint32_t* cb = c.col.data() + c.row_ptr[i];
                            const std::uint32_t* ce = c.col.data() + c.row_ptr[i + 1];
                            for (std::size_t y = y0; y < std::min(y0 + 8, mt); ++y) {
                                const std::uint32_t j = T[y];
                                bool earlier = false;  // the pair belongs to an earlier band's block
                                for (int b2 = 0; b2 < band && !earlier; ++b2)
                                    earlier = ids_p[static_cast<std::size_t>(b2) * n + i] ==
                                              ids_q[static_cast<std::size_t>(b2) * m + j];
                                if (earlier) continue;
                                const std::uint32_t* it = std::lower_bound(cb, ce, j);
                                if (it == ce || *it != j)
                                    throw InvalidArgument("build_correction_blocked: pair outside the support");
                                const std::size_t e = static_cast<std::size_t>(it - c.col.data());
                                ++visited;
                                const double exact = std::exp(c.log_sp[e]);
                                if (std::isinf(exact)) {
                                    overflow = true;
                                    continue;
                                }
                                const double nys = s[r][(y - y0) / 4][(y - y0) % 4];
                                c.nys_vals[e] = nys;
                                c.delta[e] = exact - nys;
                                max_abs = std::max(max_abs, std::abs(c.delta[e]));
                            }
                        }
                    }
                }
            }
        }
    }
    if (overflow) throw StabilizationError("build_correction: kernel value overflows linear space");
    if (visited != c.col.size())
        throw InvalidArgument("build_correction_blocked: support is not the union of the bucket blocks");
    c.max_abs_delta = max_abs;
    c.build_csc();
    return c;
}

}  // namespace lcn
