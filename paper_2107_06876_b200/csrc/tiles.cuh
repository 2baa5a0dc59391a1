// Tiled exact pairwise evaluation shared by k-means assignment, the K_sp
// bucket blocks, the Nystrom factors and the LCN correction.
#pragma once
#include "common.cuh"

namespace lcnb {

// ---------------------------------------------------------------------------
// Tiled exact pairwise evaluation. A CTA of 256 threads covers a 64 x 64 tile
// of (row, col) pairs, staging KC-wide slabs of both operand rows in shared
// memory; each thread owns a 4 x 4 register tile and folds over the feature
// index in increasing order, so every pair's value is bit-identical to the
// reference's sequential loop.
// ---------------------------------------------------------------------------
constexpr int TP = 64, TC = 64, KC = 16;

template <int MODE>  // 0: sum (a-b)^2   1: sum a*b
__device__ __forceinline__ void tile_fold(const double (*As)[TP + 1], const double (*Bs)[TC + 1], int ty, int tx,
                                          double acc[4][4]) {
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (MODE == 0) {
                    double df = xsub(a[i], b[j]);
                    acc[i][j] = xadd(acc[i][j], xmul(df, df));
                } else {
                    acc[i][j] = xadd(acc[i][j], xmul(a[i], b[j]));
                }
            }
    }
}

// Loads a KC-slab (features [k0, k0+KC)) of 64 gathered rows into S[kk][r].
template <typename T>
__device__ __forceinline__ void load_slab(double (*S)[TP + 1], const T* __restrict__ X, const uint32_t* rows,
                                          long long row0, long long nrows, int d, int k0) {
    for (int e = threadIdx.x; e < TP * KC; e += blockDim.x) {
        int r = e / KC, kk = e % KC;
        long long rr = row0 + r;
        double v = 0.0;
        if (rr < nrows && k0 + kk < d) {
            long long src = rows ? rows[rr] : rr;
            v = static_cast<double>(X[src * d + k0 + kk]);
        }
        S[kk][r] = v;
    }
}

}  // namespace lcnb
