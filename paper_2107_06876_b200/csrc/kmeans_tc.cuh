#pragma once
#include <cstdint>

#include "ctx.cuh"

namespace lcnb {
// tcgen05 (3xTF32) assignment filter, see kmeans_tc.cu: writes the assignment
// of every unambiguous point to out[] and appends the others to amb[]
// (count in *namb). Returns false when the shape is not handled. With rows,
// the call covers the points rows[0 .. N) (out / amb hold their indices);
// with ub / lb it also writes, per unambiguous point, an upper bound on its
// true distance to the chosen centroid and a lower bound on its distance to
// every other centroid (Lloyd's bound test, lloyd_device).
bool assign_filter_tc(Ctx& ctx, const float* X, long long N, int d, const double* C, int k, uint32_t* out,
                      uint32_t* amb, unsigned* namb, float* dbg_acc = nullptr, int hh_only = 0,
                      const uint32_t* rows = nullptr, float* ub = nullptr, float* lb = nullptr);
}  // namespace lcnb
