#pragma once
#include <cstdint>

#include "ctx.cuh"

namespace lcnb {
// tcgen05 (3xTF32) assignment filter, see kmeans_tc.cu: writes the assignment
// of every unambiguous point to out[] and appends the others to amb[]
// (count in *namb). Returns false when the shape is not handled.
bool assign_filter_tc(Ctx& ctx, const float* X, long long N, int d, const double* C, int k, uint32_t* out,
                      uint32_t* amb, unsigned* namb, float* dbg_acc = nullptr, int hh_only = 0);
}  // namespace lcnb
