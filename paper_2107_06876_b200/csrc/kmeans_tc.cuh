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
                      const uint32_t* rows = nullptr, float* ub = nullptr, float* lb = nullptr,
                      const int* tl_off = nullptr, const int* tl = nullptr, float* lbt = nullptr,
                      const uint32_t* perm = nullptr);
// tile skipping (Lloyd): with tl_off / tl, cluster c of the launch (2 CTAs,
// 256 consecutive points of the call) evaluates only the centroid tiles
// tl[tl_off[c] .. tl_off[c + 1]) (ascending); lbt (2 floats per point and
// tile of 128 centroids, point-major) receives per evaluated tile a lower
// bound on the true distance to all of its centroids (one per half tile).
// perm (slot -> centroid index): the centroids are packed into tiles in
// that order (tiles of nearby centroids skip better); outputs stay in
// centroid indices.
int assign_tc_tile_count(int k);
// the filter's work counter on the current device: point x 128-centroid tile
// products evaluated since the last reset (synchronous read)
unsigned long long tc_point_tiles(bool reset);
}  // namespace lcnb
