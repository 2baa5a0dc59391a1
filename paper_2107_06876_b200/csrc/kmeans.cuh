#pragma once
#include <vector>

#include "ctx.cuh"

namespace lcnb {

// kmeans_pp_indices (kmeans.cpp:23-65). raw = the caller engine's 64-bit draws.
template <typename T>
void kmeans_pp_device(Ctx& ctx, const T* X, long long N, int d, int k, uint64_t first,
                      const std::vector<unsigned long long>& raw, uint32_t* d_chosen, int* draws_used);
// assign_nearest (kmeans.cpp:67-85).
template <typename T>
void assign_device(Ctx& ctx, const T* X, long long N, int d, const double* C, int k, uint32_t* out);
// lloyd (kmeans.cpp:87-143): centroids (k x d) and assignment, both device.
template <typename T>
void lloyd_device(Ctx& ctx, const T* X, long long N, int d, int k, int iters, uint64_t seed, double* d_ctr,
                  uint32_t* d_assign);

// lsh.cpp:17-27
inline uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline uint64_t fn_seed(uint64_t seed, int band, int fn) {
    return mix64(seed ^ mix64(static_cast<uint64_t>(band) * 0x100000001b3ull + static_cast<uint64_t>(fn)));
}

}  // namespace lcnb
