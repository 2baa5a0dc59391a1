#pragma once
#include <vector>

#include "ctx.cuh"

namespace lcnb {

// kmeans_pp_indices (kmeans.cpp:23-65). raw = the caller engine's 64-bit draws.
template <typename T>
void kmeans_pp_device(Ctx& ctx, const T* X, long long N, int d, int k, uint64_t first,
                      const std::vector<unsigned long long>& raw, uint32_t* d_chosen, int* draws_used);
// One k-means++ sequence of a batch: k seeds, the first index and the
// engine's draws (as kmeans_pp_device), the k indices go to d_chosen.
struct PPSeq {
    int k;
    uint64_t first;
    std::vector<unsigned long long> raw;
    uint32_t* d_chosen;
    int* draws_used;
};
// Several sequences over the same points in one step chain (each kernel
// launch serves all of them); results identical to separate calls.
template <typename T>
void kmeans_pp_batch(Ctx& ctx, const T* X, long long N, int d, const std::vector<PPSeq>& seqs);
// The sequence lloyd(seed) seeds with (kmeans.cpp:93-94): mt19937_64(seed),
// first = uniform_int(0, N - 1), then k - 1 raw draws.
PPSeq lloyd_seed_seq(uint64_t seed, long long N, int k, uint32_t* d_chosen);
// assign_nearest (kmeans.cpp:67-85).
template <typename T>
void assign_device(Ctx& ctx, const T* X, long long N, int d, const double* C, int k, uint32_t* out);
// lloyd (kmeans.cpp:87-143): centroids (k x d) and assignment, both device.
// init: the k-means++ indices when already seeded (kmeans_pp_batch), else
// seeded here from seed.
template <typename T>
void lloyd_device(Ctx& ctx, const T* X, long long N, int d, int k, int iters, uint64_t seed, double* d_ctr,
                  uint32_t* d_assign, const uint32_t* init = nullptr);

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
