// Bucket-sharded partition of one LCN problem over the ranks of a
// communicator: points are owned by the rank of their
// band-0 bucket, so the band-0 blocks -- the bulk of the support -- stay on
// one rank; a later band's bucket that spans ranks makes each participating
// rank read the other ranks' members as halo points. Host-only C++ (no CUDA),
// shared by the library's sharded build / solve and by the C-ABI plan query
// (lcn_shard_plan_*), which the CPU multi-rank tests drive.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace lcnb {

struct ShardRank {
    // local point order: owned points ascending by global index, then halo
    // points ascending by global index
    std::vector<uint32_t> src, tgt;          // local -> global
    uint32_t n_own = 0, m_own = 0;
    // exported: local indices (< n_own / m_own) of owned points some other
    // rank reads as halo, ascending global index; this rank's slot k of the
    // exchange buffer carries the value of exp_*[k]
    std::vector<uint32_t> exp_s, exp_t;
    // per halo point (local index n_own + k): owner rank and its slot
    std::vector<uint32_t> imp_s_rank, imp_s_slot, imp_t_rank, imp_t_slot;
    double cost = 0.0;                       // modelled bytes per iteration
    unsigned long long band0_pairs = 0;      // sum n_b m_b over owned band-0 buckets
};

struct ShardPlan {
    int world = 1, bands = 0;
    size_t n = 0, m = 0, l = 0;
    std::vector<uint32_t> range;             // bucket range per band
    std::vector<int> owner0;                 // band-0 bucket -> rank
    std::vector<ShardRank> ranks;
    size_t max_exp_s = 0, max_exp_t = 0;     // exchange slots per rank (padded length)
    size_t groups = 0;                       // band-0 bucket groups before the rank assignment
};

// ids_src: bands x n, ids_tgt: bands x m (dense bucket ids < range[b]).
// Deterministic: every rank computes the same plan from the same ids.
ShardPlan make_shard_plan(const uint32_t* ids_src, size_t n, const uint32_t* ids_tgt, size_t m, int bands,
                          const uint32_t* range, size_t l, int world);

}  // namespace lcnb
