// Bucket-sharded partition plan (shard.h) and its C-ABI query.
//
// The shard unit is the band-0 bucket: neighbor_pairs emits every pair inside
// a bucket (lsh.cpp:222-239), so a rank that owns a band-0 bucket's sources
// and targets holds that whole block. Later bands' buckets are different
// clusterings of the same points; the plan keeps them local where it can by
// grouping band-0 buckets that share later-band buckets before assigning
// groups to ranks:
//   1. cost of band-0 bucket c: modelled bytes per iteration of its points
//      (band blocks in both passes + the low-rank rows),
//   2. affinity: for each later-band bucket, every band-0 bucket among its
//      members is tied to the bucket's dominant band-0 bucket with weight =
//      its member count there,
//   3. Kruskal merge by affinity, heaviest first, while a group stays under
//      half a rank's share,
//   4. groups -> ranks by longest-processing-time greedy.
// Halo: a point owned by rank o is read by rank r != o when one of its
// later-band buckets holds a point of the other side owned by r.
#include "shard.h"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/lcn_b200.h"

namespace lcnb {

namespace {

struct Dsu {
    std::vector<uint32_t> p;
    explicit Dsu(size_t n) : p(n) { std::iota(p.begin(), p.end(), 0u); }
    uint32_t find(uint32_t x) {
        while (p[x] != x) x = p[x] = p[p[x]];
        return x;
    }
};

}  // namespace

ShardPlan make_shard_plan(const uint32_t* ids_src, size_t n, const uint32_t* ids_tgt, size_t m, int bands,
                          const uint32_t* range, size_t l, int world) {
    if (world < 1 || world > 64) throw std::invalid_argument("shard plan: world size must be in [1, 64]");
    if (bands < 1) throw std::invalid_argument("shard plan: the sharded solve needs at least one LSH band");
    if (n >= 0xffffffffull || m >= 0xffffffffull) throw std::invalid_argument("shard plan: more than 2^32 points");
    ShardPlan P;
    P.world = world;
    P.bands = bands;
    P.n = n;
    P.m = m;
    P.l = l;
    P.range.assign(range, range + bands);
    for (int b = 0; b < bands; ++b) {
        for (size_t i = 0; i < n; ++i)
            if (ids_src[b * n + i] >= range[b]) throw std::invalid_argument("shard plan: bucket id out of range");
        for (size_t j = 0; j < m; ++j)
            if (ids_tgt[b * m + j] >= range[b]) throw std::invalid_argument("shard plan: bucket id out of range");
    }
    const size_t nb0 = range[0];
    const double lp = static_cast<double>((l + 3) / 4 * 4);
    std::vector<double> ns(nb0, 0.0), mt(nb0, 0.0);
    for (size_t i = 0; i < n; ++i) ns[ids_src[i]] += 1.0;
    for (size_t j = 0; j < m; ++j) mt[ids_tgt[j]] += 1.0;
    // 1. modelled bytes per iteration: band-0 block in both passes (fp32),
    // a later band of similar size, low-rank rows (fp32, lp columns) and the
    // per-row vectors
    std::vector<double> cost(nb0);
    double total = 0.0;
    for (size_t c = 0; c < nb0; ++c) {
        cost[c] = 8.0 * ns[c] * mt[c] * bands + (4.0 * lp + 64.0) * (ns[c] + mt[c]);
        total += cost[c];
    }
    // 2. affinity edges (c, dominant band-0 bucket of the later-band bucket)
    std::vector<std::pair<uint64_t, double>> edges;  // key = c1 << 32 | c2 (c1 < c2)
    for (int b = 1; b < bands; ++b) {
        std::vector<uint64_t> keys;  // (later-band bucket, band-0 bucket) per point
        keys.reserve(n + m);
        for (size_t i = 0; i < n; ++i) keys.push_back(uint64_t(ids_src[b * n + i]) << 32 | ids_src[i]);
        for (size_t j = 0; j < m; ++j) keys.push_back(uint64_t(ids_tgt[b * m + j]) << 32 | ids_tgt[j]);
        std::sort(keys.begin(), keys.end());
        size_t a = 0;
        while (a < keys.size()) {
            const uint64_t bk = keys[a] >> 32;
            size_t e = a;
            while (e < keys.size() && (keys[e] >> 32) == bk) ++e;
            // runs of equal band-0 bucket inside [a, e)
            std::vector<std::pair<uint32_t, double>> runs;
            for (size_t x = a; x < e;) {
                size_t y = x;
                while (y < e && keys[y] == keys[x]) ++y;
                runs.push_back({static_cast<uint32_t>(keys[x] & 0xffffffffu), double(y - x)});
                x = y;
            }
            uint32_t dom = runs[0].first;
            double best = runs[0].second;
            for (const auto& r : runs)
                if (r.second > best) { best = r.second; dom = r.first; }
            for (const auto& r : runs)
                if (r.first != dom) {
                    const uint32_t c1 = std::min(r.first, dom), c2 = std::max(r.first, dom);
                    edges.push_back({uint64_t(c1) << 32 | c2, r.second});
                }
            a = e;
        }
    }
    std::sort(edges.begin(), edges.end());
    std::vector<std::pair<uint64_t, double>> merged;
    for (const auto& e : edges) {
        if (!merged.empty() && merged.back().first == e.first) merged.back().second += e.second;
        else merged.push_back(e);
    }
    std::stable_sort(merged.begin(), merged.end(),
                     [](const auto& x, const auto& y) { return x.second > y.second; });
    // 3. capped Kruskal merge
    Dsu dsu(nb0);
    std::vector<double> gcost = cost;
    const double cap = world > 1 ? total / world / 2.0 : total;
    for (const auto& e : merged) {
        uint32_t a = dsu.find(static_cast<uint32_t>(e.first >> 32)), b = dsu.find(static_cast<uint32_t>(e.first));
        if (a == b || gcost[a] + gcost[b] > cap) continue;
        if (b < a) std::swap(a, b);
        dsu.p[b] = a;
        gcost[a] += gcost[b];
    }
    // 4. LPT over the groups (largest first, ties by root id), least-loaded rank
    std::vector<uint32_t> roots;
    for (uint32_t c = 0; c < nb0; ++c)
        if (dsu.find(c) == c) roots.push_back(c);
    P.groups = roots.size();
    std::stable_sort(roots.begin(), roots.end(), [&](uint32_t x, uint32_t y) { return gcost[x] > gcost[y]; });
    std::vector<int> owner_root(nb0, 0);
    {
        using Load = std::pair<double, int>;
        std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
        for (int r = 0; r < world; ++r) heap.push({0.0, r});
        for (uint32_t g : roots) {
            Load ld = heap.top();
            heap.pop();
            owner_root[g] = ld.second;
            ld.first += gcost[g];
            heap.push(ld);
        }
    }
    P.owner0.resize(nb0);
    P.ranks.assign(world, ShardRank{});
    for (uint32_t c = 0; c < nb0; ++c) {
        P.owner0[c] = owner_root[dsu.find(c)];
        P.ranks[P.owner0[c]].cost += cost[c];
        P.ranks[P.owner0[c]].band0_pairs += static_cast<unsigned long long>(ns[c] * mt[c]);
    }
    // owners and halo masks
    std::vector<uint8_t> own_s(n), own_t(m);
    for (size_t i = 0; i < n; ++i) own_s[i] = static_cast<uint8_t>(P.owner0[ids_src[i]]);
    for (size_t j = 0; j < m; ++j) own_t[j] = static_cast<uint8_t>(P.owner0[ids_tgt[j]]);
    std::vector<uint64_t> halo_s(n, 0), halo_t(m, 0);  // ranks that read the point
    for (int b = 1; b < bands; ++b) {
        std::vector<uint64_t> smask(range[b], 0), tmask(range[b], 0);
        for (size_t i = 0; i < n; ++i) smask[ids_src[b * n + i]] |= uint64_t(1) << own_s[i];
        for (size_t j = 0; j < m; ++j) tmask[ids_tgt[b * m + j]] |= uint64_t(1) << own_t[j];
        for (size_t i = 0; i < n; ++i) halo_s[i] |= tmask[ids_src[b * n + i]];
        for (size_t j = 0; j < m; ++j) halo_t[j] |= smask[ids_tgt[b * m + j]];
    }
    for (size_t i = 0; i < n; ++i) halo_s[i] &= ~(uint64_t(1) << own_s[i]);
    for (size_t j = 0; j < m; ++j) halo_t[j] &= ~(uint64_t(1) << own_t[j]);
    // local orders, exports (slot of each exported point), imports
    auto side = [&](size_t cnt, const std::vector<uint8_t>& own, const std::vector<uint64_t>& halo, bool src) {
        std::vector<uint32_t> slot(cnt, 0xffffffffu);
        std::vector<uint32_t> own_local(cnt, 0);
        for (int r = 0; r < world; ++r) {
            ShardRank& R = P.ranks[r];
            std::vector<uint32_t>& loc = src ? R.src : R.tgt;
            std::vector<uint32_t>& ex = src ? R.exp_s : R.exp_t;
            loc.clear();
            for (size_t i = 0; i < cnt; ++i)
                if (own[i] == r) {
                    own_local[i] = static_cast<uint32_t>(loc.size());
                    if (halo[i]) {
                        slot[i] = static_cast<uint32_t>(ex.size());
                        ex.push_back(own_local[i]);
                    }
                    loc.push_back(static_cast<uint32_t>(i));
                }
            (src ? R.n_own : R.m_own) = static_cast<uint32_t>(loc.size());
        }
        for (int r = 0; r < world; ++r) {
            ShardRank& R = P.ranks[r];
            std::vector<uint32_t>& loc = src ? R.src : R.tgt;
            std::vector<uint32_t>& ir = src ? R.imp_s_rank : R.imp_t_rank;
            std::vector<uint32_t>& is = src ? R.imp_s_slot : R.imp_t_slot;
            for (size_t i = 0; i < cnt; ++i)
                if (halo[i] >> r & 1u) {
                    loc.push_back(static_cast<uint32_t>(i));
                    ir.push_back(own[i]);
                    is.push_back(slot[i]);
                }
        }
    };
    side(n, own_s, halo_s, true);
    side(m, own_t, halo_t, false);
    for (const ShardRank& R : P.ranks) {
        P.max_exp_s = std::max(P.max_exp_s, R.exp_s.size());
        P.max_exp_t = std::max(P.max_exp_t, R.exp_t.size());
    }
    return P;
}

}  // namespace lcnb

// ---------------------------------------------------------------------------
// C-ABI query (host only: callable without a GPU)
// ---------------------------------------------------------------------------
struct lcn_shard_plan {
    lcnb::ShardPlan p;
};

namespace {
thread_local std::string g_plan_error;

template <typename F>
int plan_guard(F&& f) {
    try {
        f();
        return LCN_OK;
    } catch (const std::exception& e) {
        g_plan_error = e.what();
        return LCN_E_INVALID_ARGUMENT;
    }
}
const lcnb::ShardRank& rank_of(const lcn_shard_plan* plan, int rank) {
    if (!plan) throw std::invalid_argument("shard plan: null handle");
    if (rank < 0 || rank >= plan->p.world) throw std::invalid_argument("shard plan: rank out of range");
    return plan->p.ranks[rank];
}
void put(uint32_t* out, const std::vector<uint32_t>& v) {
    if (out && !v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
}
}  // namespace

extern "C" {

int lcn_shard_plan_create(const uint32_t* ids_src, size_t n, const uint32_t* ids_tgt, size_t m, int bands,
                          const uint32_t* range, size_t l, int world, lcn_shard_plan** out) {
    return plan_guard([&] {
        if (!out || !range || (n && !ids_src) || (m && !ids_tgt)) throw std::invalid_argument("shard plan: null pointer");
        auto h = new lcn_shard_plan();
        try {
            h->p = lcnb::make_shard_plan(ids_src, n, ids_tgt, m, bands, range, l, world);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int lcn_shard_plan_destroy(lcn_shard_plan* plan) {
    delete plan;
    return LCN_OK;
}

const char* lcn_shard_plan_last_error(void) { return g_plan_error.c_str(); }

int lcn_shard_plan_rank_info(const lcn_shard_plan* plan, int rank, lcn_shard_rank_info* info) {
    return plan_guard([&] {
        const lcnb::ShardRank& R = rank_of(plan, rank);
        if (!info) throw std::invalid_argument("shard plan: null info");
        info->n_own = R.n_own;
        info->n_halo = R.src.size() - R.n_own;
        info->m_own = R.m_own;
        info->m_halo = R.tgt.size() - R.m_own;
        info->exp_s = R.exp_s.size();
        info->exp_t = R.exp_t.size();
        info->max_exp_s = plan->p.max_exp_s;
        info->max_exp_t = plan->p.max_exp_t;
        info->cost = R.cost;
        info->band0_pairs = R.band0_pairs;
        info->groups = plan->p.groups;
    });
}

int lcn_shard_plan_rank_points(const lcn_shard_plan* plan, int rank, uint32_t* src, uint32_t* tgt) {
    return plan_guard([&] {
        const lcnb::ShardRank& R = rank_of(plan, rank);
        put(src, R.src);
        put(tgt, R.tgt);
    });
}

int lcn_shard_plan_rank_exchange(const lcn_shard_plan* plan, int rank, uint32_t* exp_s, uint32_t* exp_t,
                                 uint32_t* imp_s_rank, uint32_t* imp_s_slot, uint32_t* imp_t_rank,
                                 uint32_t* imp_t_slot) {
    return plan_guard([&] {
        const lcnb::ShardRank& R = rank_of(plan, rank);
        put(exp_s, R.exp_s);
        put(exp_t, R.exp_t);
        put(imp_s_rank, R.imp_s_rank);
        put(imp_s_slot, R.imp_s_slot);
        put(imp_t_rank, R.imp_t_rank);
        put(imp_t_slot, R.imp_t_slot);
    });
}

}  // extern "C"
