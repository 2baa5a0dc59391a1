// Support diagnostic of the sparse operator (sinkhorn.cpp:122-128 ->
// sparse_kernel.cpp:189-244 -> matching.cpp:12-92): a maximum bipartite
// matching over the CSR pattern; the pattern has support iff it matches
// min(n, m) rows. Host-side (it only feeds a warning).
// Hopcroft-Karp with BFS layering and an explicit-stack DFS.
#include <cstddef>
#include <cstdint>
#include <limits>
#include <vector>

namespace lcnb {

size_t max_bipartite_matching(size_t n, size_t m, const uint32_t* row_ptr, const uint32_t* col) {
    constexpr uint32_t kNone = std::numeric_limits<uint32_t>::max();
    std::vector<uint32_t> mate_l(n, kNone), mate_r(m, kNone), layer(n), queue(n), it(n), stack;
    size_t matched = 0;
    while (true) {
        // BFS from free left vertices.
        size_t qh = 0, qt = 0;
        bool found = false;
        for (size_t i = 0; i < n; ++i) {
            if (mate_l[i] == kNone) {
                layer[i] = 0;
                queue[qt++] = static_cast<uint32_t>(i);
            } else {
                layer[i] = kNone;
            }
        }
        while (qh < qt) {
            uint32_t u = queue[qh++];
            for (uint32_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
                uint32_t w = mate_r[col[e]];
                if (w == kNone) {
                    found = true;
                } else if (layer[w] == kNone) {
                    layer[w] = layer[u] + 1;
                    queue[qt++] = w;
                }
            }
        }
        if (!found) break;
        // DFS along layers.
        for (size_t i = 0; i < n; ++i) it[i] = row_ptr[i];
        for (size_t root = 0; root < n; ++root) {
            if (mate_l[root] != kNone) continue;
            stack.assign(1, static_cast<uint32_t>(root));
            bool augmented = false;
            while (!stack.empty() && !augmented) {
                uint32_t u = stack.back();
                if (it[u] == row_ptr[u + 1]) {
                    layer[u] = kNone;  // dead end
                    stack.pop_back();
                    continue;
                }
                uint32_t v = col[it[u]++];
                uint32_t w = mate_r[v];
                if (w == kNone) {
                    // augment along the stack
                    for (size_t k = stack.size(); k-- > 0;) {
                        uint32_t x = stack[k];
                        uint32_t prev = mate_l[x];
                        mate_l[x] = v;
                        mate_r[v] = x;
                        v = prev;
                    }
                    augmented = true;
                } else if (layer[w] != kNone && layer[w] == layer[u] + 1) {
                    stack.push_back(w);
                }
            }
            if (augmented) ++matched;
        }
    }
    return matched;
}

}  // namespace lcnb
