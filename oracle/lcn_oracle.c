/*
 * ORACLE TEST INFRASTRUCTURE — CPU restatement of the reference hot path
 * (/root/reference/proj), plain C11, single-threaded, fp64 with no FMA
 * contraction (built with -ffp-contract=off, no -march).
 * Every function names the reference lines it restates. See lcn_oracle.h for
 * how it is pinned. Never linked into the product.
 */
#include "lcn_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- errors (error.hpp:8-38 -> status codes) ---------------------------- */
enum { E_DIM = 1, E_ARG = 2, E_STAB = 3, E_NEG = 4, E_FACT = 5 };
static _Thread_local char g_err[512];
static _Thread_local int g_code;

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    g_code = code;
    return code;
}
const char* orc_last_error(void) { return g_err; }

#define TRY(x)                 \
    do {                       \
        int rc__ = (x);        \
        if (rc__) return rc__; \
    } while (0)

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) abort();
    return p;
}

/* ---- libstdc++ <random> (GCC 13) ------------------------------------------ */
/* std::mt19937_64 (a standard-specified engine). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

/* uniform_int_distribution<size_t>(0, n-1): Lemire's nearly divisionless
 * downscaling with a 128-bit product (bits/uniform_int_dist.h, _S_nd). */
static uint64_t uniform_index(mt64* g, uint64_t n) {
    unsigned __int128 prod = (unsigned __int128)mt64_next(g) * n;
    uint64_t low = (uint64_t)prod;
    if (low < n) {
        uint64_t thr = (uint64_t)(-n) % n;
        while (low < thr) {
            prod = (unsigned __int128)mt64_next(g) * n;
            low = (uint64_t)prod;
        }
    }
    return (uint64_t)(prod >> 64);
}

/* uniform_real_distribution<double>(0, b): generate_canonical<double, 53>
 * (bits/random.tcc) = double(u)/2^64 clamped below 1, times (b - 0) plus 0. */
static double uniform_real(mt64* g, double b) {
    double sum = (double)mt64_next(g);
    double c = sum / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return c * (b - 0.0) + 0.0;
}

uint64_t orc_mt19937_64_nth(uint64_t seed, size_t skip) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t i = 0; i < skip; ++i) mt64_next(&g);
    return mt64_next(&g);
}
uint64_t orc_uniform_index(uint64_t seed, uint64_t n) {
    mt64 g;
    mt64_seed(&g, seed);
    return uniform_index(&g, n);
}

/* ---- k-means (kmeans.cpp) ------------------------------------------------- */
/* kmeans.cpp:12-19 */
static double sqdist(const double* x, const double* y, size_t d) {
    double s = 0.0;
    for (size_t k = 0; k < d; ++k) {
        double diff = x[k] - y[k];
        s += diff * diff;
    }
    return s;
}

/* kmeans.cpp:23-65 */
static int kmeans_pp(const double* pts, size_t n, size_t d, size_t k, mt64* rng, uint32_t* chosen) {
    if (k == 0 || k > n) return fail(E_ARG, "kmeans++: k must be in [1, n]");
    chosen[0] = (uint32_t)uniform_index(rng, n);
    double* dist2 = xmalloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) dist2[i] = INFINITY;
    for (size_t t = 1; t < k; ++t) {
        const double* last = pts + (size_t)chosen[t - 1] * d;
        double total = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double d2 = sqdist(pts + i * d, last, d);
            if (d2 < dist2[i]) dist2[i] = d2;
            total += dist2[i];
        }
        size_t pick;
        if (total <= 0.0) {
            char* used = xcalloc(n, 1);
            for (size_t c = 0; c < t; ++c) used[chosen[c]] = 1;
            pick = 0;
            while (pick < n && used[pick]) ++pick;
            free(used);
        } else {
            double target = uniform_real(rng, total);
            double acc = 0.0;
            pick = n - 1;
            for (size_t i = 0; i < n; ++i) {
                acc += dist2[i];
                if (acc >= target && dist2[i] > 0.0) {
                    pick = i;
                    break;
                }
            }
        }
        chosen[t] = (uint32_t)pick;
        dist2[pick] = 0.0;
    }
    free(dist2);
    return 0;
}

/* kmeans.cpp:67-85 */
static void assign_nearest(const double* pts, size_t n, size_t d, const double* ctr, size_t k, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) {
        double best = INFINITY;
        uint32_t arg = 0;
        for (size_t c = 0; c < k; ++c) {
            double d2 = sqdist(pts + i * d, ctr + c * d, d);
            if (d2 < best) {
                best = d2;
                arg = (uint32_t)c;
            }
        }
        out[i] = arg;
    }
}

/* kmeans.cpp:87-143 */
static int lloyd(const double* pts, size_t n, size_t d, size_t k, int iters, uint64_t seed, double* ctr,
                 uint32_t* assign) {
    if (n == 0) return fail(E_ARG, "k-means on empty input");
    if (k == 0 || k > n) return fail(E_ARG, "k-means: more buckets than points");
    mt64 rng;
    mt64_seed(&rng, seed);
    uint32_t* init = xmalloc(k * sizeof(uint32_t));
    TRY(kmeans_pp(pts, n, d, k, &rng, init));
    for (size_t c = 0; c < k; ++c) memcpy(ctr + c * d, pts + (size_t)init[c] * d, d * sizeof(double));
    free(init);
    memset(assign, 0, n * sizeof(uint32_t));
    size_t* counts = xcalloc(k, sizeof(size_t));
    double* sums = xmalloc(k * d * sizeof(double));
    for (int it = 0; it < iters; ++it) {
        assign_nearest(pts, n, d, ctr, k, assign);
        memset(sums, 0, k * d * sizeof(double));
        memset(counts, 0, k * sizeof(size_t));
        for (size_t i = 0; i < n; ++i) {
            uint32_t c = assign[i];
            ++counts[c];
            for (size_t kk = 0; kk < d; ++kk) sums[c * d + kk] += pts[i * d + kk];
        }
        for (size_t c = 0; c < k; ++c) {
            if (counts[c] == 0) continue;
            double inv = 1.0 / (double)counts[c];
            for (size_t kk = 0; kk < d; ++kk) ctr[c * d + kk] = sums[c * d + kk] * inv;
        }
        for (size_t c = 0; c < k; ++c) {
            if (counts[c] != 0) continue;
            double far = -1.0;
            size_t arg = 0;
            for (size_t i = 0; i < n; ++i) {
                if (counts[assign[i]] <= 1) continue;
                double d2 = sqdist(pts + i * d, ctr + (size_t)assign[i] * d, d);
                if (d2 > far) {
                    far = d2;
                    arg = i;
                }
            }
            memcpy(ctr + c * d, pts + arg * d, d * sizeof(double));
            --counts[assign[arg]];
            assign[arg] = (uint32_t)c;
            counts[c] = 1;
        }
    }
    assign_nearest(pts, n, d, ctr, k, assign);
    free(counts);
    free(sums);
    return 0;
}

int orc_kmeans_pp(const double* pts, size_t n, size_t d, size_t k, uint64_t seed, uint32_t* out) {
    mt64 g;
    mt64_seed(&g, seed);
    return kmeans_pp(pts, n, d, k, &g, out);
}
int orc_assign_nearest(const double* pts, size_t n, size_t d, const double* ctr, size_t k, uint32_t* out) {
    assign_nearest(pts, n, d, ctr, k, out);
    return 0;
}
int orc_lloyd(const double* pts, size_t n, size_t d, size_t k, int iters, uint64_t seed, double* centroids,
              uint32_t* assign) {
    return lloyd(pts, n, d, k, iters, seed, centroids, assign);
}

/* ---- LSH (lsh.cpp) ------------------------------------------------------- */
/* lsh.cpp:17-27 */
static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static uint64_t fn_seed(uint64_t seed, int band, int fn) {
    return mix64(seed ^ mix64((uint64_t)band * 0x100000001b3ull + (uint64_t)fn));
}

typedef struct {
    size_t n, m, nnz;
    uint32_t* row;
    uint32_t* col;
} pairs_t;

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* NeighborPairs::from_pairs (lsh.cpp:163-177): range check, sort, unique. */
static int pairs_from_keys(size_t n, size_t m, uint64_t* keys, size_t cnt, pairs_t** out) {
    for (size_t e = 0; e < cnt; ++e)
        if ((keys[e] >> 32) >= n || (keys[e] & 0xffffffffu) >= m) return fail(E_ARG, "neighbor pair index out of range");
    qsort(keys, cnt, sizeof(uint64_t), cmp_u64);
    size_t u = 0;
    for (size_t e = 0; e < cnt; ++e)
        if (e == 0 || keys[e] != keys[u - 1]) keys[u++] = keys[e];
    pairs_t* p = xcalloc(1, sizeof(pairs_t));
    p->n = n;
    p->m = m;
    p->nnz = u;
    p->row = xmalloc(u * sizeof(uint32_t));
    p->col = xmalloc(u * sizeof(uint32_t));
    for (size_t e = 0; e < u; ++e) {
        p->row[e] = (uint32_t)(keys[e] >> 32);
        p->col[e] = (uint32_t)(keys[e] & 0xffffffffu);
    }
    *out = p;
    return 0;
}

typedef struct {
    uint64_t id;
    uint32_t idx;
} idpair;
static int cmp_idpair(const void* a, const void* b) {
    const idpair *x = a, *y = b;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return x->idx < y->idx ? -1 : x->idx > y->idx;
}

/* neighbor_pairs (lsh.cpp:212-243): group by bucket (sorted_by_bucket,
 * lsh.cpp:193-208, a stable grouping), emit the p x q product per shared
 * bucket per band, then from_pairs. */
static int neighbor_pairs(const uint64_t* ids_p, size_t n, const uint64_t* ids_q, size_t m, int bands,
                          pairs_t** out) {
    size_t cap = 1024, cnt = 0;
    uint64_t* keys = xmalloc(cap * sizeof(uint64_t));
    idpair* sp = xmalloc((n ? n : 1) * sizeof(idpair));
    idpair* sq = xmalloc((m ? m : 1) * sizeof(idpair));
    for (int b = 0; b < bands; ++b) {
        for (size_t i = 0; i < n; ++i) sp[i] = (idpair){ids_p[(size_t)b * n + i], (uint32_t)i};
        for (size_t j = 0; j < m; ++j) sq[j] = (idpair){ids_q[(size_t)b * m + j], (uint32_t)j};
        qsort(sp, n, sizeof(idpair), cmp_idpair);
        qsort(sq, m, sizeof(idpair), cmp_idpair);
        size_t a = 0, c = 0;
        while (a < n && c < m) {
            if (sp[a].id < sq[c].id) ++a;
            else if (sq[c].id < sp[a].id) ++c;
            else {
                uint64_t id = sp[a].id;
                size_t ae = a, ce = c;
                while (ae < n && sp[ae].id == id) ++ae;
                while (ce < m && sq[ce].id == id) ++ce;
                for (size_t x = a; x < ae; ++x)
                    for (size_t y = c; y < ce; ++y) {
                        if (cnt == cap) {
                            cap *= 2;
                            keys = realloc(keys, cap * sizeof(uint64_t));
                            if (!keys) abort();
                        }
                        keys[cnt++] = ((uint64_t)sp[x].idx << 32) | sq[y].idx;
                    }
                a = ae;
                c = ce;
            }
        }
    }
    free(sp);
    free(sq);
    int rc = pairs_from_keys(n, m, keys, cnt, out);
    free(keys);
    return rc;
}

/* lsh.cpp:245-283 (k-means scheme): band b clusters the union with
 * hash_kmeans (lsh.cpp:148-161) = lloyd(seed = fn_seed(seed, b, 0)). */
int orc_lsh_kmeans_buckets(const double* p, size_t n, const double* q, size_t m, size_t d, int bands, int buckets,
                           int iters, uint64_t seed, uint64_t* ids) {
    if (bands < 1) return fail(E_ARG, "lsh: bands and rows_per_band must be >= 1");
    if (buckets < 2) return fail(E_ARG, "lsh: buckets_per_fn must be >= 2");
    size_t N = n + m;
    if ((size_t)buckets > N) return fail(E_ARG, "hash_kmeans: more buckets than points");
    double* all = xmalloc(N * d * sizeof(double));
    memcpy(all, p, n * d * sizeof(double));
    memcpy(all + n * d, q, m * d * sizeof(double));
    double* ctr = xmalloc((size_t)buckets * d * sizeof(double));
    uint32_t* a = xmalloc(N * sizeof(uint32_t));
    int rc = 0;
    for (int b = 0; b < bands && !rc; ++b) {
        rc = lloyd(all, N, d, (size_t)buckets, iters, fn_seed(seed, b, 0), ctr, a);
        for (size_t i = 0; i < N && !rc; ++i) ids[(size_t)b * N + i] = a[i];
    }
    free(all);
    free(ctr);
    free(a);
    return rc;
}

/* normal_distribution<double>(0, 1) over mt19937_64 (bits/random.tcc,
 * Marsaglia polar method): draws come in pairs from two canonical uniforms
 * x, y in [-1, 1) with 0 < r2 = x^2 + y^2 <= 1; the call returns y * mult and
 * caches x * mult for the next call. */
typedef struct {
    mt64 g;
    int saved_ok;
    double saved;
} gauss_t;

static double canonical(mt64* g) {
    double c = (double)mt64_next(g) / 18446744073709551616.0;
    return c >= 1.0 ? nextafter(1.0, 0.0) : c;
}

static double gauss_next(gauss_t* s) {
    if (s->saved_ok) {
        s->saved_ok = 0;
        return s->saved * 1.0 + 0.0;
    }
    double x, y, r2;
    do {
        x = 2.0 * canonical(&s->g) - 1.0;
        y = 2.0 * canonical(&s->g) - 1.0;
        r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    double mult = sqrt(-2 * log(r2) / r2);
    s->saved = x * mult;
    s->saved_ok = 1;
    return y * mult * 1.0 + 0.0;
}

int orc_normal_draws(uint64_t seed, size_t count, double* out) {
    gauss_t s;
    mt64_seed(&s.g, seed);
    s.saved_ok = 0;
    for (size_t i = 0; i < count; ++i) out[i] = gauss_next(&s);
    return 0;
}

/* cross_polytope_bucket (lsh.cpp:55-71): argmax over c of [x^T R || -x^T R],
 * sequential dot, strict > (first maximum). proj is d x half, row-major. */
static uint32_t cp_bucket(const double* x, size_t d, const double* proj, size_t half) {
    double best = -INFINITY;
    uint32_t arg = 0;
    for (size_t c = 0; c < 2 * half; ++c) {
        size_t col = c < half ? c : c - half;
        double v = 0.0;
        for (size_t k = 0; k < d; ++k) v += x[k] * proj[k * half + col];
        if (c >= half) v = -v;
        if (v > best) {
            best = v;
            arg = (uint32_t)c;
        }
    }
    return arg;
}

int orc_cross_polytope_bucket(const double* x, size_t n, size_t d, const double* proj, size_t half, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = cp_bucket(x + i * d, d, proj, half);
    return 0;
}

/* hierarchical_assign (lsh.cpp:107-143): FIFO queue of clusters; a cluster
 * is a leaf once queue + leaves + 1 >= target or it has < 2 points, else
 * lloyd(k = min(branching, size), iters, mix64(seed ^ ++splits)) splits it and
 * the non-empty children are queued in child order. */
typedef struct {
    uint32_t* idx;
    size_t len;
} cluster_t;

static int hierarchical_assign(const double* pts, size_t n, size_t d, size_t target, int branching, int iters,
                               uint64_t seed, uint32_t* assign) {
    /* the queue never holds more than n clusters; a ring of n + 1 slots */
    size_t cap = n + 1, head = 0, tail = 0, qn = 0, nleaves = 0;
    cluster_t* q = xmalloc(cap * sizeof(cluster_t));
    cluster_t* leaves = xmalloc(cap * sizeof(cluster_t));
    q[tail].idx = xmalloc((n ? n : 1) * sizeof(uint32_t));
    q[tail].len = n;
    for (size_t i = 0; i < n; ++i) q[tail].idx[i] = (uint32_t)i;
    tail = (tail + 1) % cap;
    qn = 1;
    uint64_t splits = 0;
    double* sub = xmalloc((n ? n : 1) * d * sizeof(double));
    double* ctr = xmalloc((size_t)branching * d * sizeof(double));
    uint32_t* a = xmalloc((n ? n : 1) * sizeof(uint32_t));
    size_t* cnt = xmalloc((size_t)branching * sizeof(size_t));
    int rc = 0;
    while (qn && !rc) {
        cluster_t cl = q[head];
        head = (head + 1) % cap;
        --qn;
        size_t live = qn + nleaves + 1;
        if (live >= target || cl.len < 2) {
            leaves[nleaves++] = cl;
            continue;
        }
        size_t k = (size_t)branching < cl.len ? (size_t)branching : cl.len;
        for (size_t i = 0; i < cl.len; ++i) memcpy(sub + i * d, pts + (size_t)cl.idx[i] * d, d * sizeof(double));
        rc = lloyd(sub, cl.len, d, k, iters, mix64(seed ^ ++splits), ctr, a);
        if (rc) {
            free(cl.idx);
            break;
        }
        memset(cnt, 0, k * sizeof(size_t));
        for (size_t i = 0; i < cl.len; ++i) ++cnt[a[i]];
        for (size_t c = 0; c < k; ++c) {
            if (!cnt[c]) continue;
            cluster_t ch = {xmalloc(cnt[c] * sizeof(uint32_t)), 0};
            for (size_t i = 0; i < cl.len; ++i)
                if (a[i] == c) ch.idx[ch.len++] = cl.idx[i];
            q[tail] = ch;
            tail = (tail + 1) % cap;
            ++qn;
        }
        free(cl.idx);
    }
    for (size_t l = 0; l < nleaves; ++l) {
        for (size_t i = 0; i < leaves[l].len; ++i) assign[leaves[l].idx[i]] = (uint32_t)l;
        free(leaves[l].idx);
    }
    while (qn) {
        free(q[head].idx);
        head = (head + 1) % cap;
        --qn;
    }
    free(q);
    free(leaves);
    free(sub);
    free(ctr);
    free(a);
    free(cnt);
    return rc;
}

/* lsh_neighbor_pairs (lsh.cpp:245-283) up to the per-band composite ids of
 * X_p ∪ X_q (p first): scheme 0 = hash_cross_polytope (lsh.cpp:73-103) with
 * proj drawn row-major from normal_distribution over mt19937_64(fn_seed);
 * 1 = hash_kmeans = lloyd; 2 = hierarchical_assign; ids = ids * b + bucket
 * over the rows_per_band functions. */
int orc_lsh_buckets(const double* p, size_t n, const double* q, size_t m, size_t d, int scheme, int bands, int rows,
                    int buckets, int iters, int branching, uint64_t seed, uint64_t* ids) {
    if (bands < 1 || rows < 1) return fail(E_ARG, "lsh: bands and rows_per_band must be >= 1");
    if (buckets < 2) return fail(E_ARG, "lsh: buckets_per_fn must be >= 2");
    size_t N = n + m;
    if (scheme == 0) {
        if (buckets % 2) return fail(E_ARG, "cross-polytope needs an even bucket count");
    } else if ((size_t)buckets > N) {
        return fail(E_ARG, "hash_kmeans: more buckets than points");
    }
    double* all = xmalloc((N ? N : 1) * d * sizeof(double));
    memcpy(all, p, n * d * sizeof(double));
    memcpy(all + n * d, q, m * d * sizeof(double));
    uint32_t* a = xmalloc((N ? N : 1) * sizeof(uint32_t));
    double* ctr = xmalloc((size_t)buckets * (d ? d : 1) * sizeof(double));
    size_t half = (size_t)buckets / 2;
    double* proj = xmalloc((d ? d : 1) * half * sizeof(double));
    memset(ids, 0, (size_t)bands * N * sizeof(uint64_t));
    int rc = 0;
    for (int b = 0; b < bands && !rc; ++b)
        for (int fn = 0; fn < rows && !rc; ++fn) {
            uint64_t s = fn_seed(seed, b, fn);
            if (scheme == 0) {
                gauss_t g;
                mt64_seed(&g.g, s);
                g.saved_ok = 0;
                for (size_t e = 0; e < d * half; ++e) proj[e] = gauss_next(&g);
                for (size_t i = 0; i < N; ++i) a[i] = cp_bucket(all + i * d, d, proj, half);
            } else if (scheme == 2) {
                rc = hierarchical_assign(all, N, d, (size_t)buckets, branching, iters, s, a);
            } else {
                rc = lloyd(all, N, d, (size_t)buckets, iters, s, ctr, a);
            }
            for (size_t i = 0; i < N && !rc; ++i) ids[(size_t)b * N + i] = ids[(size_t)b * N + i] * buckets + a[i];
        }
    free(all);
    free(a);
    free(ctr);
    free(proj);
    return rc;
}

int orc_lsh_pairs(const double* p, size_t n, const double* q, size_t m, size_t d, int bands, int buckets, int iters,
                  uint64_t seed, void** out) {
    size_t N = n + m;
    uint64_t* ids = xmalloc((size_t)bands * N * sizeof(uint64_t));
    int rc = orc_lsh_kmeans_buckets(p, n, q, m, d, bands, buckets, iters, seed, ids);
    if (!rc) {
        uint64_t* ip = xmalloc((size_t)bands * n * sizeof(uint64_t));
        uint64_t* iq = xmalloc((size_t)bands * m * sizeof(uint64_t));
        for (int b = 0; b < bands; ++b) {
            memcpy(ip + (size_t)b * n, ids + (size_t)b * N, n * sizeof(uint64_t));
            memcpy(iq + (size_t)b * m, ids + (size_t)b * N + n, m * sizeof(uint64_t));
        }
        rc = neighbor_pairs(ip, n, iq, m, bands, (pairs_t**)out);
        free(ip);
        free(iq);
    }
    free(ids);
    return rc;
}

int orc_pairs_from_buckets(const uint64_t* ids_p, size_t n, const uint64_t* ids_q, size_t m, int bands,
                           uint64_t range, void** out) {
    (void)range;
    return neighbor_pairs(ids_p, n, ids_q, m, bands, (pairs_t**)out);
}

int orc_pairs_from_arrays(size_t n, size_t m, const uint32_t* rows, const uint32_t* cols, size_t count, void** out) {
    uint64_t* keys = xmalloc(count * sizeof(uint64_t));
    for (size_t e = 0; e < count; ++e) keys[e] = ((uint64_t)rows[e] << 32) | cols[e];
    int rc = pairs_from_keys(n, m, keys, count, (pairs_t**)out);
    free(keys);
    return rc;
}
size_t orc_pairs_nnz(void* h) { return ((pairs_t*)h)->nnz; }
void orc_pairs_copy(void* h, uint32_t* rows, uint32_t* cols) {
    pairs_t* p = h;
    memcpy(rows, p->row, p->nnz * sizeof(uint32_t));
    memcpy(cols, p->col, p->nnz * sizeof(uint32_t));
}
void orc_pairs_free(void* h) {
    pairs_t* p = h;
    if (!p) return;
    free(p->row);
    free(p->col);
    free(p);
}

/* ---- cost (geometry.cpp:45-76, + squared L2 kind 3) ----------------------- */
static int cost_value(int kind, const double* x, const double* y, size_t d, double* out) {
    if (kind == 0 || kind == 3) {
        double s = 0.0;
        for (size_t k = 0; k < d; ++k) {
            double diff = x[k] - y[k];
            s += diff * diff;
        }
        *out = kind == 0 ? sqrt(s) : s;
        return 0;
    }
    if (kind == 1) {
        double s = 0.0;
        for (size_t k = 0; k < d; ++k) s += x[k] * y[k];
        *out = -s;
        return 0;
    }
    if (kind == 2) {
        double dot = 0.0, nx = 0.0, ny = 0.0;
        for (size_t k = 0; k < d; ++k) {
            dot += x[k] * y[k];
            nx += x[k] * x[k];
            ny += y[k] * y[k];
        }
        if (nx == 0.0 || ny == 0.0) return fail(E_ARG, "cosine-derived cost undefined for zero vectors");
        double c = dot / sqrt(nx * ny);
        if (c > 1.0) c = 1.0;
        if (c < -1.0) c = -1.0;
        *out = sqrt(1.0 - c);
        return 0;
    }
    return fail(E_ARG, "unknown cost kind");
}

/* ---- operator state -------------------------------------------------------- */
enum { K_DENSE = 0, K_SPARSE = 1, K_NYS = 2, K_LCN = 3 };

typedef struct {
    size_t n, m, nnz;
    uint32_t *row_ptr, *col, *col_ptr, *row_idx, *perm;
    double* vals;   /* sparse: log K; lcn: delta */
    double* log_sp; /* lcn */
    double* nys;    /* lcn */
} csr_t;

typedef struct {
    int kind;
    size_t n, m, l, d;
    double lambda;
    double* logk; /* dense n x m */
    csr_t s;
    double *u, *w, *lm; /* n x l, l x m, l x d */
    double max_abs_delta, cond;
} op_t;

/* build_csc_arrays (sparse_kernel.cpp:17-35) */
static void build_csc(csr_t* s) {
    s->col_ptr = xcalloc(s->m + 1, sizeof(uint32_t));
    s->row_idx = xmalloc(s->nnz * sizeof(uint32_t));
    s->perm = xmalloc(s->nnz * sizeof(uint32_t));
    for (size_t e = 0; e < s->nnz; ++e) ++s->col_ptr[s->col[e] + 1];
    for (size_t j = 0; j < s->m; ++j) s->col_ptr[j + 1] += s->col_ptr[j];
    uint32_t* cur = xmalloc((s->m + 1) * sizeof(uint32_t));
    memcpy(cur, s->col_ptr, (s->m + 1) * sizeof(uint32_t));
    for (size_t i = 0; i < s->n; ++i)
        for (uint32_t e = s->row_ptr[i]; e < s->row_ptr[i + 1]; ++e) {
            uint32_t pos = cur[s->col[e]]++;
            s->row_idx[pos] = (uint32_t)i;
            s->perm[pos] = e;
        }
    free(cur);
}

/* build_sparse (sparse_kernel.cpp:51-80) */
static int build_sparse(const double* p, size_t n, const double* q, size_t m, size_t d, const pairs_t* pr, int kind,
                        double lambda, csr_t* s) {
    if (!(lambda > 0.0)) return fail(E_ARG, "build_sparse: lambda must be positive");
    if (pr->n != n || pr->m != m) return fail(E_DIM, "build_sparse: pattern shape mismatch");
    memset(s, 0, sizeof *s);
    s->n = n;
    s->m = m;
    s->nnz = pr->nnz;
    s->row_ptr = xcalloc(n + 1, sizeof(uint32_t));
    for (size_t e = 0; e < pr->nnz; ++e) ++s->row_ptr[pr->row[e] + 1];
    for (size_t i = 0; i < n; ++i) s->row_ptr[i + 1] += s->row_ptr[i];
    s->col = xmalloc(pr->nnz * sizeof(uint32_t));
    s->vals = xmalloc(pr->nnz * sizeof(double));
    memcpy(s->col, pr->col, pr->nnz * sizeof(uint32_t));
    const double inv = 1.0 / lambda;
    for (size_t i = 0; i < n; ++i)
        for (uint32_t e = s->row_ptr[i]; e < s->row_ptr[i + 1]; ++e) {
            double c;
            TRY(cost_value(kind, p + i * d, q + (size_t)s->col[e] * d, d, &c));
            s->vals[e] = 0.0 - c * inv;
        }
    build_csc(s);
    return 0;
}

static void free_csr(csr_t* s) {
    free(s->row_ptr);
    free(s->col);
    free(s->col_ptr);
    free(s->row_idx);
    free(s->perm);
    free(s->vals);
    free(s->log_sp);
    free(s->nys);
}

/* ---- Nystrom (nystrom.cpp:28-196) ------------------------------------------ */
typedef long double LD;

/* Diagonal-pivoted LDL^T in long double (Eigen::LDLT<long double>,
 * nystrom.cpp:108): pivot = largest remaining diagonal, zero pivots zeroed
 * in the solve. */
typedef struct {
    size_t l;
    LD* f;
    size_t* perm;
    int ok;
} ldlt_t;

static void ldlt_factor(ldlt_t* F, const LD* a, size_t l) {
    F->l = l;
    F->ok = 1;
    F->f = xmalloc(l * l * sizeof(LD));
    F->perm = xmalloc(l * sizeof(size_t));
    memcpy(F->f, a, l * l * sizeof(LD));
    LD* f = F->f;
    for (size_t i = 0; i < l; ++i) F->perm[i] = i;
    LD* w = xmalloc(l * sizeof(LD));
    for (size_t k = 0; k < l; ++k) {
        size_t piv = k;
        LD best = fabsl(f[k * l + k]);
        for (size_t i = k + 1; i < l; ++i)
            if (fabsl(f[i * l + i]) > best) {
                best = fabsl(f[i * l + i]);
                piv = i;
            }
        if (piv != k) {
            for (size_t c = 0; c < l; ++c) {
                LD t = f[k * l + c];
                f[k * l + c] = f[piv * l + c];
                f[piv * l + c] = t;
            }
            for (size_t r = 0; r < l; ++r) {
                LD t = f[r * l + k];
                f[r * l + k] = f[r * l + piv];
                f[r * l + piv] = t;
            }
            size_t t = F->perm[k];
            F->perm[k] = F->perm[piv];
            F->perm[piv] = t;
        }
        for (size_t j = 0; j < k; ++j) w[j] = f[j * l + j] * f[k * l + j];
        LD dk = f[k * l + k];
        for (size_t j = 0; j < k; ++j) dk -= f[k * l + j] * w[j];
        f[k * l + k] = dk;
        for (size_t i = k + 1; i < l; ++i) {
            LD v = f[i * l + k];
            for (size_t j = 0; j < k; ++j) v -= f[i * l + j] * w[j];
            f[i * l + k] = v;
        }
        if (fabsl(dk) > 0) {
            for (size_t i = k + 1; i < l; ++i) f[i * l + k] /= dk;
        } else {
            for (size_t i = k + 1; i < l; ++i)
                if (f[i * l + k] != 0) F->ok = 0;
        }
    }
    free(w);
}

static void ldlt_solve(const ldlt_t* F, LD* b) {
    size_t l = F->l;
    const LD* f = F->f;
    LD* y = xmalloc(l * sizeof(LD));
    for (size_t k = 0; k < l; ++k) y[k] = b[F->perm[k]];
    for (size_t i = 0; i < l; ++i)
        for (size_t j = 0; j < i; ++j) y[i] -= f[i * l + j] * y[j];
    for (size_t i = 0; i < l; ++i) y[i] = fabsl(f[i * l + i]) > LDBL_MIN ? y[i] / f[i * l + i] : 0;
    for (size_t ii = l; ii-- > 0;)
        for (size_t j = ii + 1; j < l; ++j) y[ii] -= f[j * l + ii] * y[j];
    for (size_t k = 0; k < l; ++k) b[F->perm[k]] = y[k];
    free(y);
}

/* select_landmarks (nystrom.cpp:28-48) */
static int select_landmarks(const double* p, size_t n, const double* q, size_t m, size_t d, size_t l, int method,
                            uint64_t seed, double* lm) {
    size_t N = n + m;
    if (l < 1 || l > N) return fail(E_ARG, "select_landmarks: l out of range");
    double* all = xmalloc(N * d * sizeof(double));
    memcpy(all, p, n * d * sizeof(double));
    memcpy(all + n * d, q, m * d * sizeof(double));
    int rc;
    if (method == 0) {
        uint32_t* a = xmalloc(N * sizeof(uint32_t));
        rc = lloyd(all, N, d, l, 10, seed, lm, a);
        free(a);
    } else {
        mt64 g;
        mt64_seed(&g, seed);
        uint32_t* rows = xmalloc(l * sizeof(uint32_t));
        rc = kmeans_pp(all, N, d, l, &g, rows);
        for (size_t a = 0; a < l && !rc; ++a) memcpy(lm + a * d, all + (size_t)rows[a] * d, d * sizeof(double));
        free(rows);
    }
    free(all);
    return rc;
}

/* kernel_block (nystrom.cpp:53-64): exp(-c * (1/lambda)) */
static int kernel_block(const double* x, size_t nx, const double* z, size_t nz, size_t d, int kind, double lambda,
                        double* out) {
    const double inv = 1.0 / lambda;
    for (size_t i = 0; i < nx; ++i)
        for (size_t j = 0; j < nz; ++j) {
            double c;
            TRY(cost_value(kind, x + i * d, z + j * d, d, &c));
            out[i * nz + j] = exp(-c * inv);
        }
    return 0;
}

/* build_factors (nystrom.cpp:68-125) */
static int build_factors(const double* p, size_t n, const double* q, size_t m, size_t d, const double* lm, size_t l,
                         int kind, double lambda, op_t* op) {
    if (!(lambda > 0.0)) return fail(E_ARG, "build_factors: lambda must be positive");
    op->u = xmalloc(n * l * sizeof(double));
    double* v = xmalloc(l * m * sizeof(double));
    TRY(kernel_block(p, n, lm, l, d, kind, lambda, op->u));
    TRY(kernel_block(lm, l, q, m, d, kind, lambda, v));
    LD* a = xmalloc(l * l * sizeof(LD));
    for (size_t i = 0; i < l; ++i)
        for (size_t j = 0; j < l; ++j) {
            double c;
            TRY(cost_value(kind, lm + i * d, lm + j * d, d, &c));
            a[i * l + j] = (LD)exp(-c / lambda);
        }
    LD trace = 0.0L;
    for (size_t i = 0; i < l; ++i) trace += a[i * l + i];
    const LD jitter_unit = trace / (LD)l;
    LD v_scale = 0.0L;
    for (size_t e = 0; e < l * m; ++e)
        if (fabsl((LD)v[e]) > v_scale) v_scale = fabsl((LD)v[e]);
    if (v_scale < 1e-300L) v_scale = 1e-300L;
    LD* aj = xmalloc(l * l * sizeof(LD));
    LD* wx = xmalloc(l * m * sizeof(LD));
    LD* col = xmalloc(l * sizeof(LD));
    int done = 0;
    for (double rel = 0.0; rel <= 1.1e-4 && !done; rel = (rel == 0.0 ? 1e-10 : rel * 10.0)) {
        memcpy(aj, a, l * l * sizeof(LD));
        for (size_t i = 0; i < l; ++i) aj[i * l + i] += rel * jitter_unit;
        ldlt_t F;
        ldlt_factor(&F, aj, l);
        if (F.ok) {
            int finite = 1;
            for (size_t j = 0; j < m; ++j) {
                for (size_t r = 0; r < l; ++r) col[r] = (LD)v[r * m + j];
                ldlt_solve(&F, col);
                for (size_t r = 0; r < l; ++r) {
                    wx[r * m + j] = col[r];
                    if (!isfinite(col[r])) finite = 0;
                }
            }
            if (finite) {
                LD resid = 0.0L;
                for (size_t r = 0; r < l; ++r)
                    for (size_t j = 0; j < m; ++j) {
                        LD acc = 0.0L;
                        for (size_t c = 0; c < l; ++c) acc += aj[r * l + c] * wx[c * m + j];
                        LD e = fabsl(acc - (LD)v[r * m + j]);
                        if (e > resid) resid = e;
                    }
                if (!(resid > 1e-6L * v_scale)) {
                    op->w = xmalloc(l * m * sizeof(double));
                    for (size_t e = 0; e < l * m; ++e) op->w[e] = (double)wx[e];
                    LD na = 0.0L, ni = 0.0L;
                    LD* ecol = xmalloc(l * sizeof(LD));
                    for (size_t c = 0; c < l; ++c) {
                        LD s = 0.0L;
                        for (size_t r = 0; r < l; ++r) s += fabsl(aj[r * l + c]);
                        if (s > na) na = s;
                        memset(ecol, 0, l * sizeof(LD));
                        ecol[c] = 1.0L;
                        ldlt_solve(&F, ecol);
                        s = 0.0L;
                        for (size_t r = 0; r < l; ++r) s += fabsl(ecol[r]);
                        if (s > ni) ni = s;
                    }
                    free(ecol);
                    LD cond = na * ni;
                    op->cond = isfinite(cond) && cond > 0 ? (double)cond : INFINITY;
                    done = 1;
                }
            }
        }
        free(F.f);
        free(F.perm);
    }
    free(a);
    free(aj);
    free(wx);
    free(col);
    free(v);
    if (!done) return fail(E_FACT, "build_factors: landmark kernel matrix numerically singular beyond jitter budget");
    return 0;
}

/* NystromFactors::entry (nystrom.cpp:127-132) */
static double nys_entry(const op_t* op, size_t i, size_t j) {
    double s = 0.0;
    for (size_t a = 0; a < op->l; ++a) s += op->u[i * op->l + a] * op->w[a * op->m + j];
    return s;
}

/* build_correction (sparse_kernel.cpp:82-117) */
static int build_correction(op_t* op) {
    csr_t* c = &op->s;
    c->log_sp = c->vals;
    c->vals = xmalloc(c->nnz * sizeof(double));
    c->nys = xcalloc(c->nnz, sizeof(double));
    double max_abs = 0.0;
    int overflow = 0;
    for (size_t i = 0; i < c->n; ++i)
        for (uint32_t e = c->row_ptr[i]; e < c->row_ptr[i + 1]; ++e) {
            double exact = exp(c->log_sp[e]);
            c->vals[e] = 0.0;
            if (isinf(exact)) {
                overflow = 1;
                continue;
            }
            double nys = nys_entry(op, i, c->col[e]);
            c->nys[e] = nys;
            c->vals[e] = exact - nys;
            if (fabs(c->vals[e]) > max_abs) max_abs = fabs(c->vals[e]);
        }
    if (overflow) return fail(E_STAB, "build_correction: kernel value overflows linear space");
    op->max_abs_delta = max_abs;
    return 0;
}

/* ---- operator products (operator.cpp:123-224, sparse_kernel.cpp:119-185,
 *      nystrom.cpp:134-194) ------------------------------------------------ */
static const char* kind_name(int k) {
    return k == K_DENSE ? "dense" : k == K_SPARSE ? "sparse" : k == K_NYS ? "nystrom" : "lcn";
}

/* nys_matvec / nys_matvec_t (nystrom.cpp:134-194): 1 on a nonpositive output
 * for a strictly positive input. */
static int nys_matvec(const op_t* op, const double* t, int transposed, double* out) {
    const size_t n = op->n, m = op->m, l = op->l;
    const size_t lin = transposed ? n : m, lout = transposed ? m : n;
    int positive = 1;
    for (size_t j = 0; j < lin; ++j)
        if (!(t[j] > 0.0)) positive = 0;
    double* mid = xcalloc(l, sizeof(double));
    if (!transposed) {
        for (size_t a = 0; a < l; ++a) {
            double s = 0.0;
            for (size_t j = 0; j < m; ++j) s += op->w[a * m + j] * t[j];
            mid[a] = s;
        }
        for (size_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (size_t a = 0; a < l; ++a) s += op->u[i * l + a] * mid[a];
            out[i] = s;
        }
    } else {
        for (size_t a = 0; a < l; ++a) {
            double acc = 0.0;
            for (size_t i = 0; i < n; ++i) acc += op->u[i * l + a] * t[i];
            mid[a] = acc;
        }
        for (size_t j = 0; j < m; ++j) {
            double acc = 0.0;
            for (size_t a = 0; a < l; ++a) acc += op->w[a * m + j] * mid[a];
            out[j] = acc;
        }
    }
    free(mid);
    if (positive)
        for (size_t i = 0; i < lout; ++i)
            if (!(out[i] > 0.0)) return 1;
    return 0;
}

/* KernelOperator::base_log_matvec(_t) (operator.cpp:123-224) */
static int op_log_matvec(const op_t* op, const double* in, int transposed, double* out) {
    const size_t n = op->n, m = op->m;
    const size_t lin = transposed ? n : m, lout = transposed ? m : n;
    if (op->kind == K_DENSE) {
        for (size_t r = 0; r < lout; ++r) {
            double hi = -INFINITY;
            for (size_t c = 0; c < lin; ++c) {
                double v = (transposed ? op->logk[c * m + r] : op->logk[r * m + c]) + in[c];
                if (v > hi) hi = v;
            }
            if (hi == -INFINITY) {
                out[r] = -INFINITY;
                continue;
            }
            double acc = 0.0;
            for (size_t c = 0; c < lin; ++c)
                acc += exp((transposed ? op->logk[c * m + r] : op->logk[r * m + c]) + in[c] - hi);
            out[r] = hi + log(acc);
        }
        return 0;
    }
    if (op->kind == K_SPARSE) {
        const csr_t* s = &op->s;
        for (size_t r = 0; r < lout; ++r) {
            uint32_t b = transposed ? s->col_ptr[r] : s->row_ptr[r];
            uint32_t e1 = transposed ? s->col_ptr[r + 1] : s->row_ptr[r + 1];
            double hi = -INFINITY;
            for (uint32_t e = b; e < e1; ++e) {
                double v = transposed ? s->vals[s->perm[e]] + in[s->row_idx[e]] : s->vals[e] + in[s->col[e]];
                if (v > hi) hi = v;
            }
            if (hi == -INFINITY) {
                out[r] = -INFINITY;
                continue;
            }
            double acc = 0.0;
            for (uint32_t e = b; e < e1; ++e)
                acc += exp((transposed ? s->vals[s->perm[e]] + in[s->row_idx[e]] : s->vals[e] + in[s->col[e]]) - hi);
            out[r] = hi + log(acc);
        }
        return 0;
    }
    double hi = -INFINITY;
    for (size_t j = 0; j < lin; ++j)
        if (in[j] > hi) hi = in[j];
    if (hi == -INFINITY) {
        for (size_t i = 0; i < lout; ++i) out[i] = -INFINITY;
        return 0;
    }
    double* tt = xmalloc(lin * sizeof(double));
    double* y = xmalloc(lout * sizeof(double));
    for (size_t j = 0; j < lin; ++j) tt[j] = exp(in[j] - hi);
    int bad = nys_matvec(op, tt, transposed, y);
    if (!bad && op->kind == K_LCN) {
        const csr_t* c = &op->s;
        for (size_t r = 0; r < lout; ++r) {
            double acc = 0.0;
            if (!transposed)
                for (uint32_t e = c->row_ptr[r]; e < c->row_ptr[r + 1]; ++e) acc += c->vals[e] * tt[c->col[e]];
            else
                for (uint32_t e = c->col_ptr[r]; e < c->col_ptr[r + 1]; ++e) acc += c->vals[c->perm[e]] * tt[c->row_idx[e]];
            y[r] += acc;
        }
    }
    for (size_t i = 0; i < lout && !bad; ++i) {
        if (!(y[i] > 0.0)) bad = 1;
        else out[i] = hi + log(y[i]);
    }
    free(tt);
    free(y);
    if (bad)
        return fail(E_NEG, "%s %s produced a nonpositive entry", kind_name(op->kind),
                    transposed ? "transposed matvec" : "matvec");
    return 0;
}

/* ---- operators ------------------------------------------------------------- */
int orc_op_sparse(const double* p, size_t n, const double* q, size_t m, size_t d, int kind, double lambda,
                  void* pairs, void** out) {
    if (!(lambda > 0.0)) return fail(E_ARG, "build_sparse: lambda must be positive");
    op_t* op = xcalloc(1, sizeof(op_t));
    op->kind = K_SPARSE;
    op->n = n;
    op->m = m;
    op->d = d;
    op->lambda = lambda;
    int rc = build_sparse(p, n, q, m, d, pairs, kind, lambda, &op->s);
    if (rc) {
        orc_op_free(op);
        return rc;
    }
    *out = op;
    return 0;
}

int orc_op_lcn(const double* p, size_t n, const double* q, size_t m, size_t d, int kind, double lambda, void* pairs,
               size_t l, int method, uint64_t lm_seed, const double* landmarks, int nystrom_only, void** out,
               double* phase_ms) {
    (void)phase_ms;
    op_t* op = xcalloc(1, sizeof(op_t));
    op->kind = nystrom_only ? K_NYS : K_LCN;
    op->n = n;
    op->m = m;
    op->d = d;
    op->l = l;
    op->lambda = lambda;
    op->lm = xmalloc(l * d * sizeof(double));
    int rc = 0;
    if (landmarks) memcpy(op->lm, landmarks, l * d * sizeof(double));
    else rc = select_landmarks(p, n, q, m, d, l, method, lm_seed, op->lm);
    if (!rc) rc = build_factors(p, n, q, m, d, op->lm, l, kind, lambda, op);
    if (!rc && !nystrom_only) {
        rc = build_sparse(p, n, q, m, d, pairs, kind, lambda, &op->s);
        if (!rc) rc = build_correction(op);
    }
    if (rc) {
        orc_op_free(op);
        return rc;
    }
    *out = op;
    return 0;
}

/* build_cost + build_kernel (geometry.cpp:113-144) */
int orc_op_dense(const double* p, size_t n, const double* q, size_t m, size_t d, int kind, double lambda, void** out) {
    if (!(lambda > 0.0)) return fail(E_ARG, "build_cost: lambda must be positive");
    op_t* op = xcalloc(1, sizeof(op_t));
    op->kind = K_DENSE;
    op->n = n;
    op->m = m;
    op->d = d;
    op->lambda = lambda;
    op->logk = xmalloc(n * m * sizeof(double));
    const double inv = 1.0 / lambda;
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < m; ++j) {
            double c;
            int rc = cost_value(kind, p + i * d, q + j * d, d, &c);
            if (rc) {
                orc_op_free(op);
                return rc;
            }
            op->logk[i * m + j] = isinf(c) ? -INFINITY : 0.0 - c * inv;
        }
    *out = op;
    return 0;
}

void orc_op_free(void* h) {
    op_t* op = h;
    if (!op) return;
    free_csr(&op->s);
    free(op->logk);
    free(op->u);
    free(op->w);
    free(op->lm);
    free(op);
}
size_t orc_op_nnz(void* h) { return ((op_t*)h)->s.nnz; }
size_t orc_op_rank(void* h) { return ((op_t*)h)->l; }
double orc_op_scalar(void* h, int which) {
    op_t* op = h;
    return which == 0 ? op->max_abs_delta : which == 1 ? op->cond : 0.0;
}

int orc_op_copy(void* h, int which, uint32_t* row_ptr, uint32_t* col, double* vals) {
    op_t* op = h;
    const csr_t* s = &op->s;
    if (which == 0 || which == 1 || which == 5 || which == 6) {
        if (!s->row_ptr) return fail(E_ARG, "orc_op_copy: nothing to copy");
        if (row_ptr) memcpy(row_ptr, s->row_ptr, (s->n + 1) * sizeof(uint32_t));
        if (col) memcpy(col, s->col, s->nnz * sizeof(uint32_t));
        const double* src = which == 0 ? (op->kind == K_LCN ? s->log_sp : s->vals)
                            : which == 1 ? s->vals
                            : which == 5 ? s->nys
                                         : s->log_sp;
        if (vals && src) memcpy(vals, src, s->nnz * sizeof(double));
        return 0;
    }
    if (which == 2 && op->u) {
        memcpy(vals, op->u, op->n * op->l * sizeof(double));
        return 0;
    }
    if (which == 3 && op->w) {
        memcpy(vals, op->w, op->l * op->m * sizeof(double));
        return 0;
    }
    if (which == 4 && op->lm) {
        memcpy(vals, op->lm, op->l * op->d * sizeof(double));
        return 0;
    }
    return fail(E_ARG, "orc_op_copy: nothing to copy");
}

int orc_op_log_matvec(void* h, const double* in, size_t len, int transposed, double* out) {
    op_t* op = h;
    if (len != (transposed ? op->n : op->m))
        return fail(E_DIM, transposed ? "log_matvec_t: vector length mismatch" : "log_matvec: vector length mismatch");
    return op_log_matvec(op, in, transposed, out);
}

/* ---- support check (sparse_kernel.cpp:189-244 via matching.cpp:12-92):
 *      maximum bipartite matching by augmenting paths ----------------------- */
static size_t max_matching(size_t n, size_t m, const uint32_t* row_ptr, const uint32_t* col) {
    uint32_t* mate_r = xmalloc((m ? m : 1) * sizeof(uint32_t));
    uint32_t* mate_l = xmalloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t* seen = xcalloc(m ? m : 1, sizeof(uint32_t));
    uint32_t* stack_u = xmalloc((n + 1) * sizeof(uint32_t));
    uint32_t* stack_e = xmalloc((n + 1) * sizeof(uint32_t));
    for (size_t j = 0; j < m; ++j) mate_r[j] = UINT32_MAX;
    for (size_t i = 0; i < n; ++i) mate_l[i] = UINT32_MAX;
    size_t matched = 0;
    uint32_t stamp = 0;
    for (size_t root = 0; root < n; ++root) {
        ++stamp;
        size_t sp = 0;
        stack_u[0] = (uint32_t)root;
        stack_e[0] = row_ptr[root];
        int found = 0;
        while (sp < n + 1 && !found) {
            uint32_t u = stack_u[sp];
            if (stack_e[sp] == row_ptr[u + 1]) {
                if (sp == 0) break;
                --sp;
                continue;
            }
            uint32_t v = col[stack_e[sp]++];
            if (seen[v] == stamp) continue;
            seen[v] = stamp;
            if (mate_r[v] == UINT32_MAX) {
                /* augment along the stack */
                for (size_t k = sp + 1; k-- > 0;) {
                    uint32_t x = stack_u[k];
                    uint32_t prev = mate_l[x];
                    mate_l[x] = v;
                    mate_r[v] = x;
                    v = prev;
                }
                found = 1;
            } else {
                ++sp;
                stack_u[sp] = mate_r[v];
                stack_e[sp] = row_ptr[mate_r[v]];
            }
        }
        if (found) ++matched;
    }
    free(mate_r);
    free(mate_l);
    free(seen);
    free(stack_u);
    free(stack_e);
    return matched;
}

/* ---- sinkhorn (sinkhorn.cpp:104-188) ------------------------------------- */
typedef struct {
    double distance, err_final;
    int iters, converged, warnings;
    size_t n, m, nnz;
    double *log_s, *log_t, *row_marg, *trace, *plan_vals, *sp_vals, *sp_nys_vals;
    int n_trace;
} res_t;

static int check_finite(const double* v, size_t n, int kind, const char* which) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(v[i]))
            return fail(E_STAB, "sinkhorn: non-finite scaling (%s) under the %s operator", which, kind_name(kind));
    return 0;
}

int orc_sinkhorn(void* h, const double* pm, size_t n, const double* qm, size_t m, double tol, int max_iters,
                 int check_support, int want_plan, void** out) {
    op_t* op = h;
    /* Marginals::validate(balanced) (geometry.cpp:97-111) */
    if (!n || !m) return fail(E_ARG, "marginals must be non-empty");
    double sp = 0.0, sq = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (!(pm[i] > 0.0) || !isfinite(pm[i])) return fail(E_ARG, "marginal p has a non-positive or non-finite entry");
    }
    for (size_t j = 0; j < m; ++j) {
        if (!(qm[j] > 0.0) || !isfinite(qm[j])) return fail(E_ARG, "marginal q has a non-positive or non-finite entry");
    }
    for (size_t i = 0; i < n; ++i) sp += pm[i];
    for (size_t j = 0; j < m; ++j) sq += qm[j];
    if (fabs(sp - sq) > 1e-12 * (sp > sq ? sp : sq))
        return fail(E_ARG, "marginals are unbalanced; balanced OT requires equal mass");
    if (n != op->n || m != op->m) return fail(E_DIM, "sinkhorn: marginal length does not match operator shape");
    if (max_iters < 1) return fail(E_ARG, "sinkhorn: max_iters must be >= 1");
    res_t* r = xcalloc(1, sizeof(res_t));
    r->n = n;
    r->m = m;
    if (op->kind == K_SPARSE && check_support) {
        size_t small = n < m ? n : m;
        if (op->s.nnz == 0 || max_matching(n, m, op->s.row_ptr, op->s.col) < small) {
            r->warnings = 1;
            fprintf(stderr, "lcn: warning: sparse kernel pattern has no support; Sinkhorn may not converge\n");
        }
    }
    double mass = 0.0;
    for (size_t i = 0; i < n; ++i) mass += pm[i];
    for (size_t j = 0; j < m; ++j) mass += qm[j];
    if (tol < 0.0) tol = 1e-6 * mass;
    double* log_p = xmalloc(n * sizeof(double));
    double* log_q = xmalloc(m * sizeof(double));
    for (size_t i = 0; i < n; ++i) log_p[i] = log(pm[i]);
    for (size_t j = 0; j < m; ++j) log_q[j] = log(qm[j]);
    r->log_s = xcalloc(n, sizeof(double));
    r->log_t = xcalloc(m, sizeof(double));
    r->row_marg = xcalloc(n, sizeof(double));
    r->trace = xcalloc((size_t)max_iters, sizeof(double));
    double* kt = xmalloc(n * sizeof(double));
    double* kts = xmalloc(m * sizeof(double));
    int rc = op_log_matvec(op, r->log_t, 0, kt);
    double err = INFINITY;
    int iter = 0, converged = 0;
    while (!rc && iter < max_iters) {
        ++iter;
        for (size_t i = 0; i < n; ++i) r->log_s[i] = log_p[i] - kt[i];
        if ((rc = check_finite(r->log_s, n, op->kind, "log s"))) break;
        if ((rc = op_log_matvec(op, r->log_s, 1, kts))) break;
        for (size_t j = 0; j < m; ++j) r->log_t[j] = log_q[j] - kts[j];
        if ((rc = check_finite(r->log_t, m, op->kind, "log t"))) break;
        if ((rc = op_log_matvec(op, r->log_t, 0, kt))) break;
        err = 0.0;
        for (size_t i = 0; i < n; ++i) {
            r->row_marg[i] = exp(r->log_s[i] + kt[i]);
            err += fabs(r->row_marg[i] - pm[i]);
        }
        r->trace[r->n_trace++] = err;
        if (err <= tol) {
            converged = 1;
            break;
        }
    }
    free(kt);
    free(kts);
    free(log_p);
    free(log_q);
    if (rc) {
        orc_result_free(r);
        return rc;
    }
    r->iters = iter;
    r->converged = converged;
    r->err_final = err;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) acc += r->log_s[i] * r->row_marg[i];
    for (size_t j = 0; j < m; ++j) acc += r->log_t[j] * qm[j];
    r->distance = op->lambda * acc;
    if (want_plan && (op->kind == K_SPARSE || op->kind == K_LCN)) {
        /* extract_plan_impl (sinkhorn.cpp:45-80) */
        const csr_t* s = &op->s;
        r->nnz = s->nnz;
        if (op->kind == K_SPARSE) {
            r->plan_vals = xmalloc(s->nnz * sizeof(double));
            for (size_t i = 0; i < n; ++i)
                for (uint32_t e = s->row_ptr[i]; e < s->row_ptr[i + 1]; ++e)
                    r->plan_vals[e] = exp(r->log_s[i] + s->vals[e] + r->log_t[s->col[e]]);
        } else {
            r->sp_vals = xmalloc(s->nnz * sizeof(double));
            r->sp_nys_vals = xmalloc(s->nnz * sizeof(double));
            for (size_t i = 0; i < n; ++i) {
                double si = exp(r->log_s[i]);
                for (uint32_t e = s->row_ptr[i]; e < s->row_ptr[i + 1]; ++e) {
                    double tj = exp(r->log_t[s->col[e]]);
                    r->sp_vals[e] = exp(r->log_s[i] + s->log_sp[e] + r->log_t[s->col[e]]);
                    r->sp_nys_vals[e] = si * s->nys[e] * tj;
                }
            }
        }
    }
    *out = r;
    return 0;
}

void orc_result_free(void* h) {
    res_t* r = h;
    if (!r) return;
    free(r->log_s);
    free(r->log_t);
    free(r->row_marg);
    free(r->trace);
    free(r->plan_vals);
    free(r->sp_vals);
    free(r->sp_nys_vals);
    free(r);
}

double orc_result_scalar(void* h, int which) {
    res_t* r = h;
    switch (which) {
        case 0: return r->distance;
        case 1: return r->iters;
        case 2: return r->converged;
        case 3: return r->err_final;
        case 4: return r->warnings;
        case 5: return r->n_trace;
    }
    return 0.0;
}

size_t orc_result_copy(void* h, int which, double* out) {
    res_t* r = h;
    const double* v = NULL;
    size_t len = 0;
    switch (which) {
        case 0: v = r->log_s; len = r->n; break;
        case 1: v = r->log_t; len = r->m; break;
        case 2: v = r->row_marg; len = r->n; break;
        case 3: v = r->trace; len = (size_t)r->n_trace; break;
        case 4: v = r->plan_vals; len = v ? r->nnz : 0; break;
        case 5: v = r->sp_vals; len = v ? r->nnz : 0; break;
        case 6: v = r->sp_nys_vals; len = v ? r->nnz : 0; break;
    }
    if (!v) return 0;
    if (out) memcpy(out, v, len * sizeof(double));
    return len;
}

/* distance_lcn (sinkhorn.cpp:222-261) */
int orc_distance_lcn(void* res, void* h, double* out) {
    res_t* r = res;
    op_t* op = h;
    const size_t n = op->n, m = op->m, l = op->l;
    double* s_lin = xmalloc(n * sizeof(double));
    double* t_lin = xmalloc(m * sizeof(double));
    double* wt = xcalloc(l, sizeof(double));
    double* su = xcalloc(l, sizeof(double));
    for (size_t i = 0; i < n; ++i) s_lin[i] = exp(r->log_s[i]);
    for (size_t j = 0; j < m; ++j) t_lin[j] = exp(r->log_t[j]);
    for (size_t a = 0; a < l; ++a) {
        double acc = 0.0;
        for (size_t j = 0; j < m; ++j) acc += op->w[a * m + j] * t_lin[j];
        wt[a] = acc;
    }
    for (size_t a = 0; a < l; ++a) {
        double acc = 0.0;
        for (size_t i = 0; i < n; ++i) acc += op->u[i * l + a] * s_lin[i];
        su[a] = acc;
    }
    double term = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double row = 0.0;
        for (size_t a = 0; a < l; ++a) row += op->u[i * l + a] * wt[a];
        term += r->log_s[i] * (s_lin[i] * row);
    }
    for (size_t j = 0; j < m; ++j) {
        double c = 0.0;
        for (size_t a = 0; a < l; ++a) c += su[a] * op->w[a * m + j];
        term += r->log_t[j] * (c * t_lin[j]);
    }
    const csr_t* c = &op->s;
    if (c->row_ptr)
        for (size_t i = 0; i < n; ++i)
            for (uint32_t e = c->row_ptr[i]; e < c->row_ptr[i + 1]; ++e) {
                double mass = s_lin[i] * c->vals[e] * t_lin[c->col[e]];
                term += mass * (r->log_s[i] + r->log_t[c->col[e]]);
            }
    free(s_lin);
    free(t_lin);
    free(wt);
    free(su);
    *out = op->lambda * term;
    return 0;
}

/* ref::solve (reference.cpp:41-105): serial linear-space Sinkhorn. */
int orc_dense_reference(const double* cost, size_t n, size_t m, const double* p, const double* q, double lambda,
                        double tol, int max_iters, double* plan, double* distance, int* iters) {
    if (!(lambda > 0.0)) return fail(E_ARG, "reference solve: lambda must be positive");
    double* K = xmalloc(n * m * sizeof(double));
    for (size_t e = 0; e < n * m; ++e) K[e] = exp(-cost[e] / lambda);
    double* s = xmalloc(n * sizeof(double));
    double* t = xmalloc(m * sizeof(double));
    for (size_t i = 0; i < n; ++i) s[i] = 1.0;
    for (size_t j = 0; j < m; ++j) t[j] = 1.0;
    int it_done = 0;
    for (int it = 1; it <= max_iters; ++it) {
        for (size_t i = 0; i < n; ++i) {
            double kt = 0.0;
            for (size_t j = 0; j < m; ++j) kt += K[i * m + j] * t[j];
            s[i] = p[i] / kt;
        }
        for (size_t j = 0; j < m; ++j) {
            double ks = 0.0;
            for (size_t i = 0; i < n; ++i) ks += K[i * m + j] * s[i];
            t[j] = q[j] / ks;
        }
        it_done = it;
        double err = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double row = 0.0;
            for (size_t j = 0; j < m; ++j) row += s[i] * K[i * m + j] * t[j];
            err += fabs(row - p[i]);
        }
        for (size_t j = 0; j < m; ++j) {
            double c = 0.0;
            for (size_t i = 0; i < n; ++i) c += s[i] * K[i * m + j] * t[j];
            err += fabs(c - q[j]);
        }
        if (err <= tol) break;
    }
    double transport = 0.0, entropy = 0.0;
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < m; ++j) {
            double v = s[i] * K[i * m + j] * t[j];
            if (plan) plan[i * m + j] = v;
            if (v <= 0.0) continue;
            transport += v * cost[i * m + j];
            entropy -= v * log(v);
        }
    *distance = transport - lambda * entropy;
    *iters = it_done;
    free(K);
    free(s);
    free(t);
    return 0;
}
