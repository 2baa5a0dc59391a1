// Internal operator / result structures and the build + solve entry points.
#pragma once
#include <functional>

#include <memory>
#include <string>
#include <vector>

#include "ctx.cuh"

namespace lcnb {

constexpr int kMaxBands = 8;

// Device-side descriptor of one band, passed by value to kernels.
struct BandView {
    const uint32_t* src_order;
    const uint32_t* tgt_order;
    const uint32_t* src_start;
    const uint32_t* tgt_start;
    const unsigned long long* blk_off;
    const unsigned long long* blkT_off;
    const uint32_t* src_bucket;
    const uint32_t* tgt_bucket;
    const uint32_t* src_local;
    const uint32_t* tgt_local;
    const uint32_t* src_pos;
    const uint32_t* tgt_pos;
};

struct BandSet {  // bucket ids of every band, for the cross-band dedup mask
    const uint32_t* src_bucket[kMaxBands];
    const uint32_t* tgt_bucket[kMaxBands];
    int bands;
};

// Iteration layout of the band streams (LCN). A panel is one output group of a
// bucket block, stored as ns rows (stream side) x row_stride(ow) entries
// starting at val_off. Stream row r is the bucket's stream position
// r < gap0 ? r : r + gapn (from s_base); output c is o_order[o_base + c].
// Bands after the first skip the pairs an earlier band already holds (the
// support is the union of the bands, lsh.cpp:163-177): inside a bucket both
// sides are ordered by their band-0 bucket, so the pairs of a target group
// that band 0 owns are one contiguous run of sources, left out of the stored
// rows (the gap). Small groups share plain panels that keep those entries as
// zeros. The first band has one plain panel per bucket on the block layout.
struct BandPanel {
    unsigned long long val_off;
    uint32_t bucket, s_base, ns, gap0, gapn, o_base, ow, pad;
};

struct BandIter {
    DevBuf<BandPanel> panels[2];         // [0] row pass (streams targets), [1] column pass (streams sources)
    std::vector<BandPanel> h_panels[2];
    DevBuf<uint32_t> src_order, tgt_order, src_pos, tgt_pos;  // compact bands: (bucket, band-0 bucket, index) order
    const uint32_t *so = nullptr, *to = nullptr, *sp = nullptr, *tp = nullptr;  // orders the kernels use
    bool compact = false;
    unsigned long long entries[2] = {0, 0};  // stored entries per pass (padded)
    unsigned long long real[2] = {0, 0};     // sum ns * ow per pass
};

struct Solver;

// Bucket-sharded LCN operator (plan in shard.h): this rank's
// operator covers its local points -- owned first (rows [0, n_own) /
// [0, m_own)), then halo -- with the band-0 ids of halo points relabelled
// into two one-sided buckets so no band-0 block is built for them.
struct ShardState {
    std::shared_ptr<Comm> comm;  // the context's communicator at build time
    int rank = 0, world = 1;
    size_t n_glob = 0, m_glob = 0;
    uint32_t n_own = 0, m_own = 0;
    unsigned long long nnz_glob = 0;  // support of the whole problem (lazy: ids_src / ids_tgt kept until asked)
    std::vector<uint32_t> ids_src, ids_tgt;  // bands x n, bands x m (host), for nnz_glob
    int bands = 0;
    std::vector<uint32_t> src_glob, tgt_glob;  // local -> global
    DevBuf<uint32_t> d_src_glob, d_tgt_glob;
    // exchange: exported local indices (slot order) and, per halo point, the
    // owner rank and slot; slots padded to max_exp_* on every rank
    DevBuf<uint32_t> exp_s, exp_t, imp_s_rank, imp_s_slot, imp_t_rank, imp_t_slot;
    size_t n_exp_s = 0, n_exp_t = 0, n_halo = 0, m_halo = 0, max_exp_s = 0, max_exp_t = 0;
    // every rank's owned global indices (the final all-gather of the result)
    std::vector<std::vector<uint32_t>> own_src_all, own_tgt_all;
    size_t groups = 0;
    double cost = 0.0;
    // per band, per local bucket: holds an owned source / an owned target
    // (a pass skips the buckets whose outputs are all halo)
    std::vector<std::vector<uint8_t>> rows_need, cols_need;
};

struct Op {
    Ctx* ctx = nullptr;
    int kind = 1;  // lcn_op_kind
    size_t n = 0, m = 0, d = 0, l = 0;
    int cost = 0;
    double lambda = 1.0;
    bool fp64 = false;
    DevBuf<double> X;                     // (n+m) x d union X_p ∪ X_q, fp64 (union_points, geometry.cpp:20-27)
    const double* P() const { return X.get(); }
    const double* Q() const { return X.get() + n * d; }
    DevBuf<float> X32;                    // fp32 copy of X when every coordinate is fp32-exact (k-means reads)
    DevBuf<double> norms;                 // per-point sum x_k^2 (cosine-derived cost only)
    bool landmarks_ready = false;         // L already selected (concurrently with the LSH k-means)
    DevBuf<uint32_t> landmark_init;       // landmark k-means++ indices, seeded with the LSH bands (or empty)
    bool factors_ready = false;           // U, V^T, W already built (concurrently with the LSH k-means)
    std::vector<Band> bands;
    std::vector<DevBuf<double>> val64;    // sparse: log K; lcn: delta (fp64 master)
    std::vector<DevBuf<float>> val32;     // iteration copy (fp32 storage mode)
    // lcn: delta blocks transposed (targets x sources), the row pass's layout
    std::vector<DevBuf<float>> val32T;
    std::vector<DevBuf<double>> val64T;
    std::vector<DevBuf<double>> logk64;   // lcn: log K^sp at stored entries
    std::function<void()> during_ldlt;     // device work overlapped with the host LDL^T (build_nystrom)
    // lcn: iteration layout per band; in fp32 storage the compact bands' val32
    // (column pass) and val32T (row pass) hold their panels instead of blocks
    std::vector<BandIter> iter;
    // dense operator (kind 0, the configs[2] anchor): log K = 0 - c * (1/lambda)
    // n x m row-major (fp64 master) and the iteration copies, plus transposes
    DevBuf<double> dk64, dk64T;
    DevBuf<float> dk32, dk32T;
    DevBuf<double> dc64;  // dense cost c (multi-head: log K per lambda from it)
    // dense kernel recomputed every half-iteration (LCN_DENSE_RECOMPUTE,
    // dense_tc.cu): packed tf32 hi/lo tiles of the union, |x|^2, per
    // (row, column tile) partials; no n x m storage
    bool dense_tc = false;
    int dtc_nta = 0, dtc_ntb = 0;
    DevBuf<unsigned char> dtc_tiles;
    DevBuf<double> dtc_norm, dtc_pm, dtc_ps;
    unsigned long long nnz = 0, stored = 0;
    // Nystrom / LCN
    DevBuf<double> L;                     // l x d landmarks
    DevBuf<double> U64, Wt64;             // n x l, m x l (W transposed)
    DevBuf<float> U32, Wt32;              // iteration copies, rows padded to lp (fp32 mode)
    DevBuf<double> U64p, Wt64p;           // iteration copies, rows padded to lp (fp64 mode)
    size_t lp = 0;
    double max_abs_delta = 0.0, cond = 0.0;
    // CSR export (lazy)
    DevBuf<uint32_t> csr_row_ptr, csr_col;
    bool csr_ready = false;
    // general pattern (KernelOperator::sparse / ::lcn from host structs,
    // operator.hpp:33-36): the support is any CSR, not bucket blocks. Values
    // fp64 in CSR order (log K for sparse, delta for lcn) and CSC order for
    // the column pass; log K^sp of an lcn operator in CSR order.
    bool gcsr = false;
    DevBuf<double> gval, gvalT, glogsp;
    DevBuf<uint32_t> gcp, gri;  // CSC col_ptr (m + 1), row index (nnz)
    std::shared_ptr<Solver> ws;           // persistent iteration workspace (sinkhorn.cu)
    // BP extension (KernelOperator::with_bp, operator.cpp:103-115): log of the
    // deletion kernels c_{p,eps} (n) and c_{eps,q} (m); set in place
    bool bp = false;
    DevBuf<double> bp_ldp, bp_ldq;
    std::shared_ptr<ShardState> shard;    // bucket-sharded operator (null: whole problem)
    size_t n_glob() const { return shard ? shard->n_glob : n; }
    size_t m_glob() const { return shard ? shard->m_glob : m; }

    BandView view(int b) const;
    BandSet bandset() const;
    const char* name() const { return kind == 1 ? "sparse" : kind == 2 ? "nystrom" : kind == 3 ? "lcn" : "dense"; }
    std::string full_name() const { return std::string(name()) + (bp ? "+bp" : ""); }  // KernelOperator::name
};

struct Result {
    double distance = 0.0;
    std::vector<double> del_p_mass, del_q_mass;  // BP plan quadrants (Plan, sinkhorn.hpp:47-51)
    double eps_mass = 0.0;
    int iters = 0;
    bool converged = false;
    double marginal_err_final = 0.0;
    double device_ms = 0.0;
    std::vector<double> phase_ms;  // profiling: col bands, col finalize+reduce, row bands, row finalize+reduce+end
    int phase_iters = 0;
    std::vector<double> log_s, log_t, row_marg, err_trace;
    std::vector<double> plan_vals, sp_vals, sp_nys_vals;
    std::vector<std::string> warnings;
    size_t n = 0, m = 0;
};

// build.cu
void build_band_layout(Ctx& ctx, Band& B, const uint32_t* d_src_bucket, const uint32_t* d_tgt_bucket, size_t n,
                       size_t m, size_t nb);
// LshConfig (lsh.hpp:22-30); scheme uses the LshScheme values (lsh.hpp:13-17).
struct LshParams {
    int scheme = 1;  // 0 cross-polytope, 1 k-means, 2 hierarchical k-means
    int bands = 1, rows = 1, buckets = 2, iters = 10, branching = 2;
    uint64_t seed = 0;
};
// A k-means seeded together with the LSH bands' (same points): its k and
// engine seed, and where its k-means++ indices go (the landmark k-means).
struct ExtraSeeding {
    int k = 0;
    uint64_t seed = 0;
    uint32_t* out = nullptr;
};
void lsh_bucket_ids(Ctx& ctx, const double* d_union, const float* d_union32, size_t n, size_t m, size_t d,
                    const LshParams& cfg, std::vector<DevBuf<uint32_t>>& ids, size_t& range,
                    const std::function<void(Ctx&)>& extra = {}, const ExtraSeeding* extra_seed = nullptr,
                    bool early_extra = false);
void cross_polytope_buckets_device(Ctx& ctx, const double* X, long long N, int d, const double* h_proj, int half,
                                   uint32_t* out);
bool nystrom_inverse_host(const double* A, int l, double rel, double* ainv, double* aj_out);
// batched.cu: configs[4], many small LCN problems in ragged launches
void batched_lcn(Ctx& ctx, const double* h_X, size_t rows, int d, int nprob, const int* h_n, const int* h_m,
                 int kind, double lambda, int buckets, int kmeans_iters, const uint64_t* lsh_seeds, int l,
                 const uint64_t* lm_seeds, int iters, double* dist_out, int* status_out, int* iters_out);
void select_landmarks_device(Op& op, Ctx& ctx, int method, uint64_t seed);
bool tc_build_part(const Op& op, int part);  // the tensor-core build covers `part` (build.cu use_tc_build)
void build_sparse_values(Op& op);
// on: the context to run on (a concurrent build job); null = op.ctx
void build_nystrom(Op& op, const double* h_landmarks, int method, uint64_t seed, Ctx* on = nullptr);
void build_dense(Op& op);
void dense_storage(Op& op);
// dense_tc.cu: the dense kernel recomputed per half-iteration on tcgen05
void dense_tc_prepare(Op& op);
void dense_tc_lse(Op& op, bool transposed, const double* lv, const int* done, double* M, double* S);
void build_dense_cost(Op& op);
void dense_logk_from_cost(Op& op, double lambda);
void build_correction(Op& op);
void finalize_storage(Op& op);
void build_csr(Op& op, Ctx* on = nullptr);  // on: a side context (stream) to build on
void export_csr(Op& op, int which, uint32_t* row_ptr, uint32_t* col, double* vals);
void csr_values_device(Op& op, int which, double* d_vals);
// staged build from host structs (the reference's stage API)
void set_general_csr(Op& op, const uint32_t* h_rp, const uint32_t* h_col, size_t nnz, const double* h_val,
                     const double* h_logsp);
void build_sparse_pairs(Op& op, const uint32_t* d_rp, const uint32_t* d_col, size_t nnz, double* d_out);
void correction_pairs(Ctx& ctx, size_t n, size_t l, const uint32_t* d_rp, const uint32_t* d_col, size_t nnz,
                      const double* d_logsp, const double* d_U, const double* d_Wt, double* d_delta, double* d_nys,
                      double* max_abs);

// Phase timing to stderr when LCN_TIMING is set (host clock around synced phases).
struct PhaseTimer {
    Ctx& ctx;
    const char* name;
    double t0;
    bool on;
    PhaseTimer(Ctx& c, const char* n);
    ~PhaseTimer();
};

// sinkhorn.cu
struct SolveOptions {
    double tol = -1.0;
    int max_iters = 500;
    bool check_support = true;
    bool want_plan = true;
};
void sinkhorn_solve(Op& op, const double* p, const double* q, bool device_ptrs, const SolveOptions& o, Result& res);
void op_log_matvec(Op& op, const double* h_in, bool transposed, double* h_out);
double distance_lcn_device(Op& op, const Result& res);
void extract_plan_device(Op& op, Result& res);
void sinkhorn_solve_bp(Op& op, const double* p, const double* q, const SolveOptions& o, Result& res);

}  // namespace lcnb
