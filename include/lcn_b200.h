/*
 * lcn_b200.h — C-ABI of the B200-native LCN-Sinkhorn hot path.
 *
 * The drop-in boundary for the reference's solver API:
 * every entry point takes plain pointers and sizes, never throws, and returns
 * an lcn_status; lcn_ctx_last_error() holds the message, whose text matches
 * the reference exception's what() so a C++ shim can rethrow the same
 * lcn::Error subtype (error.hpp:8-38) with the same message.
 *
 * Handles are re-entrant per handle (SURVEY.md §8(b) "Threading"): each
 * lcn_ctx owns one device, one stream and its buffers; cudaSetDevice is
 * applied on every entry. There is no global mutable state.
 *
 * Host pointers are row-major fp64 like the reference's PointSet /
 * DenseMatrix (geometry.hpp:14-29, matrix.hpp:10-24). The *_device entry
 * points take device-resident fp32 points (the synthetic configs are fp32,
 * promoted exactly) for timing runs.
 *
 * Each declaration names the reference interface it replaces (file:line,
 * relative to /root/reference/proj).
 */
#ifndef LCN_B200_H
#define LCN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCN_B200_ABI_VERSION 5  /* 3: lcn_op_info_t.streamed; 4: bucket-sharded solve, loopback, shard plan; 5: staged build */

typedef struct lcn_ctx lcn_ctx;
typedef struct lcn_op lcn_op;
typedef struct lcn_result lcn_result;

/* Status codes: 1..6 mirror the lcn::Error subtypes (error.hpp:8-38). */
enum lcn_status {
    LCN_OK = 0,
    LCN_E_DIMENSION = 1,         /* DimensionError */
    LCN_E_INVALID_ARGUMENT = 2,  /* InvalidArgument */
    LCN_E_STABILIZATION = 3,     /* StabilizationError */
    LCN_E_NEGATIVE_KERNEL = 4,   /* NegativeKernelError */
    LCN_E_FACTORIZATION = 5,     /* FactorizationError */
    LCN_E_ERROR = 6,             /* lcn::Error */
    LCN_E_CUDA = 100,            /* CUDA runtime failure */
    LCN_E_NO_DEVICE = 101        /* no usable sm_100 device */
};

/* CostKind (geometry.hpp:35-39) plus the documented squared-L2 extension. */
enum lcn_cost { LCN_COST_EUCLIDEAN = 0, LCN_COST_NEGATIVE_DOT = 1, LCN_COST_COSINE_DERIVED = 2, LCN_COST_SQEUCLIDEAN = 3 };

/* LandmarkMethod (nystrom.hpp:14-17). */
enum lcn_landmark_method { LCN_LANDMARK_KMEANS = 0, LCN_LANDMARK_KMEANSPP = 1 };

/* Operator kinds (operator.hpp:33 KernelOperator::Kind). */
enum lcn_op_kind { LCN_OP_DENSE = 0, LCN_OP_SPARSE = 1, LCN_OP_NYSTROM = 2, LCN_OP_LCN = 3 };

/* Context flags: value storage of the iteration operands. FP64 keeps every
 * stored kernel value in fp64 (API-compatibility mode, passes the reference
 * unit tests' 1e-12 tolerances); FP32 stores them in fp32 with fp64
 * accumulation (performance mode, 1e-4 parity). */
enum lcn_ctx_flags { LCN_STORE_FP32 = 0, LCN_STORE_FP64 = 1, LCN_EXACT_BUILD = 2, LCN_DENSE_RECOMPUTE = 4 };
/* LCN_DENSE_RECOMPUTE (fp32 storage, configs[2]'s wording): lcn_op_dense /
 * lcn_op_dense_device keep no n x m log K; every half-iteration recomputes
 * the kernel as a tcgen05 3xTF32 GEMM of the points (x.y, fp64 norms) fused
 * with the row / column log-sum-exp (dense_tc.cu). The plan and
 * export_dense rebuild the exact log K on demand. Not for the cosine cost. */
/* Build contractions. FP32 storage computes the within-bucket distance
 * blocks of K^sp, the point x landmark blocks U and V, and the delta SDDMM
 * U_b W_b on the tcgen05 tensor cores in the FP32-accurate 3xTF32 split
 * (values within ~1e-5 of the reference, support unchanged). LCN_EXACT_BUILD
 * (or FP64 storage) keeps the exact fp64 CUDA-core tiles instead: the
 * reference's sequential fp64 folds, log K bit-exact (the export mode). The
 * landmark Gram matrix A and W = A^-1 V are always fp64 (the reference's
 * 1e-6 residual acceptance test, nystrom.cpp:104-124). */

/* LshScheme (lsh.hpp:13-17), same values. */
enum lcn_lsh_scheme { LCN_LSH_CROSS_POLYTOPE = 0, LCN_LSH_KMEANS = 1, LCN_LSH_HIERARCHICAL_KMEANS = 2 };

/* LshConfig (lsh.hpp:22-30). ABI 2 appended `scheme` and `branching`; a
 * zero-initialised tail means scheme 0 (cross-polytope), so set scheme
 * explicitly (LCN_LSH_KMEANS is the reference default). */
typedef struct {
    int bands;
    int rows_per_band;
    int buckets_per_fn;  /* even for cross-polytope */
    int kmeans_iters;
    uint64_t seed;
    int scheme;          /* enum lcn_lsh_scheme */
    int branching;       /* hierarchical k-means only (reference default 2) */
} lcn_lsh_config;

/* SinkhornOptions (sinkhorn.hpp:11-20). tol < 0 selects 1e-6 (sum p + sum q). */
typedef struct {
    double tol;
    int max_iters;
    int check_support;
    int want_plan;
} lcn_sinkhorn_options;

typedef struct {
    int kind;                 /* lcn_op_kind */
    size_t n, m, l, d;
    int bands;
    size_t nnz;               /* deduplicated support size (= pairs.size()) */
    size_t stored;            /* bucket-block entries held in HBM (>= nnz) */
    double lambda;
    double max_abs_delta;     /* LcnCorrection::max_abs_delta (sparse_kernel.hpp:46) */
    double cond_estimate;     /* NystromFactors::cond_estimate (nystrom.hpp:37) */
    int store_fp64;
    size_t streamed;          /* band entries one column pass streams (LCN iteration layout, >= nnz) */
} lcn_op_info_t;

typedef struct {
    double distance;
    int iters;
    int converged;
    double marginal_err_final;
    int n_warnings;
    double device_ms;         /* CUDA-event time of the iteration loop */
} lcn_result_info_t;

/* ---- context ---------------------------------------------------------- */
int lcn_ctx_create(int device, int flags, lcn_ctx** out);
int lcn_ctx_destroy(lcn_ctx* ctx);
const char* lcn_ctx_last_error(const lcn_ctx* ctx);
/* Run the context's work on an external stream (a cudaStream_t, e.g. torch's
 * current stream, so the caller's CUDA events bracket it); NULL restores the
 * context's own stream. */
int lcn_ctx_set_stream(lcn_ctx* ctx, void* stream);
/* Record per-phase CUDA events inside lcn_sinkhorn (see lcn_result_phase_ms). */
int lcn_ctx_set_profile(lcn_ctx* ctx, int on);
/* Work counter of the tensor-core assignment filter on the context's device
 * (profiling; no reference counterpart): point x 128-centroid tile products
 * evaluated since the last reset, one product = 2 * 128 * 128 * 3 MMA flops
 * (3xTF32) at d <= 128. Synchronous; reset != 0 zeroes it after the read. */
int lcn_ctx_tc_work(lcn_ctx* ctx, int reset, unsigned long long* point_tiles);

/* ---- sharded solve over several GPUs ------------------ */
/* A fresh NCCL unique id (128 bytes) on the calling rank (rank 0 makes it,
 * the caller broadcasts it). */
int lcn_nccl_unique_id(uint8_t* out128);
/* Join `world` ranks (one process or thread per GPU) into one NCCL
 * communicator; collective over the ranks. LCN operators built afterwards on
 * this context are bucket-sharded: every rank passes the same full inputs;
 * the LSH bucket ids and the landmarks are computed on every rank (bit-exact,
 * so identical), then each rank keeps only the points of its band-0 buckets
 * plus the halo points a later band makes it read (lcn_shard_plan_*), and
 * builds K_sp / delta / U / W for those alone. lcn_sinkhorn* then solve ONE
 * problem together: per half-iteration one all-gather of each rank's packed
 * [low-rank partial (l), shift, error, flags, exported halo scalings]; the
 * owned slices of log s / log t / P1 are all-gathered once at the end, so
 * every rank returns the full result. world = 1 is valid. */
int lcn_ctx_set_comm(lcn_ctx* ctx, int world, int rank, const uint8_t* id128);
/* Bucket-sharded partition plan (host only; no GPU needed). The plan a
 * sharded context builds internally, exposed so callers and tests can see
 * the partition: ids_src (bands x n) / ids_tgt (bands x m) are dense bucket
 * ids < range[b]. Points are owned by the rank of their band-0 bucket (the
 * shard unit: neighbor_pairs emits every pair inside a bucket,
 * lsh.cpp:222-239); a later band's bucket that spans ranks makes its members
 * halo points of the other ranks. Local point order per rank: owned points
 * ascending by global index, then halo points ascending. */
typedef struct lcn_shard_plan lcn_shard_plan;
typedef struct {
    size_t n_own, n_halo, m_own, m_halo;  /* local sources / targets */
    size_t exp_s, exp_t;                  /* owned points other ranks read */
    size_t max_exp_s, max_exp_t;          /* exchange slots (max over ranks) */
    double cost;                          /* modelled bytes per iteration */
    unsigned long long band0_pairs;       /* sum n_b m_b of the owned band-0 buckets */
    size_t groups;                        /* band-0 bucket groups of the plan */
} lcn_shard_rank_info;
int lcn_shard_plan_create(const uint32_t* ids_src, size_t n, const uint32_t* ids_tgt, size_t m, int bands,
                          const uint32_t* range, size_t l, int world, lcn_shard_plan** out);
int lcn_shard_plan_rank_info(const lcn_shard_plan* plan, int rank, lcn_shard_rank_info* info);
/* local -> global indices (n_own + n_halo, m_own + m_halo entries) */
int lcn_shard_plan_rank_points(const lcn_shard_plan* plan, int rank, uint32_t* src, uint32_t* tgt);
/* exp_*: local indices of the exported owned points (slot order); imp_*: per
 * halo point, its owner rank and the slot it has in the owner's export */
int lcn_shard_plan_rank_exchange(const lcn_shard_plan* plan, int rank, uint32_t* exp_s, uint32_t* exp_t,
                                 uint32_t* imp_s_rank, uint32_t* imp_s_slot, uint32_t* imp_t_rank,
                                 uint32_t* imp_t_slot);
const char* lcn_shard_plan_last_error(void);
int lcn_shard_plan_destroy(lcn_shard_plan* plan);
/* In-process loopback communicator: `world` ranks as host threads sharing
 * one device (each with its own lcn_ctx); the all-gather is a host barrier
 * plus device copies, and no kernel ever waits on another rank's kernel.
 * For testing the sharded CUDA path with fewer GPUs than ranks. A rank that
 * fails should call lcn_loopback_abort so the others leave the barrier. */
typedef struct lcn_loopback lcn_loopback;
int lcn_loopback_create(int world, lcn_loopback** out);
int lcn_ctx_set_loopback(lcn_ctx* ctx, lcn_loopback* lb, int rank);
int lcn_loopback_abort(lcn_loopback* lb);
int lcn_loopback_destroy(lcn_loopback* lb);
const char* lcn_status_name(int status);
int lcn_abi_version(void);

/* ---- k-means (kmeans.hpp:18-29) --------------------------------------- */
/* kmeans_pp_indices (kmeans.cpp:23-65). The caller's std::mt19937_64 supplies
 * first_index = uniform_int_distribution<size_t>(0,n-1)(rng) and then up to
 * k-1 raw 64-bit draws; *draws_used reports how many the reference would have
 * consumed (a step with total <= 0 consumes none, kmeans.cpp:42-47), so the
 * shim can advance its engine identically. */
int lcn_kmeans_pp_indices(lcn_ctx* ctx, const double* points, size_t n, size_t d, size_t k,
                          uint64_t first_index, const uint64_t* raw_draws, size_t n_draws,
                          uint32_t* out, size_t* draws_used);
/* assign_nearest (kmeans.cpp:67-85): ties to the lowest index. */
int lcn_assign_nearest(lcn_ctx* ctx, const double* points, size_t n, size_t d,
                       const double* centroids, size_t k, uint32_t* out);
/* lloyd (kmeans.cpp:87-143), mt19937_64(seed) k-means++ init. */
int lcn_lloyd(lcn_ctx* ctx, const double* points, size_t n, size_t d, size_t k, int iters,
              uint64_t seed, double* centroids_out, uint32_t* assign_out);

/* ---- LSH (lsh.hpp:49-68) ---------------------------------------------- */
/* Bucket ids of lsh_neighbor_pairs (lsh.cpp:245-283) for cfg->scheme:
 * ids_out is bands x (n+m) (p's points first), the composite mixed-radix id
 * over the rows_per_band functions; cross-polytope = hash_cross_polytope
 * (lsh.cpp:73-103) of p and q, k-means / hierarchical = hash_kmeans
 * (lsh.cpp:145-158) of X_p ∪ X_q with fn_seed(seed, band, fn). */
int lcn_lsh_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m,
                    size_t d, const lcn_lsh_config* cfg, uint64_t* ids_out);
/* ABI-1 name of lcn_lsh_buckets (same behaviour). */
int lcn_lsh_kmeans_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m,
                           size_t d, const lcn_lsh_config* cfg, uint64_t* ids_out);
/* cross_polytope_bucket (lsh.cpp:55-71) of n points against an explicit
 * projection proj (d x half, row-major): argmax of [x^T R || -x^T R]. */
int lcn_cross_polytope_buckets(lcn_ctx* ctx, const double* points, size_t n, size_t d,
                               const double* proj, size_t half, uint32_t* out);

/* ---- operators (operator.hpp:29-82) ----------------------------------- */
/* Sparse operator on the k-means LSH support: lsh_neighbor_pairs
 * (lsh.cpp:245) -> build_sparse (sparse_kernel.cpp:51) -> KernelOperator::sparse
 * (operator.cpp:67). */
int lcn_op_sparse_lsh(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                      int cost, double lambda, const lcn_lsh_config* cfg, lcn_op** out);
/* Same from external bucket ids (neighbor_pairs(BandBuckets...), lsh.cpp:212):
 * ids_p is bands x n, ids_q bands x m, values < range. */
int lcn_op_sparse_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                          int cost, double lambda, const uint64_t* ids_p, const uint64_t* ids_q,
                          int bands, uint64_t range, lcn_op** out);
/* LCN operator: LSH support + select_landmarks (nystrom.cpp:28) +
 * build_factors (nystrom.cpp:68) + build_correction (sparse_kernel.cpp:82) +
 * KernelOperator::lcn (operator.cpp:90). */
int lcn_op_lcn_lsh(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                   int cost, double lambda, const lcn_lsh_config* cfg, size_t l, int landmark_method,
                   uint64_t landmark_seed, lcn_op** out);
/* Same from external bucket ids and (optionally) explicit landmarks (l x d);
 * landmarks == NULL selects them with select_landmarks(l, method, seed).
 * bands == 0 builds a pure Nystrom operator (KernelOperator::nystrom). */
int lcn_op_lcn_buckets(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                       int cost, double lambda, const uint64_t* ids_p, const uint64_t* ids_q, int bands,
                       uint64_t range, const double* landmarks, size_t l, int landmark_method,
                       uint64_t landmark_seed, lcn_op** out);
/* Device-resident variant for timing runs: d_p (n x d) and d_q (m x d) are
 * fp32 device pointers. landmarks <= 0 builds the sparse operator. */
int lcn_op_create_device(lcn_ctx* ctx, const float* d_p, size_t n, const float* d_q, size_t m, size_t d,
                         int cost, double lambda, const lcn_lsh_config* cfg, size_t l, int landmark_method,
                         uint64_t landmark_seed, lcn_op** out);
/* Dense operator (configs[2] anchor): build_cost + build_kernel +
 * KernelOperator::dense (geometry.cpp:113-144, operator.cpp:55-64); log K of
 * every pair from the sequential fp64 fold (bit-exact). The plan of a dense
 * solve is the full n x m matrix (lcn_result_copy which 4, row-major). */
int lcn_op_dense(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                 double lambda, lcn_op** out);
/* Same from device-resident fp32 points (timing runs). */
int lcn_op_dense_device(lcn_ctx* ctx, const float* d_p, size_t n, const float* d_q, size_t m, size_t d, int cost,
                        double lambda, lcn_op** out);
/* DenseKernel::logk (n x m, row-major). */
int lcn_op_export_dense(lcn_op* op, double* out);
/* multihead_lambdas + multihead (sinkhorn.cpp:322-353): lambda_k =
 * 2^(k - heads/2) lambda for k = 1..heads, independent dense solves over one
 * cost matrix (computed once on the device). Per head: lambda, distance,
 * iterations, converged flag and status (0, or the lcn_status of the head's
 * error; lcn_ctx_last_error holds the last head error message). */
int lcn_multihead(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, int cost,
                  double lambda, int heads, const double* pmarg, const double* qmarg,
                  const lcn_sinkhorn_options* opts, double* lambdas_out, double* dist_out, int* iters_out,
                  int* converged_out, int* status_out);
/* configs[4]: nprob independent small LCN problems in ragged launches (one
 * CTA per problem). X holds the problems back to back, problem k as n[k]
 * source rows then m[k] target rows (d columns, row-major). Per problem, as
 * the reference pipeline: lsh_neighbor_pairs with k-means LSH (1 band,
 * `buckets`, kmeans_iters, lsh_seeds[k]) -> build_sparse -> select_landmarks
 * (KMeans, l, landmark_seeds[k]) -> build_factors -> build_correction ->
 * KernelOperator::lcn -> sinkhorn with uniform marginals, tol 0, `iters`
 * iterations. Outputs per problem: the distance, the status (0, or the
 * lcn_status of the reference's first error for that problem; its distance
 * is NaN) and the iterations run. Limits on this path: d <= 32,
 * n + m <= 1024, buckets and l in [2 or 1, 16], cost euclidean or squared
 * euclidean. */
int lcn_batched_lcn(lcn_ctx* ctx, const double* X, size_t rows, size_t d, int nprob, const int* n, const int* m,
                    int cost, double lambda, int buckets, int kmeans_iters, const uint64_t* lsh_seeds, size_t l,
                    const uint64_t* landmark_seeds, int iters, double* distance_out, int* status_out,
                    int* iters_out);
/* KernelOperator::with_bp (operator.cpp:103-115), in place: deletion kernels
 * c_{p,eps} (n) and c_{eps,q} (m), finite and >= 0 (BpExtension::from_costs
 * gives exp(-c / lambda), operator.cpp:33-43). Solves then use the extended
 * problem of sinkhorn.cpp:115-120 with unbalanced marginals allowed. NULL,
 * NULL removes the extension. Not on sharded contexts. */
int lcn_op_set_bp(lcn_op* op, const double* del_p, const double* del_q);
int lcn_op_destroy(lcn_op* op);
int lcn_op_get_info(const lcn_op* op, lcn_op_info_t* info);
/* CSR export in the reference's order (rows ascending, columns ascending,
 * sparse_kernel.hpp:19-21). which: 0 log K^sp (SparseKernel::logvals),
 * 1 delta, 2 log_sp, 3 nys_vals (LcnCorrection, sparse_kernel.hpp:43-45).
 * row_ptr has n+1 entries; col/vals nnz (lcn_op_get_info). Any may be NULL. */
int lcn_op_export_csr(lcn_op* op, int which, uint32_t* row_ptr, uint32_t* col, double* vals);
/* Dense factor export: 0 U (n x l), 1 W (l x m), 2 landmarks (l x d). */
int lcn_op_export_factor(lcn_op* op, int which, double* out);
/* log_matvec / log_matvec_t (operator.cpp:226-252), host vectors. */
int lcn_op_log_matvec(lcn_op* op, const double* in, int transposed, double* out);

/* ---- staged build from host structs ------------------------------------ */
/* The reference's caller builds an LCN operator in stages and hands host
 * structs between them (runner.cpp:258-271): lsh_neighbor_pairs ->
 * build_sparse -> select_landmarks -> build_factors -> build_correction ->
 * KernelOperator::lcn(factors, correction). Each stage below takes and returns
 * the plain arrays of those structs, so a shim can keep the reference's types
 * (integration/lcn_shim.cpp). Patterns are CSR: row_ptr
 * (n + 1), col (nnz), sorted and unique within a row, as NeighborPairs /
 * SparseKernel / LcnCorrection hold them (sparse_kernel.hpp:17-50). */
typedef struct lcn_pairs lcn_pairs;
/* lsh_neighbor_pairs (lsh.hpp:67-68, lsh.cpp:245-283): the support of the
 * configured LSH as a NeighborPairs CSR (pairs sorted row-major, unique). */
int lcn_lsh_neighbor_pairs(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                           const lcn_lsh_config* cfg, lcn_pairs** out);
int lcn_pairs_info(const lcn_pairs* pairs, size_t* n, size_t* m, size_t* nnz);
int lcn_pairs_copy(const lcn_pairs* pairs, uint32_t* row_ptr, uint32_t* col);
int lcn_pairs_destroy(lcn_pairs* pairs);
/* build_sparse (sparse_kernel.hpp:32-33, sparse_kernel.cpp:51-80): logvals
 * = 0 - c(p_i, q_j) * (1 / lambda) at the pattern, bit-exact (the reference's
 * sequential fp64 folds on the device). */
int lcn_build_sparse(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                     const uint32_t* row_ptr, const uint32_t* col, size_t nnz, int cost, double lambda,
                     double* logvals);
/* select_landmarks (nystrom.hpp:26-27, nystrom.cpp:28-48): l x d, bit-exact. */
int lcn_select_landmarks(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d, size_t l,
                         int method, uint64_t seed, double* out);
/* build_factors (nystrom.hpp:46-47, nystrom.cpp:68-125): U = k(X_p, L)
 * (n x l) and W = A^-1 V (l x m), row-major like NystromFactors::u / ::w;
 * same jitter schedule and FactorizationError. */
int lcn_build_factors(lcn_ctx* ctx, const double* p, size_t n, const double* q, size_t m, size_t d,
                      const double* landmarks, size_t l, int cost, double lambda, double* U, double* W,
                      double* cond_estimate);
/* build_correction (sparse_kernel.hpp:54, sparse_kernel.cpp:82-117): delta
 * = exp(log_sp) - (U W)_ij and nys_vals = (U W)_ij at the pattern (the
 * reference's sequential entry() fold); max |delta|; StabilizationError on
 * overflow. */
int lcn_build_correction(lcn_ctx* ctx, size_t n, size_t m, size_t l, const uint32_t* row_ptr, const uint32_t* col,
                         size_t nnz, const double* log_sp, const double* U, const double* W, double* delta,
                         double* nys_vals, double* max_abs_delta);
/* KernelOperator factories (operator.hpp:33-36) from the host structs:
 * dense(DenseKernel) = n x m log K; sparse(SparseKernel) = any CSR pattern
 * with its log K; nystrom(NystromFactors); lcn(NystromFactors,
 * LcnCorrection) = factors + any CSR pattern with delta and log K^sp. General
 * patterns run on CSR / CSC kernels (fp64 values); the bucket-blocked fast
 * path is the lcn_op_*_lsh / _buckets family. */
int lcn_op_from_dense(lcn_ctx* ctx, size_t n, size_t m, const double* logk, double lambda, lcn_op** out);
int lcn_op_from_sparse(lcn_ctx* ctx, size_t n, size_t m, const uint32_t* row_ptr, const uint32_t* col, size_t nnz,
                       const double* logvals, double lambda, lcn_op** out);
int lcn_op_from_nystrom(lcn_ctx* ctx, size_t n, size_t m, size_t l, const double* U, const double* W, double lambda,
                        lcn_op** out);
int lcn_op_from_lcn(lcn_ctx* ctx, size_t n, size_t m, size_t l, const double* U, const double* W, double lambda,
                    const uint32_t* row_ptr, const uint32_t* col, size_t nnz, const double* delta,
                    const double* log_sp, double max_abs_delta, lcn_op** out);

/* ---- solver (sinkhorn.hpp:68-121) ------------------------------------- */
/* sinkhorn (sinkhorn.cpp:104-188). p (n), q (m) host marginals. */
int lcn_sinkhorn(lcn_op* op, const double* p, const double* q, const lcn_sinkhorn_options* opts,
                 lcn_result** out);
/* Device-resident marginals (fp64 device pointers); no plan extraction.
 * Marginal validation is the caller's (timing entry point). */
int lcn_sinkhorn_device(lcn_op* op, const double* d_p, const double* d_q, const lcn_sinkhorn_options* opts,
                        lcn_result** out);
/* Profiling (lcn_ctx_set_profile): summed ms of the four phases of
 * iterations 1..iters: column band blocks, column finalize + reduce, row band
 * blocks, row finalize + reduce + iteration end. */
int lcn_result_phase_ms(const lcn_result* res, double* out4, int* iters);
int lcn_result_destroy(lcn_result* res);
int lcn_result_get_info(const lcn_result* res, lcn_result_info_t* info);
/* which: 0 log_s (n), 1 log_t (m), 2 row_marginal (n), 3 marginal_err trace,
 * 4 sparse plan values (Plan::sparse_vals, CSR order), 5 lcn sp_vals,
 * 6 lcn sp_nys_vals; under BP (lcn_op_set_bp): 7 del_p_mass (n), 8 del_q_mass
 * (m), 9 eps_mass (1) (Plan, sinkhorn.hpp:47-51), and 0-3 are the extended
 * (n + m) vectors. out == NULL returns the length in *len only. */
int lcn_result_copy(const lcn_result* res, int which, double* out, size_t* len);
/* grad_cost (sinkhorn.cpp:263-320). which: 0 dense / sparse d d / d C (the plan:
 * n x m row-major, or CSR order), 1 lcn / nystrom d d / d U (n x l),
 * 2 d d / d W (l x m), 3 lcn d d / d log K^sp = -lambda P^sp, 4 lcn
 * d d / d log K^sp_Nys = +lambda P^sp_Nys. out == NULL returns the length in
 * *len; *stale = 1 when the result did not converge (a warning is printed). */
int lcn_grad_cost(const lcn_result* res, const lcn_op* op, int which, double* out, size_t* len, int* stale);
/* distance_lcn (sinkhorn.cpp:222-261). */
int lcn_distance_lcn(const lcn_result* res, const lcn_op* op, double* out);
/* Warning text i (SinkhornResult::warnings, sinkhorn.cpp:122-128). */
const char* lcn_result_warning(const lcn_result* res, int i);

/* ---- Data formats and generators either side of the path (host only, no
 * device needed). Errors: LCN_E_INVALID_ARGUMENT with
 * the reference's InvalidArgument text in lcn_io_last_error(). ---- */
/* read_points_file (io.cpp:105-116): LCNPTS1 binary (magic, u64-LE n, u64-LE
 * d, n*d f64-LE; io.cpp:77-95) or text (`n d` then rows, '#' comments;
 * io.cpp:33-63), PointSet::validate (geometry.cpp:10-18). out == NULL returns
 * the shape in *n, *d; otherwise *n, *d must hold that shape. */
int lcn_points_read(const char* path, double* out, size_t* n, size_t* d);
/* write_points_file (io.cpp:118-126): binary != 0 LCNPTS1, else text with 17
 * significant digits (io.cpp:65-75). */
int lcn_points_write(const char* path, const double* pts, size_t n, size_t d, int binary);
/* sample_uniform_ball (generators.cpp:26-40): n x d, the reference's draws. */
int lcn_sample_uniform_ball(size_t n, size_t d, uint64_t seed, double* out);
/* sample_clustered (generators.cpp:42-106): p and q n x d each, centers c x d
 * (centers_out may be NULL). */
int lcn_sample_clustered(size_t n, size_t d, size_t c, double D, double r, uint64_t seed, double* p_out,
                         double* q_out, double* centers_out);
const char* lcn_io_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LCN_B200_H */
