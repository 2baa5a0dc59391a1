/*
 * ORACLE TEST INFRASTRUCTURE — a CPU restatement of the reference's LCN-Sinkhorn
 * hot path in plain C (oracle/lcn_oracle.c). It is the checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's baseline may load
 * it. It is never linked into the product.
 *
 * Parity pin: tests/test_oracle_cpu.py checks it bit-for-bit (bucket ids,
 * support, log K) and to 1e-12 (distances, plans) against oracle/_ref (the
 * reference's own sources compiled unmodified), and against the golden vectors
 * in tests/golden/ (known answers from the reference's test suite and outputs
 * of oracle/_ref committed with tests/golden/make_golden.py).
 *
 * The exported functions mirror oracle/ref_shims/ref_capi.cpp with the orc_
 * prefix so both checkers share oracle/bindings.py.
 */
#ifndef LCN_ORACLE_H
#define LCN_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_kmeans_pp(const double* pts, size_t n, size_t d, size_t k, uint64_t seed, uint32_t* out);
int orc_assign_nearest(const double* pts, size_t n, size_t d, const double* ctr, size_t k, uint32_t* out);
int orc_lloyd(const double* pts, size_t n, size_t d, size_t k, int iters, uint64_t seed, double* centroids,
              uint32_t* assign);
int orc_lsh_kmeans_buckets(const double* p, size_t n, const double* q, size_t m, size_t d, int bands, int buckets,
                           int iters, uint64_t seed, uint64_t* ids);
int orc_lsh_buckets(const double* p, size_t n, const double* q, size_t m, size_t d, int scheme, int bands, int rows,
                    int buckets, int iters, int branching, uint64_t seed, uint64_t* ids);
int orc_cross_polytope_bucket(const double* x, size_t n, size_t d, const double* proj, size_t half, uint32_t* out);
int orc_normal_draws(uint64_t seed, size_t count, double* out);
int orc_lsh_pairs(const double* p, size_t n, const double* q, size_t m, size_t d, int bands, int buckets, int iters,
                  uint64_t seed, void** out);
int orc_pairs_from_buckets(const uint64_t* ids_p, size_t n, const uint64_t* ids_q, size_t m, int bands,
                           uint64_t range, void** out);
int orc_pairs_from_arrays(size_t n, size_t m, const uint32_t* rows, const uint32_t* cols, size_t count, void** out);
size_t orc_pairs_nnz(void* h);
void orc_pairs_copy(void* h, uint32_t* rows, uint32_t* cols);
void orc_pairs_free(void* h);
int orc_op_sparse(const double* p, size_t n, const double* q, size_t m, size_t d, int kind, double lambda,
                  void* pairs, void** out);
int orc_op_lcn(const double* p, size_t n, const double* q, size_t m, size_t d, int kind, double lambda, void* pairs,
               size_t l, int method, uint64_t lm_seed, const double* landmarks, int nystrom_only, void** out,
               double* phase_ms);
int orc_op_dense(const double* p, size_t n, const double* q, size_t m, size_t d, int kind, double lambda, void** out);
void orc_op_free(void* h);
size_t orc_op_nnz(void* h);
size_t orc_op_rank(void* h);
double orc_op_scalar(void* h, int which);
int orc_op_copy(void* h, int which, uint32_t* row_ptr, uint32_t* col, double* vals);
int orc_op_log_matvec(void* h, const double* in, size_t len, int transposed, double* out);
int orc_sinkhorn(void* h, const double* pm, size_t n, const double* qm, size_t m, double tol, int max_iters,
                 int check_support, int want_plan, void** out);
void orc_result_free(void* h);
double orc_result_scalar(void* h, int which);
size_t orc_result_copy(void* h, int which, double* out);
int orc_distance_lcn(void* res, void* op, double* out);
int orc_dense_reference(const double* cost, size_t n, size_t m, const double* p, const double* q, double lambda,
                        double tol, int max_iters, double* plan, double* distance, int* iters);
/* libstdc++ engine/distribution restatements, exposed for pinning tests. */
uint64_t orc_mt19937_64_nth(uint64_t seed, size_t skip);
uint64_t orc_uniform_index(uint64_t seed, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
