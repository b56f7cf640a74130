/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's CPU algorithms for the CAGNET GCN
 * training step (arXiv 2005.03300, reference /root/reference/proj).  Used only
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker.  Every function cites the reference file:line it restates.  All
 * arithmetic is fp64 with the reference's accumulation order; compiled with
 * -ffp-contract=off it reproduces the reference bit for bit (pinned against
 * the reference's golden vectors and against oracle/_ref in tests/).
 *
 * Index arrays are int64; dense matrices are row-major with ld == cols.
 */
#ifndef CAGNET_ORACLE_H
#define CAGNET_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:29-82 — xoshiro256** seeded by splitmix64 */
typedef struct { uint64_t s[4]; } orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_double(orc_rng* r);
uint64_t orc_rng_bounded(orc_rng* r, uint64_t bound);
/* Fisher-Yates permutation (rng.hpp:74-82). */
void orc_rng_permutation(orc_rng* r, int64_t n, int64_t* out);

/* dist_common.cpp:24-36 — ceiling-rule block range; writes [begin, end). */
void orc_block_range(int64_t n, int parts, int idx, int64_t* begin, int64_t* end);

/* csr.cpp:195-218 — directed ER.  col_idx == NULL: count only.  Returns nnz. */
int64_t orc_er_generate(int64_t n, double degree, uint64_t seed, int64_t* row_ptr,
                        int64_t* col_idx);

/* csr.cpp:195-218 on `threads` host threads, bit-identical to orc_er_generate:
 * row u of the reference loop consumes exactly n-1 draws, so a chunk of rows
 * starting at u0 starts its sub-stream at draw u0*(n-1), reached by GF(2)
 * jump-ahead of the (linear) xoshiro256** state update.  Allocates *col_idx
 * (malloc, caller frees); row_ptr has n+1 entries.  Returns nnz or -1. */
int64_t orc_er_generate_mt(int64_t n, double degree, uint64_t seed, int threads,
                           int64_t* row_ptr, int64_t** col_idx);
void orc_free(void* p);
/* Jump-ahead of a seeded generator by `draws` draws (used above; exposed for tests). */
void orc_rng_jump(orc_rng* r, uint64_t draws);

/* csr.cpp:59-92 — from_edge_list (sort + dedup, optional mirroring).  Returns
 * nnz; col_idx == NULL: count only.  Edges are (u[i], v[i]). */
int64_t orc_from_edge_list(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                           int undirected, int64_t* row_ptr, int64_t* col_idx);

/* csr.cpp:94-116 — D^-1/2 (A+I) D^-1/2.  out_col == NULL: count only. */
int64_t orc_normalize(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                      int64_t* out_row_ptr, int64_t* out_col, double* out_vals);

/* csr.cpp:118-138 — counting-sort transpose (columns come out sorted). */
void orc_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                   const int64_t* col_idx, const double* vals, int64_t* t_row_ptr,
                   int64_t* t_col, double* t_vals);

/* csr.cpp:140-162 — block [r0,r1) x [c0,c1) with re-based indices.
 * out_col == NULL: count only.  Returns nnz. */
int64_t orc_extract_block(const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                          int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                          int64_t* out_row_ptr, int64_t* out_col, double* out_vals);

/* csr.cpp:164-179 — acc += A * H (H is n_cols x f). */
void orc_spmm_add(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* vals, const double* h, int64_t f, double* acc);

/* dense.cpp:37-61 — acc += op(a) op(b); a is ar x ac, b is br x bc. */
void orc_gemm_add(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br,
                  int64_t bc, double* acc, int ta, int tb);

/* dense.cpp:80-107 */
void orc_relu(const double* z, int64_t count, double* out);
void orc_log_softmax_rows(const double* z, int64_t rows, int64_t cols, double* out);

/* dense.cpp:109-136 — returns the undivided loss partial; grad is rows x cols. */
double orc_nll_tile(const double* logp, int64_t rows, int64_t cols, const int64_t* labels,
                    const uint8_t* mask, int64_t train_total, int64_t col_begin,
                    double* grad);

/* dataset.cpp:92-108 */
void orc_random_features(int64_t n, int64_t f, uint64_t seed, double* out);
void orc_random_labels(int64_t n, int64_t classes, uint64_t seed, int64_t* out);

/* gnn.cpp:24-44 — weights for all layers concatenated (layer l is dims[l] x dims[l+1]). */
void orc_init_glorot(const int64_t* dims, int ndims, uint64_t seed, double* weights);

/* gnn.cpp:68-132 — full-batch serial training (forward_serial, backward_serial,
 * sgd_step per epoch).  weights in/out (concatenated).  Outputs of the LAST
 * epoch: h_final (n x dims[L-1]), y (concatenated like weights) and g
 * (concatenated, g[l] is n x dims[l+1]).  Any output pointer may be NULL. */
int orc_train_serial(int64_t n, const int64_t* adj_rp, const int64_t* adj_ci,
                     const double* adj_v, const int64_t* adjt_rp, const int64_t* adjt_ci,
                     const double* adjt_v, const double* features, const int64_t* labels,
                     const uint8_t* mask, const int64_t* dims, int ndims, double lr,
                     int epochs, double* weights, double* losses, double* h_final,
                     double* y, double* g);

#ifdef __cplusplus
}
#endif

#endif
