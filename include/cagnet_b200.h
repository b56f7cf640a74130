/*
 * cagnet_b200 — C-ABI of the B200-native CAGNET full-batch GCN training step
 * (arXiv 2005.03300).  Plain pointers and sizes only; no torch or C++ types.
 *
 * Two levels:
 *   1. kernel seams  — the device equivalents of the free functions the
 *      reference strategies call: spmm_add, gemm_add, the fused
 *      log_softmax/NLL tile, relu/hadamard epilogues, sgd_step.  All device
 *      pointers are caller-owned; `stream` is a cudaStream_t (NULL = legacy
 *      default stream).
 *   2. API level     — the reference's graph-loading / partitioning /
 *      training-loop API (dataset.hpp, gnn.hpp, dist.hpp) with device-resident
 *      state behind opaque handles owned by the library until *_free.
 *
 * Every function returns CAGNET_OK (0) or an error code; the message for the
 * calling thread is available from cagnet_last_error().  Shape errors are
 * validated on the host before any launch (mirroring the reference's
 * std::invalid_argument "who: shape ..." messages).
 */
#ifndef CAGNET_B200_H
#define CAGNET_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CAGNET_API __attribute__((visibility("default")))
#else
#define CAGNET_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CAGNET_OK 0
#define CAGNET_EINVAL 1    /* std::invalid_argument in the reference */
#define CAGNET_ECUDA 2     /* CUDA runtime / launch failure */
#define CAGNET_ENCCL 3     /* NCCL failure (collective misuse, peer loss) */
#define CAGNET_ERUNTIME 4  /* std::runtime_error in the reference (I/O, divergence) */

/* gemm epilogues (fused after the tcgen05 accumulation) */
#define CAGNET_EPI_NONE 0        /* C (+)= op(A) op(B) */
#define CAGNET_EPI_RELU 1        /* C = Z; aux_out = relu(Z)         dense.cpp:80-85 */
#define CAGNET_EPI_RELU_PRIME 2  /* C = acc * (aux > 0)              dense.cpp:72-92 */

/* strategies (dist.hpp:41) */
#define CAGNET_1D 0
#define CAGNET_15D 1
#define CAGNET_2D 2
#define CAGNET_3D 3

/* dataset generators */
#define CAGNET_GEN_REFERENCE 0  /* bit-exact reference ER (csr.cpp:195-218), O(n^2) draws on GPU */
#define CAGNET_GEN_SKIP 1       /* O(nnz) geometric-skip ER-shaped graph (Amazon/Protein scale) */

CAGNET_API const char* cagnet_last_error(void);
CAGNET_API int cagnet_version(void);
CAGNET_API int cagnet_device_count(int* out);

/* ------------------------------------------------------------------------ */
/* 0. host-only partition geometry (no GPU needed)                           */
/* ------------------------------------------------------------------------ */

/* block_range (dist_common.cpp:29-36): out2 = {begin, end} of part idx. */
CAGNET_API int cagnet_block_range(int64_t n, int parts, int idx, int64_t* out2);
/* make_grid (dist_common.cpp:55-65): out4 = {grid kind, rows, cols, layers};
 * CAGNET_EINVAL for impossible shapes (non-square 2D, non-cube 3D, c ∤ P). */
CAGNET_API int cagnet_grid_shape(int kind, int ranks, int repl, int* out4);
/* ProcessGrid groups (grid.cpp:142-189): which 0 world, 1 row, 2 column,
 * 3 fiber; members ascending (capacity `ranks`). */
CAGNET_API int cagnet_grid_group(int kind, int ranks, int repl, int rank, int which, int* members,
                      int* count);
/* Trainer::tile_rows / tile_cols / tile_owner without a trainer:
 * out5 = {r0, r1, c0, c1, owner}. */
CAGNET_API int cagnet_tile_geometry(int kind, int ranks, int repl, int64_t n, int rank, int64_t width,
                         int64_t* out5);

/* ------------------------------------------------------------------------ */
/* 1. kernel seams                                                           */
/* ------------------------------------------------------------------------ */

/* spmm_add (csr.cpp:164-179; csr.hpp:71-75): T[i,:] (+)= sum_k vals[k] * H[col[k],:]
 * in ascending-nonzero order per row.  row_ptr int64[n_rows+1], col_idx int32[nnz],
 * vals fp32[nnz].  H is n_cols x f (leading dim ldh), T is n_rows x f (ldt).
 * accumulate=0 overwrites T (spmm, csr.cpp:181-185). */
CAGNET_API int cagnet_spmm_csr_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const float* vals, const float* H, int64_t ldh,
                        int32_t f, float* T, int64_t ldt, int accumulate, void* stream);

/* spmm (csr.cpp:181-185) fused with the next dense step of the GCN layer, for
 * f <= 32 and 16 B-aligned rows (ldh, ldt multiples of 4): t = A·H (row by
 * row, in registers); raw_out (optional) = t; z = W ? t·W : t with W f x fo
 * (element (k, c) at W[k*w_sk + c*w_sn], fo <= 64; gemm, dense.cpp:37-70);
 * z *= 1[mask > 0] when mask (hadamard with relu_prime, dense.cpp:72-92);
 * T = z; relu_out (optional) = relu(z) (dense.cpp:72-80). */
CAGNET_API int cagnet_spmm_fused_f32(int64_t n_rows, int64_t n_cols, int64_t nnz,
                          const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                          const float* H, int64_t ldh, int32_t f, const float* W, int64_t w_sk,
                          int64_t w_sn, int32_t fo, const float* mask, int64_t mask_ld, float* T,
                          int64_t ldt, float* relu_out, int64_t relu_ld, float* raw_out,
                          int64_t raw_ld, void* stream);

/* gemm_add / gemm (dense.cpp:37-70; dense.hpp:63-71): C (+)= op(A) op(B) on
 * tcgen05 tensor cores, split-TF32 (3 MMAs: hi*hi + hi*lo + lo*hi), fp32
 * accumulation in TMEM.  op(A) is m x k, op(B) is k x n; A is stored
 * (ta ? k x m : m x k) with leading dim lda, B (tb ? n x k : k x n) with ldb.
 * Epilogue per CAGNET_EPI_*: RELU writes Z to C and relu(Z) to aux_out (ldao);
 * RELU_PRIME multiplies by 1[aux > 0] (ldaux).  Large k is split across CTAs
 * and reduced deterministically. */
CAGNET_API int cagnet_gemm_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* A,
                    int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                    int accumulate, int epilogue, const float* aux, int64_t ldaux,
                    float* aux_out, int64_t ldao, void* stream);

/* log_softmax_rows + nll_tile fused (dense.cpp:94-136).  Z holds full rows
 * (rows x cols, ldz).  Writes the column tile [c0, c1) of log-probabilities to
 * logp (ldl) and of the gradient (softmax - onehot)/train_total on masked rows
 * to G (ldg); *loss_partial (device fp64) receives the undivided
 * -sum logp[y] over masked rows whose label lies in [c0, c1).
 * labels int32[rows] (may be NULL when G is NULL), mask uint8[rows] (NULL = all). */
CAGNET_API int cagnet_logsoftmax_nll_f32(const float* Z, int64_t rows, int32_t cols, int64_t ldz,
                              int32_t c0, int32_t c1, float* logp, int64_t ldl, float* G,
                              int64_t ldg, const int32_t* labels, const uint8_t* mask,
                              int64_t train_total, double* loss_partial, void* stream);

/* relu (dense.cpp:80-85), out-of-place, rows x cols with leading dims. */
CAGNET_API int cagnet_relu_f32(const float* Z, int64_t rows, int32_t cols, int64_t ldz, float* H,
                    int64_t ldh, void* stream);

/* sgd_step (gnn.cpp:106-120): W -= lr * Y elementwise over `count` floats. */
CAGNET_API int cagnet_sgd_f32(float* W, const float* Y, int64_t count, float lr, void* stream);

/* ------------------------------------------------------------------------ */
/* 2. API level                                                              */
/* ------------------------------------------------------------------------ */

typedef struct cagnet_csr_s* cagnet_csr_t;         /* device CSR (int64 row_ptr, int32 col, fp32 vals) */
typedef struct cagnet_dataset_s* cagnet_dataset_t; /* device GraphDataset (dataset.hpp:31-45) */
typedef struct cagnet_trainer_s* cagnet_trainer_t; /* one rank of a Trainer (dist.hpp:83-131) */

/* --- device CSR ------------------------------------------------------------ */
CAGNET_API int cagnet_csr_upload(int device, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                      const int64_t* col_idx, const double* vals, cagnet_csr_t* out);
/* shape = {n_rows, n_cols, nnz} */
CAGNET_API int cagnet_csr_shape(cagnet_csr_t a, int64_t* shape);
/* Any output may be NULL.  vals are the fp32 device values. */
CAGNET_API int cagnet_csr_download(cagnet_csr_t a, int64_t* row_ptr, int64_t* col_idx, float* vals);
/* Raw device pointers (for the kernel seams). */
CAGNET_API int cagnet_csr_device_ptrs(cagnet_csr_t a, const int64_t** row_ptr, const int32_t** col_idx,
                           const float** vals);
CAGNET_API int cagnet_csr_free(cagnet_csr_t a);

/* generate_erdos_renyi (csr.cpp:195-218) on the GPU, bit-exact: every ordered
 * pair draws once from the same xoshiro256** stream (rows start at a GF(2)
 * jump of u*(n-1) draws). */
CAGNET_API int cagnet_er_generate(int device, int64_t n, double degree, uint64_t seed, cagnet_csr_t* out);
/* add_self_loops_and_normalize (csr.cpp:94-116) on the GPU: fp64 1/sqrt(d_i d_j) rounded to fp32. */
CAGNET_API int cagnet_csr_normalize(cagnet_csr_t raw, cagnet_csr_t* out);
/* transpose (csr.cpp:118-138) on the GPU (stable radix sort by column). */
CAGNET_API int cagnet_csr_transpose(cagnet_csr_t a, cagnet_csr_t* out);
/* extract_block (csr.cpp:140-162) on the GPU. */
CAGNET_API int cagnet_csr_extract_block(cagnet_csr_t a, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                             cagnet_csr_t* out);

/* --- datasets (dataset.hpp:46-93) ------------------------------------------- */
/* generate_dataset(n, d, f, C, sg, sf, sl) built on `device`: ER (generator per
 * CAGNET_GEN_*), normalization, transpose, U[0,1) features, uniform labels,
 * all-ones mask. */
CAGNET_API int cagnet_dataset_generate(int device, int64_t n, double degree, int64_t num_features,
                            int64_t num_classes, uint64_t seed_graph, uint64_t seed_features,
                            uint64_t seed_labels, int generator, cagnet_dataset_t* out);
/* make_dataset (dataset.cpp:76-90) from a raw host CSR (unit values implied),
 * fp64 features (n x f), labels int64[n], mask uint8[n] (NULL = all ones). */
CAGNET_API int cagnet_dataset_make(int device, int64_t n, const int64_t* raw_row_ptr,
                        const int64_t* raw_col_idx, const double* features, int64_t f,
                        const int64_t* labels, const uint8_t* mask, int64_t num_classes,
                        cagnet_dataset_t* out);
/* info = {n, nnz, num_features, num_classes, train_count} */
/* load_dataset (dataset.hpp:96-97, dataset.cpp:293-307): edge list ("u v" per
 * line, '#' comments, optional "% n <count>" header), features CSV (one row of
 * doubles per vertex) and labels ("vertex,label" per line); from_edge_list
 * (both directions when undirected), normalisation and transpose on `device`.
 * I/O and format errors return CAGNET_ERUNTIME with the reference's message. */
/* Binary dataset cache (the survey's §8(f).2 CSR cache): a finished
 * GraphDataset — normalised adj and adj_t, features, labels, mask — written
 * once ("CAGNETD1" header + raw arrays) and mapped back without generation,
 * parsing or sorting. */
CAGNET_API int cagnet_dataset_save(cagnet_dataset_t d, const char* path);
CAGNET_API int cagnet_dataset_load_binary(int device, const char* path, cagnet_dataset_t* out);
CAGNET_API int cagnet_dataset_load(int device, const char* edges_path, const char* features_path,
                        const char* labels_path, int undirected, cagnet_dataset_t* out);
/* permute_random (dataset.hpp:70-77, dataset.cpp:120-144): relabels vertices
 * by the seeded Fisher-Yates permutation; position i of the result holds the
 * data of original vertex perm[i] (perm_out: n entries, or NULL); adjacency
 * values are moved, never recomputed (bit-exact with the reference). */
CAGNET_API int cagnet_dataset_permute_random(cagnet_dataset_t d, uint64_t seed, int64_t* perm_out,
                                  cagnet_dataset_t* out);
CAGNET_API int cagnet_dataset_info(cagnet_dataset_t d, int64_t* info);
/* which: 0 = adj, 1 = adj_t.  Borrowed handle, owned by the dataset. */
CAGNET_API int cagnet_dataset_csr(cagnet_dataset_t d, int which, cagnet_csr_t* out);
CAGNET_API int cagnet_dataset_features(cagnet_dataset_t d, float* out /* n x f, host */);
CAGNET_API int cagnet_dataset_labels(cagnet_dataset_t d, int64_t* out);
CAGNET_API int cagnet_dataset_free(cagnet_dataset_t d);

/* from_edge_list (csr.cpp:79-92): canonical unit-valued CSR of the m (u, v)
 * pairs (duplicates collapse; undirected adds (v, u) for u != v), sorted and
 * deduplicated on the GPU. */
CAGNET_API int cagnet_csr_from_edge_list(int device, int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                                         int undirected, cagnet_csr_t* out);

/* --- model (gnn.hpp:29-42) --------------------------------------------------- */
/* init_glorot (gnn.cpp:24-44): fp64 weights for every layer, concatenated
 * (layer l is dims[l] x dims[l+1], row major), from one seeded generator. */
CAGNET_API int cagnet_init_glorot(const int64_t* dims, int ndims, uint64_t seed, double* weights);

/* --- training (dist.hpp:43-150) --------------------------------------------- */
/* NCCL bootstrap: rank 0 creates the id, the launcher broadcasts its 128 bytes. */
CAGNET_API int cagnet_comm_unique_id(uint8_t* out128);
/* In-process world (replaces SimRuntime::run's thread-per-rank world,
 * runtime.cpp:270-285): `ranks` ranks as host threads of this process, all on
 * `device`, exchanging data through device memory with the same device-flag
 * protocol as the NVLink peer-memory exchange.  The 128-byte id it writes is
 * passed to cagnet_trainer_create like an NCCL id (one trainer per rank, each
 * driven from its own thread).  Used where the GPUs are fewer than the ranks. */
CAGNET_API int cagnet_comm_local_id(int ranks, int device, uint8_t* out128);
/* Fails every pending and future wait of a local world (a rank that raised
 * must release its peers, like the reference's SimError propagation). */
CAGNET_API int cagnet_comm_local_abort(const uint8_t* id128, const char* why);

/* Creates rank `rank` of Strategy{kind, ranks, repl, block} on the dataset's
 * device.  dims[ndims] are the layer widths; weights are the fp64 Glorot
 * weights concatenated layer by layer (gnn.hpp:29-35), rounded to fp32 on
 * device.  nccl_id may be NULL when ranks == 1. */
CAGNET_API int cagnet_trainer_create(cagnet_dataset_t data, const int64_t* dims, int ndims,
                          const double* weights, double learning_rate, int kind, int ranks,
                          int repl, int block, int rank, const uint8_t* nccl_id,
                          cagnet_trainer_t* out);
/* Trainer::distribute (dist.hpp:87): per-rank CSR blocks and H0 tiles, on device. */
CAGNET_API int cagnet_trainer_distribute(cagnet_trainer_t t);
/* Trainer::forward_layer (1-based l) and Trainer::epoch (dist_common.cpp:97-100). */
CAGNET_API int cagnet_trainer_forward_layer(cagnet_trainer_t t, int l);
CAGNET_API int cagnet_trainer_epoch(cagnet_trainer_t t, double* loss);
CAGNET_API int cagnet_trainer_run_epochs(cagnet_trainer_t t, int epochs, double* losses);
/* Queues one epoch without waiting (losses stay on the device until read). */
CAGNET_API int cagnet_trainer_epoch_async(cagnet_trainer_t t);
/* Every epoch loss so far (waits for queued epochs); count = total epochs. */
CAGNET_API int cagnet_trainer_losses(cagnet_trainer_t t, double* out, int cap, int* count);
/* Blocks until all work queued by this rank has finished. */
CAGNET_API int cagnet_trainer_sync(cagnet_trainer_t t);
/* tile_rows / tile_cols / tile_owner (dist.hpp:96-101): out = {r0, r1, c0, c1, owner} */
CAGNET_API int cagnet_trainer_tile(cagnet_trainer_t t, int rank, int64_t width, int64_t* out);
/* Local tiles of h[layer] (0 = features .. L-1 = log-probabilities) and g[idx]
 * (idx 0..L-2), downloaded as fp32 rows x cols (dense, ld = cols). */
CAGNET_API int cagnet_trainer_h_tile(cagnet_trainer_t t, int layer, float* out);
CAGNET_API int cagnet_trainer_g_tile(cagnet_trainer_t t, int idx, float* out);
/* Replicated weights / weight gradients of layer l (dims[l] x dims[l+1]). */
CAGNET_API int cagnet_trainer_weight(cagnet_trainer_t t, int l, float* out);
CAGNET_API int cagnet_trainer_y(cagnet_trainer_t t, int l, float* out);
/* Local partition structure: part index within this rank's a_parts/at_parts
 * (which 0 = A, 1 = A^T).  shape = {n_rows, n_cols, nnz}. */
CAGNET_API int cagnet_trainer_num_parts(cagnet_trainer_t t, int* out);
CAGNET_API int cagnet_trainer_part(cagnet_trainer_t t, int which, int part, cagnet_csr_t* out);
/* shape3 = {n_rows, n_cols, nnz} of a part without copying it. */
CAGNET_API int cagnet_trainer_part_shape(cagnet_trainer_t t, int which, int part, int64_t* shape3);
/* Per-category device time of the last epoch in ms: [spmm, gemm, elementwise,
 * dbcast, sbcast, reduce, allgather, epoch_total] and per-category NCCL bytes
 * received by this rank per the reference ledger conventions
 * (runtime.cpp:142-184) accumulated since creation: [dbcast, sbcast, reduce, allgather]. */
CAGNET_API int cagnet_trainer_stats(cagnet_trainer_t t, double* ms8, uint64_t* words_received4);
/* Reference-ledger counters of this rank (ledger.hpp:41-47), 4 categories
 * [dbcast, sbcast, reduce, allgather] x {messages, words_sent, words_received,
 * payload_words, calls}. */
CAGNET_API int cagnet_trainer_ledger(cagnet_trainer_t t, uint64_t* out20);
/* Enable/disable per-category CUDA-event timing (adds event records; default off). */
CAGNET_API int cagnet_trainer_set_timing(cagnet_trainer_t t, int on);
/* Trainer options: "reassociate" (1 = narrow-first propagation Aᵀ(H W) when
 * f_out < f_in, Tᵀ G backward when f_out > f_in; same products, narrower panels),
 * "timing" (per-launch CUDA-event profile), "fuse" (SpMM row epilogues: 0/1/2),
 * "graph" (CUDA-graph epochs), "resident_sparse" (2D/3D tiles kept in HBM),
 * "p2p" (1D stage panels through NVLink peer memory), "overlap" (1D peer-memory
 * stages: own vertex block SpMM while the pushes fly), "pipeline" (1D peer-memory
 * stages with >= 32 MB slots: per-destination pushes, per-block SpMMs as slots land).  Set before distribute()
 * for resident_sparse / p2p / overlap. */
CAGNET_API int cagnet_trainer_set_option(cagnet_trainer_t t, const char* name, int64_t value);
/* Per-launch CUDA-event profile, aggregated by kernel name (e.g. "spmm_f602"):
 * out4 = {launches, total_ms, algorithmic_bytes, flops} (SURVEY §8(d) byte model). */
CAGNET_API int cagnet_trainer_profile_count(cagnet_trainer_t t, int* n);
CAGNET_API int cagnet_trainer_profile_entry(cagnet_trainer_t t, int i, char* name, int cap,
                                            double* out4);
CAGNET_API int cagnet_trainer_profile_reset(cagnet_trainer_t t);
/* One epoch from HOST buffers (the end-to-end call): H2D of this rank's
 * feature tile (dense rows x cols fp32, pinned for full speed) and label rows,
 * the epoch, D2H of the loss (blocking). */
CAGNET_API int cagnet_trainer_step_host(cagnet_trainer_t t, const float* x_tile,
                                        const int32_t* labels_tile, double* loss);
/* --- collective seams: RankContext (runtime.hpp:55-96) ----------------------
 * One rank's communicator for the groups of Strategy{kind, ranks, repl}'s
 * process grid (grid.hpp:44-81): NCCL with ncclCommSplit per group when id128
 * came from cagnet_comm_unique_id, the in-process world when it came from
 * cagnet_comm_local_id (NULL when ranks == 1).  Buffers are device memory;
 * `stream` is a cudaStream_t (all collectives of one communicator on one
 * stream, like NCCL).  Every call meters the reference ledger's counters;
 * singleton groups short-circuit and meter nothing (runtime.cpp:142-184). */
typedef struct cagnet_comm_s* cagnet_comm_t;
#define CAGNET_GROUP_WORLD 0
#define CAGNET_GROUP_ROW 1
#define CAGNET_GROUP_COL 2
#define CAGNET_GROUP_FIBER 3
#define CAGNET_DTYPE_F32 0
#define CAGNET_DTYPE_F64 1
#define CAGNET_DTYPE_I32 2
#define CAGNET_DTYPE_I64 3
/* category: 0 dbcast, 1 sbcast, 2 reduce, 3 allgather (ledger.hpp:27-33) */
CAGNET_API int cagnet_comm_create(int kind, int ranks, int repl, int rank, const uint8_t* id128,
                                  int device, cagnet_comm_t* out);
/* Members (global ranks, ascending) of this rank's group `which`. */
CAGNET_API int cagnet_comm_group(cagnet_comm_t c, int which, int* members, int* size);
/* broadcast (runtime.hpp:64-65): `count` elements in place. */
CAGNET_API int cagnet_comm_bcast(cagnet_comm_t c, int which, int root_rank, void* buf, int64_t count,
                                 int dtype, int category, void* stream);
/* broadcast_csr (runtime.hpp:66-67): the three CSR arrays of the root; ledger payload = nnz. */
CAGNET_API int cagnet_comm_bcast_csr(cagnet_comm_t c, int which, int root_rank, int64_t* row_ptr,
                                     int64_t n_rows, int32_t* col_idx, float* vals, int64_t nnz,
                                     int category, void* stream);
/* all_reduce / all_reduce_scalar (runtime.hpp:69-73): in-place sum, f32 or f64. */
CAGNET_API int cagnet_comm_allreduce(cagnet_comm_t c, int which, void* buf, int64_t count, int dtype,
                                     int category, void* stream);
/* reduce_scatter_rows (runtime.hpp:75-79): send is sum(row_counts) x cols
 * (dense); member m receives its row_counts[m] x cols block of the sum. */
CAGNET_API int cagnet_comm_reduce_scatter_rows(cagnet_comm_t c, int which, const float* send, float* recv,
                                               const int64_t* row_counts, int64_t cols, int category,
                                               void* stream);
/* all_gather_rows (runtime.hpp:81-83): member m contributes row_counts[m] x
 * cols rows; recv = the blocks concatenated in member order. */
CAGNET_API int cagnet_comm_allgather_rows(cagnet_comm_t c, int which, const float* send, float* recv,
                                          const int64_t* row_counts, int64_t cols, int category,
                                          void* stream);
/* Ledger counters of this rank, as cagnet_trainer_ledger. */
CAGNET_API int cagnet_comm_ledger(cagnet_comm_t c, uint64_t* out20);
CAGNET_API int cagnet_comm_free(cagnet_comm_t c);

/* --- run_distributed → DistOutcome (dist.hpp:138-150, dist_common.cpp:117-222) ---
 * The whole distributed run on the device path: one host thread per rank
 * (SimRuntime::run's thread-per-rank model), each rank a Trainer on its GPU,
 * then the outcome assembled on the host with the reference's bitwise replica
 * checks (replica divergence -> CAGNET_ERUNTIME, message as the reference).
 * backend: CAGNET_BACKEND_AUTO (NCCL with one GPU per rank when there are at
 * least `ranks` GPUs, else the in-process world on the dataset's GPU),
 * _NCCL or _LOCAL.  The dataset is read-only and shared; the NCCL backend
 * copies it to each rank's GPU. */
typedef struct cagnet_outcome_s* cagnet_outcome_t;
#define CAGNET_BACKEND_AUTO 0
#define CAGNET_BACKEND_NCCL 1
#define CAGNET_BACKEND_LOCAL 2
#define CAGNET_OPT_REASSOCIATE 1u           /* narrow-first propagation (extension) */
#define CAGNET_OPT_NO_GRAPH 2u              /* eager epochs instead of CUDA-graph replays */
#define CAGNET_OPT_NO_RESIDENT_SPARSE 4u    /* 2D/3D: the reference's per-stage sparse broadcasts */
#define CAGNET_OPT_NO_P2P 8u                /* 1D: NCCL all-gather instead of peer-memory pushes */
#define CAGNET_OPT_FUSE0 16u                /* no fused SpMM row epilogues */
#define CAGNET_OPT_FUSE2 32u                /* fused epilogues incl. the dense W transforms */
#define CAGNET_OPT_OVERLAP 64u              /* 1D peer memory: own-block SpMM during the pushes */
#define CAGNET_OPT_PIPELINE 128u            /* 1D peer memory: per-destination pipelined stages */
CAGNET_API int cagnet_run_distributed(cagnet_dataset_t data, const int64_t* dims, int ndims,
                                      const double* weights, double learning_rate, int kind,
                                      int ranks, int repl, int block, int epochs, int backend,
                                      uint32_t options, cagnet_outcome_t* out);
/* out8 = {n, ndims, epochs, ranks, backend used, #prereduction totals,
 *         last epoch device time in microseconds (max over ranks), 0}. */
CAGNET_API int cagnet_outcome_info(cagnet_outcome_t o, int64_t* out8);
CAGNET_API int cagnet_outcome_losses(cagnet_outcome_t o, double* out /* epochs */);
CAGNET_API int cagnet_outcome_h_final(cagnet_outcome_t o, double* out /* n x dims[L-1] */);
CAGNET_API int cagnet_outcome_g(cagnet_outcome_t o, int l, double* out /* n x dims[l+1] */);
CAGNET_API int cagnet_outcome_y(cagnet_outcome_t o, int l, double* out /* dims[l] x dims[l+1] */);
CAGNET_API int cagnet_outcome_weight(cagnet_outcome_t o, int l, double* out /* dims[l] x dims[l+1] */);
/* rank's ledger: [dbcast, sbcast, reduce, allgather] x {messages, words_sent,
 * words_received, payload_words, calls} (ledger.hpp:41-47). */
CAGNET_API int cagnet_outcome_ledger(cagnet_outcome_t o, int rank, uint64_t* out20);
CAGNET_API int cagnet_outcome_prereduction_totals(cagnet_outcome_t o, uint64_t* out);
CAGNET_API int cagnet_outcome_memory_peaks(cagnet_outcome_t o, uint64_t* out /* ranks */);
CAGNET_API int cagnet_outcome_free(cagnet_outcome_t o);

/* --- analytic communication model (cost.hpp:27-115, cost.cpp:48-161) ---------
 * params6 = {n, nnz, f, layers, ranks, repl}.  out6 = {words, messages, term0,
 * term1, term2, #terms} per rank per epoch; terms: 1D {embedding_broadcast,
 * weight_gradient_reduce}, 1.5D {embedding_broadcast, partial_reduce}, 2D
 * {dense_panels, sparse_panels, weight_gradient_gather}, 3D {sparse_panels,
 * dense_panels}.  Invalid shapes -> CAGNET_EINVAL with the reference's message. */
CAGNET_API int cagnet_cost_predict(int kind, const int64_t* params6, int64_t* out6);
CAGNET_API int cagnet_cost_ceil_lg(int64_t p, int64_t* out);
CAGNET_API int cagnet_cost_2d_rect_layer(const int64_t* params6, int64_t p_rows, int64_t p_cols,
                                         double alpha, double beta, double* out);
/* out4 = {serial, repl15d, repl15d_single_adj, split3d_peak} words. */
CAGNET_API int cagnet_cost_memory(int64_t n, int64_t nnz, int64_t f, int64_t fmax, int64_t dims,
                                  int64_t repl, int64_t ranks, int64_t* out4);
/* compare_cost: ledgers = ranks x 20 counters (cagnet_*_ledger layout) of a
 * run of `epochs` epochs.  out4 = {predicted_words, extra_words,
 * measured_words, ratio}; flags3 = {exact, degenerate, within_band}. */
CAGNET_API int cagnet_cost_compare(int kind, const int64_t* params6, const uint64_t* ledgers, int ranks,
                                   int epochs, double* out4, int* flags3);

/* Pipelined end-to-end steps: prefetch_host queues the H2D copies of a later
 * step's inputs (same layout as step_host; host buffers pinned for full
 * speed, and left untouched until the step consumes them) on a copy stream
 * and returns at once; step_prefetched consumes the oldest staged inputs,
 * runs the epoch and returns its loss (blocking).  Step k+1's copies overlap
 * step k's epoch; at most two steps staged ahead. */
CAGNET_API int cagnet_trainer_prefetch_host(cagnet_trainer_t t, const float* x_tile,
                                            const int32_t* labels_tile);
CAGNET_API int cagnet_trainer_step_prefetched(cagnet_trainer_t t, double* loss);

/* Total hot-path kernel launches issued by this library so far. */
CAGNET_API int cagnet_kernel_launches(uint64_t* out);
/* The compute stream the trainer launches on (a cudaStream_t). */
CAGNET_API int cagnet_trainer_stream(cagnet_trainer_t t, void** out);
CAGNET_API int cagnet_trainer_free(cagnet_trainer_t t);

#ifdef __cplusplus
}
#endif

#endif /* CAGNET_B200_H */
