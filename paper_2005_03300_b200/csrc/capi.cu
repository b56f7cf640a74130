// extern "C" boundary of libcagnet_b200.so (include/cagnet_b200.h).  Every
// entry point validates shapes on the host, maps C++ exceptions to status
// codes and records the message per thread.
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/cagnet_b200.h"
#include <cmath>

#include "kernels.cuh"
#include "rng.hpp"
#include "cost.hpp"
#include "run.hpp"
#include "trainer.hpp"

struct cagnet_csr_s {
  cagnet::DeviceCsr csr;
  bool borrowed = false;
};
struct cagnet_dataset_s {
  std::unique_ptr<cagnet::DeviceDataset> data;
  cagnet_csr_s adj, adj_t;
};
struct cagnet_comm_s {
  int device = 0;
  int rank = 0;
  cagnet::ProcessGrid grid;
  std::unique_ptr<cagnet::Comm> comm;
  cagnet::DevBuf<float> pad_send, pad_recv;
};
struct cagnet_outcome_s {
  cagnet::DistOutcome o;
};
struct cagnet_trainer_s {
  std::unique_ptr<cagnet::Trainer> t;
  bool timing = false;
};

namespace {

// Process defaults, applied before the first CUDA call of this process when
// the library is loaded first (an explicit setting always wins):
// * a hardware work queue per stream for up to 16 streams of in-process ranks;
// * module data loaded eagerly: with lazy loading, the first launch of a
//   kernel may wait for a context-wide synchronisation, which never comes
//   while a rank sharing the GPU spins in a device-side wait for this rank
//   (the CUDA programming guide's documented lazy-loading hazard for kernels
//   that wait on each other; CUDA_MODULE_DATA_LOADING=EAGER is its remedy).
__attribute__((constructor)) void cagnet_env_defaults() {
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
  setenv("CUDA_MODULE_DATA_LOADING", "EAGER", 0);
}

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return CAGNET_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return CAGNET_EINVAL;
  } catch (const cagnet::CudaError& e) {
    g_error = e.what();
    return CAGNET_ECUDA;
  } catch (const cagnet::NcclError& e) {
    g_error = e.what();
    return CAGNET_ENCCL;
  } catch (const std::exception& e) {
    g_error = e.what();
    return CAGNET_ERUNTIME;
  }
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void set_device(int device) { CG_CUDA(cudaSetDevice(device)); }

cagnet::Strategy make_strategy(int kind, int ranks, int repl, int block) {
  if (kind < 0 || kind > 3) throw std::invalid_argument("strategy: unknown kind");
  cagnet::Strategy s;
  s.kind = static_cast<cagnet::StrategyKind>(kind);
  s.ranks = ranks;
  s.repl = repl;
  s.block = block;
  return s;
}

}  // namespace

extern "C" {

const char* cagnet_last_error(void) { return g_error.c_str(); }
int cagnet_version(void) { return 1; }

int cagnet_device_count(int* out) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

// ---- host-only partition geometry -----------------------------------------------
int cagnet_block_range(int64_t n, int parts, int idx, int64_t* out2) {
  return guarded([&] {
    const cagnet::BlockRange r = cagnet::block_range(n, parts, idx);
    out2[0] = r.begin;
    out2[1] = r.end;
  });
}

int cagnet_grid_shape(int kind, int ranks, int repl, int* out4) {
  return guarded([&] {
    const cagnet::ProcessGrid g = cagnet::ProcessGrid::make(make_strategy(kind, ranks, repl, 0));
    out4[0] = static_cast<int>(g.kind());
    out4[1] = g.rows();
    out4[2] = g.cols();
    out4[3] = g.layers();
  });
}

int cagnet_grid_group(int kind, int ranks, int repl, int rank, int which, int* members, int* count) {
  return guarded([&] {
    const cagnet::ProcessGrid g = cagnet::ProcessGrid::make(make_strategy(kind, ranks, repl, 0));
    cagnet::require(rank >= 0 && rank < g.ranks(), "grid_group: rank outside the grid");
    const cagnet::Group* grp = nullptr;
    switch (which) {
      case 0: grp = &g.world(); break;
      case 1: grp = &g.row_group(rank); break;
      case 2: grp = &g.col_group(rank); break;
      case 3: grp = &g.fiber_group(rank); break;
      default: throw std::invalid_argument("grid_group: which must be 0..3");
    }
    *count = static_cast<int>(grp->size());
    for (size_t i = 0; i < grp->size(); ++i) members[i] = grp->members[i];
  });
}

int cagnet_tile_geometry(int kind, int ranks, int repl, int64_t n, int rank, int64_t width,
                         int64_t* out5) {
  return guarded([&] {
    const cagnet::ProcessGrid g = cagnet::ProcessGrid::make(make_strategy(kind, ranks, repl, 0));
    cagnet::require(rank >= 0 && rank < g.ranks(), "tile_geometry: rank outside the grid");
    const cagnet::BlockRange r = cagnet::tile_rows_of(g, n, rank), c = cagnet::tile_cols_of(g, rank, width);
    out5[0] = r.begin;
    out5[1] = r.end;
    out5[2] = c.begin;
    out5[3] = c.end;
    out5[4] = cagnet::tile_owner_of(g, rank);
  });
}

// ---- kernel seams --------------------------------------------------------------
int cagnet_spmm_csr_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const float* vals, const float* H, int64_t ldh,
                        int32_t f, float* T, int64_t ldt, int accumulate, void* stream) {
  return guarded([&] {
    cagnet::require(n_rows >= 0 && n_cols >= 0 && nnz >= 0 && f >= 0, "spmm: negative shape");
    cagnet::require(ldh >= f && ldt >= f, "spmm: leading dimension smaller than f");
    cagnet::require(n_rows == 0 || (row_ptr && T), "spmm: null row_ptr or output");
    cagnet::require(nnz == 0 || (col_idx && vals && H), "spmm: null input arrays");
    cagnet::kern::spmm_csr(n_rows, row_ptr, col_idx, vals, H, ldh, f, T, ldt, accumulate != 0,
                           as_stream(stream), nnz);
  });
}

int cagnet_spmm_fused_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                          const int32_t* col_idx, const float* vals, const float* H, int64_t ldh,
                          int32_t f, const float* W, int64_t w_sk, int64_t w_sn, int32_t fo,
                          const float* mask, int64_t mask_ld, float* T, int64_t ldt,
                          float* relu_out, int64_t relu_ld, float* raw_out, int64_t raw_ld,
                          void* stream) {
  return guarded([&] {
    cagnet::require(n_rows >= 0 && n_cols >= 0 && nnz >= 0 && f >= 0, "spmm_fused: negative shape");
    cagnet::require(f <= cagnet::kern::kSpmmEpiMaxF, "spmm_fused: f > 32");
    const int32_t width = W ? fo : f;
    cagnet::require(!W || (fo > 0 && fo <= cagnet::kern::kSpmmEpiMaxFo), "spmm_fused: fo outside [1, 64]");
    cagnet::require(ldh >= f && ldt >= width, "spmm_fused: leading dimension too small");
    cagnet::require(!mask || mask_ld >= width, "spmm_fused: mask leading dimension too small");
    cagnet::require(!relu_out || relu_ld >= width, "spmm_fused: relu_out leading dimension too small");
    cagnet::require(!raw_out || raw_ld >= f, "spmm_fused: raw_out leading dimension too small");
    cagnet::require(n_rows == 0 || (row_ptr && T), "spmm_fused: null row_ptr or output");
    cagnet::require(nnz == 0 || (col_idx && vals && H), "spmm_fused: null input arrays");
    cagnet::kern::SpmmEpi e;
    e.W = W;
    e.w_sk = w_sk;
    e.w_sn = w_sn;
    e.fo = W ? fo : 0;
    e.mask = mask;
    e.mask_ld = mask_ld;
    e.relu_out = relu_out;
    e.relu_ld = relu_ld;
    e.raw_out = raw_out;
    e.raw_ld = raw_ld;
    cagnet::kern::spmm_csr(n_rows, row_ptr, col_idx, vals, H, ldh, f, T, ldt, false,
                           as_stream(stream), nnz, &e);
  });
}

int cagnet_gemm_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
                    const float* B, int64_t ldb, float* C, int64_t ldc, int accumulate, int epilogue,
                    const float* aux, int64_t ldaux, float* aux_out, int64_t ldao, void* stream) {
  return guarded([&] {
    cagnet::require(m >= 0 && n >= 0 && k >= 0, "gemm: negative shape");
    cagnet::require(ldc >= n, "gemm: accumulator leading dimension smaller than n");
    cagnet::require(lda >= (ta ? m : k) && ldb >= (tb ? k : n), "gemm: operand leading dimension too small");
    cagnet::require(epilogue >= 0 && epilogue <= 2, "gemm: unknown epilogue");
    cagnet::require(epilogue != CAGNET_EPI_RELU_PRIME || (aux && ldaux >= n), "gemm: relu' epilogue needs aux");
    cagnet::kern::GemmDesc d;
    d.m = m;
    d.n = n;
    d.k = k;
    d.A = A;
    d.a_sm = ta ? 1 : lda;
    d.a_sk = ta ? lda : 1;
    d.B = B;
    d.b_sk = tb ? 1 : ldb;
    d.b_sn = tb ? ldb : 1;
    d.C = C;
    d.ldc = ldc;
    d.accumulate = accumulate != 0;
    d.epilogue = epilogue;
    d.aux = aux;
    d.ldaux = ldaux;
    d.aux_out = aux_out;
    d.ldao = ldao;
    cagnet::kern::gemm_tf32x3(d, as_stream(stream));
  });
}

int cagnet_logsoftmax_nll_f32(const float* Z, int64_t rows, int32_t cols, int64_t ldz, int32_t c0,
                              int32_t c1, float* logp, int64_t ldl, float* G, int64_t ldg,
                              const int32_t* labels, const uint8_t* mask, int64_t train_total,
                              double* loss_partial, void* stream) {
  return guarded([&] {
    if (cols == 0) throw std::invalid_argument("log_softmax_rows: zero columns");
    cagnet::require(0 <= c0 && c0 <= c1 && c1 <= cols, "nll_tile: column tile outside the row");
    cagnet::require(!G || labels, "nll_tile: labels required for the gradient");
    if (G && train_total == 0) throw std::invalid_argument("nll_tile: empty training set");
    cagnet::kern::logsoftmax_nll(Z, rows, cols, ldz, c0, c1, logp, ldl, G, ldg, labels, mask,
                                 train_total, loss_partial, as_stream(stream));
  });
}

int cagnet_relu_f32(const float* Z, int64_t rows, int32_t cols, int64_t ldz, float* H, int64_t ldh,
                    void* stream) {
  return guarded([&] { cagnet::kern::relu(Z, rows, cols, ldz, H, ldh, as_stream(stream)); });
}

int cagnet_sgd_f32(float* W, const float* Y, int64_t count, float lr, void* stream) {
  return guarded([&] { cagnet::kern::sgd(W, Y, count, lr, as_stream(stream)); });
}

// ---- device CSR -------------------------------------------------------------------
int cagnet_csr_upload(int device, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                      const int64_t* col_idx, const double* vals, cagnet_csr_t* out) {
  return guarded([&] {
    set_device(device);
    auto h = std::make_unique<cagnet_csr_s>();
    h->csr = cagnet::upload_csr(n_rows, n_cols, row_ptr, col_idx, vals, nullptr);
    *out = h.release();
  });
}

int cagnet_csr_shape(cagnet_csr_t a, int64_t* shape) {
  return guarded([&] {
    shape[0] = a->csr.n_rows;
    shape[1] = a->csr.n_cols;
    shape[2] = a->csr.nnz;
  });
}

int cagnet_csr_download(cagnet_csr_t a, int64_t* row_ptr, int64_t* col_idx, float* vals) {
  return guarded([&] {
    const cagnet::DeviceCsr& c = a->csr;
    set_device(c.device);
    if (row_ptr)
      CG_CUDA(cudaMemcpy(row_ptr, c.row_ptr.get(), (c.n_rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (col_idx && c.nnz) {
      std::vector<int32_t> tmp(static_cast<size_t>(c.nnz));
      CG_CUDA(cudaMemcpy(tmp.data(), c.col_idx.get(), c.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
      for (int64_t k = 0; k < c.nnz; ++k) col_idx[k] = tmp[static_cast<size_t>(k)];
    }
    if (vals && c.nnz)
      CG_CUDA(cudaMemcpy(vals, c.vals.get(), c.nnz * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

int cagnet_csr_device_ptrs(cagnet_csr_t a, const int64_t** row_ptr, const int32_t** col_idx,
                           const float** vals) {
  return guarded([&] {
    if (row_ptr) *row_ptr = a->csr.row_ptr.get();
    if (col_idx) *col_idx = a->csr.col_idx.get();
    if (vals) *vals = a->csr.vals.get();
  });
}

int cagnet_csr_free(cagnet_csr_t a) {
  return guarded([&] {
    if (a && !a->borrowed) {
      set_device(a->csr.device);
      delete a;
    }
  });
}

int cagnet_er_generate(int device, int64_t n, double degree, uint64_t seed, cagnet_csr_t* out) {
  return guarded([&] {
    set_device(device);
    auto h = std::make_unique<cagnet_csr_s>();
    h->csr = cagnet::er_generate_device(n, degree, seed, nullptr);
    *out = h.release();
  });
}

int cagnet_csr_normalize(cagnet_csr_t raw, cagnet_csr_t* out) {
  return guarded([&] {
    set_device(raw->csr.device);
    auto h = std::make_unique<cagnet_csr_s>();
    h->csr = cagnet::normalize_device(raw->csr, nullptr, nullptr);
    *out = h.release();
  });
}

int cagnet_csr_transpose(cagnet_csr_t a, cagnet_csr_t* out) {
  return guarded([&] {
    set_device(a->csr.device);
    auto h = std::make_unique<cagnet_csr_s>();
    h->csr = cagnet::transpose_device(a->csr, nullptr);
    *out = h.release();
  });
}

int cagnet_csr_extract_block(cagnet_csr_t a, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                             cagnet_csr_t* out) {
  return guarded([&] {
    set_device(a->csr.device);
    auto h = std::make_unique<cagnet_csr_s>();
    h->csr = cagnet::extract_block_device(a->csr, r0, r1, c0, c1, nullptr);
    *out = h.release();
  });
}

// ---- datasets -------------------------------------------------------------------------
static void wrap_dataset(cagnet_dataset_s* d) {
  // Borrowed CSR views share the dataset's device buffers without copying.
  d->adj.borrowed = d->adj_t.borrowed = true;
}

int cagnet_dataset_generate(int device, int64_t n, double degree, int64_t num_features,
                            int64_t num_classes, uint64_t seed_graph, uint64_t seed_features,
                            uint64_t seed_labels, int generator, cagnet_dataset_t* out) {
  return guarded([&] {
    cagnet::require(generator == CAGNET_GEN_REFERENCE || generator == CAGNET_GEN_SKIP,
                    "dataset: unknown generator");
    set_device(device);
    auto d = std::make_unique<cagnet_dataset_s>();
    d->data = cagnet::dataset_generate(n, degree, num_features, num_classes, seed_graph,
                                       seed_features, seed_labels, generator);
    wrap_dataset(d.get());
    *out = d.release();
  });
}

int cagnet_dataset_make(int device, int64_t n, const int64_t* raw_row_ptr, const int64_t* raw_col_idx,
                        const double* features, int64_t f, const int64_t* labels, const uint8_t* mask,
                        int64_t num_classes, cagnet_dataset_t* out) {
  return guarded([&] {
    set_device(device);
    auto d = std::make_unique<cagnet_dataset_s>();
    d->data = cagnet::dataset_make(n, raw_row_ptr, raw_col_idx, features, f, labels, mask, num_classes);
    wrap_dataset(d.get());
    *out = d.release();
  });
}

int cagnet_dataset_load(int device, const char* edges_path, const char* features_path,
                        const char* labels_path, int undirected, cagnet_dataset_t* out) {
  return guarded([&] {
    cagnet::require(edges_path && features_path && labels_path, "load_dataset: null path");
    auto d = std::make_unique<cagnet_dataset_s>();
    // Parsing (and its errors) happens on the host before the device is touched.
    d->data = cagnet::dataset_load(edges_path, features_path, labels_path, undirected != 0, device);
    wrap_dataset(d.get());
    *out = d.release();
  });
}

int cagnet_dataset_save(cagnet_dataset_t d, const char* path) {
  return guarded([&] {
    cagnet::require(d && path, "save_dataset: null argument");
    cagnet::dataset_save(*d->data, path);
  });
}

int cagnet_dataset_load_binary(int device, const char* path, cagnet_dataset_t* out) {
  return guarded([&] {
    cagnet::require(path != nullptr, "load_dataset_binary: null path");
    auto d = std::make_unique<cagnet_dataset_s>();
    d->data = cagnet::dataset_load_binary(path, device);
    wrap_dataset(d.get());
    *out = d.release();
  });
}

int cagnet_csr_from_edge_list(int device, int64_t n, int64_t m, const int64_t* u, const int64_t* v, int undirected,
                              cagnet_csr_t* out) {
  return guarded([&] {
    cagnet::require(m == 0 || (u && v), "from_edge_list: null edge arrays");
    set_device(device);
    auto h = std::make_unique<cagnet_csr_s>();
    cudaStream_t s;
    CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      h->csr = cagnet::csr_from_edges_device(n, m, u, v, undirected != 0, s);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    CG_CUDA(cudaStreamDestroy(s));
    *out = h.release();
  });
}

int cagnet_dataset_permute_random(cagnet_dataset_t d, uint64_t seed, int64_t* perm_out,
                                  cagnet_dataset_t* out) {
  return guarded([&] {
    set_device(d->data->device);
    auto p = std::make_unique<cagnet_dataset_s>();
    std::vector<int64_t> perm;
    p->data = cagnet::dataset_permute(*d->data, seed, &perm);
    if (perm_out && !perm.empty()) std::memcpy(perm_out, perm.data(), perm.size() * sizeof(int64_t));
    wrap_dataset(p.get());
    *out = p.release();
  });
}

int cagnet_dataset_info(cagnet_dataset_t d, int64_t* info) {
  return guarded([&] {
    info[0] = d->data->n;
    info[1] = d->data->adj.nnz;
    info[2] = d->data->f;
    info[3] = d->data->num_classes;
    info[4] = d->data->train_count;
  });
}

int cagnet_dataset_csr(cagnet_dataset_t d, int which, cagnet_csr_t* out) {
  return guarded([&] {
    cagnet::require(which == 0 || which == 1, "dataset_csr: which must be 0 (adj) or 1 (adj_t)");
    cagnet_csr_s* h = which == 0 ? &d->adj : &d->adj_t;
    // Shallow view: copy the metadata, alias the buffers (never freed through the view).
    const cagnet::DeviceCsr& src = which == 0 ? d->data->adj : d->data->adj_t;
    h->csr.device = src.device;
    h->csr.n_rows = src.n_rows;
    h->csr.n_cols = src.n_cols;
    h->csr.nnz = src.nnz;
    h->csr.row_ptr.ptr = src.row_ptr.ptr;
    h->csr.row_ptr.count = 0;
    h->csr.col_idx.ptr = src.col_idx.ptr;
    h->csr.col_idx.count = 0;
    h->csr.vals.ptr = src.vals.ptr;
    h->csr.vals.count = 0;
    *out = h;
  });
}

int cagnet_dataset_features(cagnet_dataset_t d, float* out) {
  return guarded([&] {
    const cagnet::DeviceDataset& ds = *d->data;
    set_device(ds.device);
    if (ds.n && ds.f)
      CG_CUDA(cudaMemcpy2D(out, ds.f * sizeof(float), ds.features.get(), ds.ldf * sizeof(float),
                           ds.f * sizeof(float), ds.n, cudaMemcpyDeviceToHost));
  });
}

int cagnet_dataset_labels(cagnet_dataset_t d, int64_t* out) {
  return guarded([&] {
    const cagnet::DeviceDataset& ds = *d->data;
    set_device(ds.device);
    std::vector<int32_t> tmp(static_cast<size_t>(ds.n));
    if (ds.n) CG_CUDA(cudaMemcpy(tmp.data(), ds.labels.get(), ds.n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < ds.n; ++i) out[i] = tmp[static_cast<size_t>(i)];
  });
}

int cagnet_dataset_free(cagnet_dataset_t d) {
  return guarded([&] {
    if (!d) return;
    set_device(d->data->device);
    // Detach the borrowed views before the owning buffers go away.
    for (cagnet_csr_s* v : {&d->adj, &d->adj_t}) {
      v->csr.row_ptr.ptr = nullptr;
      v->csr.col_idx.ptr = nullptr;
      v->csr.vals.ptr = nullptr;
    }
    delete d;
  });
}

// ---- training ---------------------------------------------------------------------------
int cagnet_init_glorot(const int64_t* dims, int ndims, uint64_t seed, double* weights) {
  return guarded([&] {
    if (ndims < 2)
      throw std::invalid_argument("init_glorot: need at least two layer dims, got " + std::to_string(ndims));
    for (int l = 0; l < ndims; ++l)
      if (dims[l] <= 0) throw std::invalid_argument("init_glorot: zero-width layer");
    // gnn.cpp:24-44: one generator, layers in order, row-major fill,
    // U(-b, b) with b = sqrt(6 / (f_in + f_out)).
    cagnet::Xoshiro rng(seed);
    int64_t off = 0;
    for (int l = 0; l + 1 < ndims; ++l) {
      const double bound = std::sqrt(6.0 / static_cast<double>(dims[l] + dims[l + 1]));
      for (int64_t e = 0; e < dims[l] * dims[l + 1]; ++e) weights[off + e] = rng.uniform(-bound, bound);
      off += dims[l] * dims[l + 1];
    }
  });
}

int cagnet_comm_unique_id(uint8_t* out128) {
  return guarded([&] {
    ncclUniqueId id;
    CG_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int cagnet_comm_local_id(int ranks, int device, uint8_t* out128) {
  return guarded([&] {
    cagnet::require(out128 != nullptr, "comm_local_id: null output");
    int n = 0;
    CG_CUDA(cudaGetDeviceCount(&n));
    cagnet::require(device >= 0 && device < n, "comm_local_id: device " + std::to_string(device) +
                                                   " outside [0, " + std::to_string(n) + ")");
    cagnet::LocalId id;
    cagnet::LocalWorld::create(ranks, device, &id);
    std::memcpy(out128, &id, sizeof(id));
  });
}

int cagnet_comm_local_abort(const uint8_t* id128, const char* why) {
  return guarded([&] {
    cagnet::require(cagnet::is_local_id(id128), "comm_local_abort: not a local world id");
    cagnet::LocalId id;
    std::memcpy(&id, id128, sizeof(id));
    cagnet::LocalWorld::abort_id(id, why ? why : "aborted by a rank");
  });
}

// ---- collective seams (RankContext, runtime.hpp:55-96) ---------------------------------
namespace {
const cagnet::Group& comm_group(cagnet_comm_t c, int which) {
  switch (which) {
    case CAGNET_GROUP_WORLD: return c->grid.world();
    case CAGNET_GROUP_ROW: return c->grid.row_group(c->rank);
    case CAGNET_GROUP_COL: return c->grid.col_group(c->rank);
    case CAGNET_GROUP_FIBER: return c->grid.fiber_group(c->rank);
    default: throw std::invalid_argument("comm: unknown group " + std::to_string(which));
  }
}
ncclDataType_t nccl_dtype(int dtype) {
  switch (dtype) {
    case CAGNET_DTYPE_F32: return ncclFloat32;
    case CAGNET_DTYPE_F64: return ncclFloat64;
    case CAGNET_DTYPE_I32: return ncclInt32;
    case CAGNET_DTYPE_I64: return ncclInt64;
    default: throw std::invalid_argument("comm: unknown dtype " + std::to_string(dtype));
  }
}
cagnet::Category comm_category(int c) {
  if (c < 0 || c >= cagnet::kNumCategories) throw std::invalid_argument("comm: unknown category");
  return static_cast<cagnet::Category>(c);
}
}  // namespace

int cagnet_comm_create(int kind, int ranks, int repl, int rank, const uint8_t* id128, int device,
                       cagnet_comm_t* out) {
  return guarded([&] {
    set_device(device);
    auto c = std::make_unique<cagnet_comm_s>();
    c->device = device;
    c->rank = rank;
    c->grid = cagnet::ProcessGrid::make(make_strategy(kind, ranks, repl, 0));
    cagnet::require(rank >= 0 && rank < c->grid.ranks(), "comm: rank outside the grid");
    ncclUniqueId id;
    if (id128) std::memcpy(&id, id128, sizeof(id));
    c->comm = std::make_unique<cagnet::Comm>(c->grid, rank, id128 ? &id : nullptr);
    *out = c.release();
  });
}

int cagnet_comm_group(cagnet_comm_t c, int which, int* members, int* size) {
  return guarded([&] {
    const cagnet::Group& g = comm_group(c, which);
    *size = static_cast<int>(g.size());
    if (members)
      for (size_t i = 0; i < g.size(); ++i) members[i] = g.members[i];
  });
}

int cagnet_comm_bcast(cagnet_comm_t c, int which, int root_rank, void* buf, int64_t count, int dtype,
                      int category, void* stream) {
  return guarded([&] {
    set_device(c->device);
    cagnet::require(count >= 0, "broadcast: negative count");
    c->comm->bcast(comm_group(c, which), root_rank, buf, static_cast<size_t>(count), nccl_dtype(dtype),
                   comm_category(category), static_cast<uint64_t>(count), as_stream(stream));
  });
}

int cagnet_comm_bcast_csr(cagnet_comm_t c, int which, int root_rank, int64_t* row_ptr, int64_t n_rows,
                          int32_t* col_idx, float* vals, int64_t nnz, int category, void* stream) {
  return guarded([&] {
    set_device(c->device);
    cagnet::require(n_rows >= 0 && nnz >= 0, "broadcast_csr: negative size");
    c->comm->bcast_csr(comm_group(c, which), root_rank, row_ptr, n_rows, col_idx, vals, nnz,
                       comm_category(category), as_stream(stream));
  });
}

int cagnet_comm_allreduce(cagnet_comm_t c, int which, void* buf, int64_t count, int dtype, int category,
                          void* stream) {
  return guarded([&] {
    set_device(c->device);
    cagnet::require(dtype == CAGNET_DTYPE_F32 || dtype == CAGNET_DTYPE_F64, "all_reduce: f32 or f64 only");
    c->comm->all_reduce(comm_group(c, which), buf, static_cast<size_t>(count), nccl_dtype(dtype),
                        comm_category(category), static_cast<uint64_t>(count), as_stream(stream));
  });
}

// Member-ordered row blocks of unequal heights move through equal padded
// slots (max rows per member), like every other reduce-scatter / all-gather
// of the library; the ledger counts the logical rows x cols per member.
int cagnet_comm_reduce_scatter_rows(cagnet_comm_t c, int which, const float* send, float* recv,
                                    const int64_t* row_counts, int64_t cols, int category, void* stream) {
  return guarded([&] {
    set_device(c->device);
    const cagnet::Group& g = comm_group(c, which);
    const cagnet::Category cat = comm_category(category);
    const cudaStream_t s = as_stream(stream);
    const int m = g.index_of(c->rank);
    int64_t maxr = 0, off = 0, mine_off = 0;
    std::vector<uint64_t> words;
    for (size_t q = 0; q < g.size(); ++q) {
      cagnet::require(row_counts[q] >= 0, "reduce_scatter_rows: negative row count");
      maxr = std::max(maxr, row_counts[q]);
      words.push_back(static_cast<uint64_t>(row_counts[q] * cols));
    }
    const size_t slot = static_cast<size_t>(maxr * cols);
    c->pad_send.resize(std::max<size_t>(slot * g.size(), 1));
    c->pad_recv.resize(std::max<size_t>(slot, 1));
    cagnet::kern::zero_bytes(c->pad_send.get(), slot * g.size() * sizeof(float), s);
    for (size_t q = 0; q < g.size(); ++q) {
      if (static_cast<int>(q) == m) mine_off = off;
      cagnet::kern::copy_bytes(c->pad_send.get() + q * slot, send + off * cols,
                               static_cast<size_t>(row_counts[q] * cols) * sizeof(float), s);
      off += row_counts[q];
    }
    (void)mine_off;
    if (g.size() == 1) {
      cagnet::kern::copy_bytes(recv, send, static_cast<size_t>(row_counts[0] * cols) * sizeof(float), s);
      return;
    }
    c->comm->reduce_scatter(g, c->pad_send.get(), c->pad_recv.get(), slot, ncclFloat32, cat, words, s);
    cagnet::kern::copy_bytes(recv, c->pad_recv.get(), static_cast<size_t>(row_counts[m] * cols) * sizeof(float), s);
  });
}

int cagnet_comm_allgather_rows(cagnet_comm_t c, int which, const float* send, float* recv,
                               const int64_t* row_counts, int64_t cols, int category, void* stream) {
  return guarded([&] {
    set_device(c->device);
    const cagnet::Group& g = comm_group(c, which);
    const cagnet::Category cat = comm_category(category);
    const cudaStream_t s = as_stream(stream);
    const int m = g.index_of(c->rank);
    int64_t maxr = 0;
    std::vector<uint64_t> words;
    for (size_t q = 0; q < g.size(); ++q) {
      cagnet::require(row_counts[q] >= 0, "all_gather_rows: negative row count");
      maxr = std::max(maxr, row_counts[q]);
      words.push_back(static_cast<uint64_t>(row_counts[q] * cols));
    }
    if (g.size() == 1) {
      cagnet::kern::copy_bytes(recv, send, static_cast<size_t>(row_counts[0] * cols) * sizeof(float), s);
      return;
    }
    const size_t slot = static_cast<size_t>(maxr * cols);
    c->pad_send.resize(std::max<size_t>(slot, 1));
    c->pad_recv.resize(std::max<size_t>(slot * g.size(), 1));
    cagnet::kern::copy_bytes(c->pad_send.get(), send, static_cast<size_t>(row_counts[m] * cols) * sizeof(float), s);
    c->comm->all_gather(g, c->pad_send.get(), c->pad_recv.get(), slot, ncclFloat32, cat, words, s);
    int64_t off = 0;
    for (size_t q = 0; q < g.size(); ++q) {
      cagnet::kern::copy_bytes(recv + off * cols, c->pad_recv.get() + q * slot,
                               static_cast<size_t>(row_counts[q] * cols) * sizeof(float), s);
      off += row_counts[q];
    }
  });
}

int cagnet_comm_ledger(cagnet_comm_t c, uint64_t* out20) {
  return guarded([&] {
    for (int k = 0; k < cagnet::kNumCategories; ++k) {
      const cagnet::CommCounter& x = c->comm->counter(static_cast<cagnet::Category>(k));
      const uint64_t v[5] = {x.messages, x.words_sent, x.words_received, x.payload_words, x.calls};
      std::memcpy(out20 + 5 * k, v, sizeof(v));
    }
  });
}

int cagnet_comm_free(cagnet_comm_t c) {
  return guarded([&] {
    if (c) set_device(c->device);
    delete c;
  });
}

// ---- analytic communication model ------------------------------------------------------
namespace {
cagnet::cost::Params cost_params(const int64_t* p6) {
  cagnet::require(p6 != nullptr, "cost model: null parameters");
  return cagnet::cost::Params{p6[0], p6[1], p6[2], p6[3], p6[4], p6[5]};
}
cagnet::StrategyKind cost_kind(int kind) {
  cagnet::require(kind >= 0 && kind <= 3, "strategy: unknown kind");
  return static_cast<cagnet::StrategyKind>(kind);
}
}  // namespace

int cagnet_cost_predict(int kind, const int64_t* params6, int64_t* out6) {
  return guarded([&] {
    const cagnet::cost::Prediction p = cagnet::cost::predict(cost_kind(kind), cost_params(params6));
    int64_t v[6] = {p.words, p.messages, 0, 0, 0, static_cast<int64_t>(p.terms.size())};
    for (size_t i = 0; i < p.terms.size() && i < 3; ++i) v[2 + i] = p.terms[i].second;
    std::memcpy(out6, v, sizeof(v));
  });
}

int cagnet_cost_ceil_lg(int64_t p, int64_t* out) {
  return guarded([&] { *out = cagnet::cost::ceil_lg(p); });
}

int cagnet_cost_2d_rect_layer(const int64_t* params6, int64_t p_rows, int64_t p_cols, double alpha, double beta,
                              double* out) {
  return guarded([&] { *out = cagnet::cost::rect_layer(cost_params(params6), p_rows, p_cols, alpha, beta); });
}

int cagnet_cost_memory(int64_t n, int64_t nnz, int64_t f, int64_t fmax, int64_t dims, int64_t repl, int64_t ranks,
                       int64_t* out4) {
  return guarded([&] {
    const cagnet::cost::Footprints m = cagnet::cost::footprints(n, nnz, f, fmax, dims, repl, ranks);
    const int64_t v[4] = {m.serial, m.repl15d, m.repl15d_single_adj, m.split3d_peak};
    std::memcpy(out4, v, sizeof(v));
  });
}

int cagnet_cost_compare(int kind, const int64_t* params6, const uint64_t* ledgers, int ranks, int epochs,
                        double* out4, int* flags3) {
  return guarded([&] {
    cagnet::require(ranks >= 1 && ledgers != nullptr, "compare_cost: no ledger");
    uint64_t payload = 0;
    for (int r = 0; r < ranks; ++r)
      for (int c = 0; c < cagnet::kNumCategories; ++c) payload += ledgers[r * 20 + c * 5 + 3];
    const cagnet::cost::Comparison c =
        cagnet::cost::compare(cost_kind(kind), cost_params(params6), payload, ranks, epochs);
    out4[0] = static_cast<double>(c.predicted_words);
    out4[1] = static_cast<double>(c.extra_words);
    out4[2] = c.measured_words;
    out4[3] = c.ratio;
    flags3[0] = c.exact;
    flags3[1] = c.degenerate;
    flags3[2] = c.within_band;
  });
}

int cagnet_run_distributed(cagnet_dataset_t data, const int64_t* dims, int ndims, const double* weights,
                           double learning_rate, int kind, int ranks, int repl, int block, int epochs,
                           int backend, uint32_t options, cagnet_outcome_t* out) {
  return guarded([&] {
    cagnet::require(data && dims && weights && out, "run_distributed: null argument");
    cagnet::require(ndims >= 2, "init_glorot: need at least two layer dims, got " + std::to_string(ndims));
    cagnet::require(backend >= 0 && backend <= 2, "run_distributed: unknown backend");
    set_device(data->data->device);
    cagnet::RunOptions opt;
    opt.reassociate = (options & CAGNET_OPT_REASSOCIATE) != 0;
    opt.graph = (options & CAGNET_OPT_NO_GRAPH) == 0;
    opt.resident_sparse = (options & CAGNET_OPT_NO_RESIDENT_SPARSE) == 0;
    opt.p2p = (options & CAGNET_OPT_NO_P2P) == 0;
    opt.fuse = (options & CAGNET_OPT_FUSE0) ? 0 : (options & CAGNET_OPT_FUSE2) ? 2 : 1;
    opt.overlap = (options & CAGNET_OPT_OVERLAP) != 0;
    opt.pipeline = (options & CAGNET_OPT_PIPELINE) != 0;
    auto o = std::make_unique<cagnet_outcome_s>();
    o->o = cagnet::run_distributed(*data->data, std::vector<int64_t>(dims, dims + ndims), weights, learning_rate,
                                   make_strategy(kind, ranks, repl, block), epochs,
                                   static_cast<cagnet::Backend>(backend), opt);
    *out = o.release();
  });
}

int cagnet_outcome_info(cagnet_outcome_t o, int64_t* out8) {
  return guarded([&] {
    const cagnet::DistOutcome& d = o->o;
    const int64_t v[8] = {d.n, static_cast<int64_t>(d.dims.size()), static_cast<int64_t>(d.losses.size()),
                          d.ranks, d.backend, static_cast<int64_t>(d.prereduction_totals.size()),
                          static_cast<int64_t>(d.epoch_ms * 1000.0), 0};
    std::memcpy(out8, v, sizeof(v));
  });
}

namespace {
void copy_out(const std::vector<double>& v, double* out) {
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(double));
}
const std::vector<double>& layer_of(const std::vector<std::vector<double>>& v, int l) {
  if (l < 0 || l >= static_cast<int>(v.size())) throw std::invalid_argument("outcome: layer index out of range");
  return v[static_cast<size_t>(l)];
}
}  // namespace

int cagnet_outcome_losses(cagnet_outcome_t o, double* out) {
  return guarded([&] { copy_out(o->o.losses, out); });
}
int cagnet_outcome_h_final(cagnet_outcome_t o, double* out) {
  return guarded([&] { copy_out(o->o.h_final, out); });
}
int cagnet_outcome_g(cagnet_outcome_t o, int l, double* out) {
  return guarded([&] { copy_out(layer_of(o->o.g_final, l), out); });
}
int cagnet_outcome_y(cagnet_outcome_t o, int l, double* out) {
  return guarded([&] { copy_out(layer_of(o->o.y_final, l), out); });
}
int cagnet_outcome_weight(cagnet_outcome_t o, int l, double* out) {
  return guarded([&] { copy_out(layer_of(o->o.weights, l), out); });
}
int cagnet_outcome_ledger(cagnet_outcome_t o, int rank, uint64_t* out20) {
  return guarded([&] {
    cagnet::require(rank >= 0 && rank < o->o.ranks, "outcome: rank out of range");
    for (int c = 0; c < cagnet::kNumCategories; ++c)
      for (int f = 0; f < 5; ++f) out20[c * 5 + f] = o->o.ledger[static_cast<size_t>(rank)][c][f];
  });
}
int cagnet_outcome_prereduction_totals(cagnet_outcome_t o, uint64_t* out) {
  return guarded([&] {
    const auto& v = o->o.prereduction_totals;
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(uint64_t));
  });
}
int cagnet_outcome_memory_peaks(cagnet_outcome_t o, uint64_t* out) {
  return guarded([&] {
    const auto& v = o->o.memory_peaks;
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(uint64_t));
  });
}
int cagnet_outcome_free(cagnet_outcome_t o) {
  return guarded([&] { delete o; });
}

int cagnet_trainer_create(cagnet_dataset_t data, const int64_t* dims, int ndims, const double* weights,
                          double learning_rate, int kind, int ranks, int repl, int block, int rank,
                          const uint8_t* nccl_id, cagnet_trainer_t* out) {
  return guarded([&] {
    set_device(data->data->device);
    cagnet::require(ndims >= 2, "init_glorot: need at least two layer dims, got " + std::to_string(ndims));
    ncclUniqueId id;
    if (nccl_id) std::memcpy(&id, nccl_id, sizeof(id));
    auto t = std::make_unique<cagnet_trainer_s>();
    t->t = cagnet::make_trainer(*data->data, std::vector<int64_t>(dims, dims + ndims), weights,
                                learning_rate, make_strategy(kind, ranks, repl, block), rank,
                                nccl_id ? &id : nullptr);
    *out = t.release();
  });
}

int cagnet_trainer_distribute(cagnet_trainer_t t) {
  return guarded([&] {
    set_device(t->t->device());
    t->t->distribute();
  });
}

int cagnet_trainer_forward_layer(cagnet_trainer_t t, int l) {
  return guarded([&] {
    set_device(t->t->device());
    t->t->run_forward_layer(l);
  });
}

int cagnet_trainer_epoch(cagnet_trainer_t t, double* loss) {
  return guarded([&] {
    set_device(t->t->device());
    std::vector<double> l = t->t->run_epochs(1);
    if (loss) *loss = l.empty() ? 0.0 : l.back();
  });
}

int cagnet_trainer_run_epochs(cagnet_trainer_t t, int epochs, double* losses) {
  return guarded([&] {
    set_device(t->t->device());
    if (epochs <= 0) throw std::invalid_argument("run_epochs: epoch count must be positive");
    std::vector<double> l = t->t->run_epochs(epochs);
    if (losses) std::memcpy(losses, l.data(), l.size() * sizeof(double));
  });
}

int cagnet_trainer_epoch_async(cagnet_trainer_t t) {
  return guarded([&] {
    set_device(t->t->device());
    t->t->epoch();
  });
}

int cagnet_trainer_losses(cagnet_trainer_t t, double* out, int cap, int* count) {
  return guarded([&] {
    const std::vector<double>& l = t->t->all_losses();
    *count = static_cast<int>(l.size());
    for (int i = 0; i < cap && i < static_cast<int>(l.size()); ++i) out[i] = l[static_cast<size_t>(i)];
  });
}

int cagnet_trainer_sync(cagnet_trainer_t t) {
  return guarded([&] { t->t->sync(); });
}

int cagnet_trainer_tile(cagnet_trainer_t t, int rank, int64_t width, int64_t* out) {
  return guarded([&] {
    const cagnet::BlockRange r = t->t->tile_rows(rank), c = t->t->tile_cols(rank, width);
    out[0] = r.begin;
    out[1] = r.end;
    out[2] = c.begin;
    out[3] = c.end;
    out[4] = t->t->tile_owner(rank);
  });
}

int cagnet_trainer_h_tile(cagnet_trainer_t t, int layer, float* out) {
  return guarded([&] {
    t->t->sync();
    t->t->h_tile(layer, out);
  });
}
int cagnet_trainer_g_tile(cagnet_trainer_t t, int idx, float* out) {
  return guarded([&] {
    t->t->sync();
    t->t->g_tile(idx, out);
  });
}
int cagnet_trainer_weight(cagnet_trainer_t t, int l, float* out) {
  return guarded([&] {
    t->t->sync();
    t->t->weight(l, out);
  });
}
int cagnet_trainer_y(cagnet_trainer_t t, int l, float* out) {
  return guarded([&] {
    t->t->sync();
    t->t->ygrad(l, out);
  });
}

int cagnet_trainer_num_parts(cagnet_trainer_t t, int* out) {
  return guarded([&] { *out = t->t->num_parts(); });
}

int cagnet_trainer_part_shape(cagnet_trainer_t t, int which, int part, int64_t* shape3) {
  return guarded([&] {
    const cagnet::DeviceCsr& src = t->t->part(which, part);
    shape3[0] = src.n_rows;
    shape3[1] = src.n_cols;
    shape3[2] = src.nnz;
  });
}

int cagnet_trainer_part(cagnet_trainer_t t, int which, int part, cagnet_csr_t* out) {
  return guarded([&] {
    const cagnet::DeviceCsr& src = t->t->part(which, part);
    auto h = std::make_unique<cagnet_csr_s>();
    h->borrowed = false;
    // Deep copy so the handle can outlive the trainer.
    h->csr.device = src.device;
    h->csr.n_rows = src.n_rows;
    h->csr.n_cols = src.n_cols;
    h->csr.nnz = src.nnz;
    h->csr.row_ptr.resize(static_cast<size_t>(src.n_rows + 1));
    h->csr.col_idx.resize(static_cast<size_t>(src.nnz));
    h->csr.vals.resize(static_cast<size_t>(src.nnz));
    CG_CUDA(cudaMemcpy(h->csr.row_ptr.get(), src.row_ptr.get(), (src.n_rows + 1) * sizeof(int64_t),
                       cudaMemcpyDeviceToDevice));
    if (src.nnz) {
      CG_CUDA(cudaMemcpy(h->csr.col_idx.get(), src.col_idx.get(), src.nnz * sizeof(int32_t),
                         cudaMemcpyDeviceToDevice));
      CG_CUDA(cudaMemcpy(h->csr.vals.get(), src.vals.get(), src.nnz * sizeof(float), cudaMemcpyDeviceToDevice));
    }
    CG_CUDA(cudaStreamSynchronize(nullptr));  // D2D cudaMemcpy returns before it completes
    *out = h.release();
  });
}

int cagnet_trainer_stats(cagnet_trainer_t t, double* ms8, uint64_t* words_received4) {
  return guarded([&] {
    if (ms8) {
      for (int i = 0; i < 8; ++i) ms8[i] = 0.0;
      ms8[7] = t->t->last_epoch_ms();
    }
    if (words_received4)
      for (int c = 0; c < 4; ++c)
        words_received4[c] = t->t->comm().counter(static_cast<cagnet::Category>(c)).words_received;
  });
}

int cagnet_trainer_ledger(cagnet_trainer_t t, uint64_t* out20) {
  return guarded([&] {
    for (int c = 0; c < 4; ++c) {
      const cagnet::CommCounter& k = t->t->comm().counter(static_cast<cagnet::Category>(c));
      out20[5 * c + 0] = k.messages;
      out20[5 * c + 1] = k.words_sent;
      out20[5 * c + 2] = k.words_received;
      out20[5 * c + 3] = k.payload_words;
      out20[5 * c + 4] = k.calls;
    }
  });
}

int cagnet_trainer_set_timing(cagnet_trainer_t t, int on) {
  return guarded([&] {
    t->timing = on != 0;
    t->t->set_timing(on != 0);
  });
}

int cagnet_trainer_set_option(cagnet_trainer_t t, const char* name, int64_t value) {
  return guarded([&] {
    const std::string n(name ? name : "");
    if (n == "reassociate")
      t->t->set_reassociate(value != 0);
    else if (n == "timing")
      t->t->set_timing(value != 0);
    else if (n == "p2p")
      t->t->set_p2p(value != 0);
    else if (n == "overlap")
      t->t->set_overlap(value != 0);
    else if (n == "pipeline")
      t->t->set_pipeline(value != 0);
    else if (n == "resident_sparse")
      t->t->set_resident_sparse(value != 0);
    else if (n == "graph")
      t->t->set_graph(value != 0);
    else if (n == "fuse")
      t->t->set_fuse(static_cast<int>(value));
    else
      throw std::invalid_argument("trainer option: unknown option '" + n + "'");
  });
}

int cagnet_trainer_profile_count(cagnet_trainer_t t, int* n) {
  return guarded([&] { *n = static_cast<int>(t->t->profile().size()); });
}

int cagnet_trainer_profile_entry(cagnet_trainer_t t, int i, char* name, int cap, double* out4) {
  return guarded([&] {
    const auto& p = t->t->profile();
    cagnet::require(i >= 0 && i < static_cast<int>(p.size()), "profile_entry: index out of range");
    const auto& e = p[static_cast<size_t>(i)];
    if (name && cap > 0) {
      std::strncpy(name, e.name.c_str(), static_cast<size_t>(cap - 1));
      name[cap - 1] = 0;
    }
    out4[0] = static_cast<double>(e.launches);
    out4[1] = e.ms;
    out4[2] = e.bytes;
    out4[3] = e.flops;
  });
}

int cagnet_trainer_profile_reset(cagnet_trainer_t t) {
  return guarded([&] { t->t->reset_profile(); });
}

int cagnet_trainer_prefetch_host(cagnet_trainer_t t, const float* x_tile, const int32_t* labels_tile) {
  return guarded([&] {
    cagnet::require(x_tile != nullptr && labels_tile != nullptr, "prefetch_host: null input");
    t->t->prefetch_host(x_tile, labels_tile);
  });
}

int cagnet_trainer_step_prefetched(cagnet_trainer_t t, double* loss) {
  return guarded([&] {
    const double l = t->t->step_prefetched();
    if (loss) *loss = l;
  });
}

int cagnet_trainer_step_host(cagnet_trainer_t t, const float* x_tile, const int32_t* labels_tile,
                             double* loss) {
  return guarded([&] {
    const double l = t->t->step_host(x_tile, labels_tile);
    if (loss) *loss = l;
  });
}

int cagnet_kernel_launches(uint64_t* out) {
  return guarded([&] { *out = cagnet::launch_counter().load(); });
}

int cagnet_trainer_stream(cagnet_trainer_t t, void** out) {
  return guarded([&] { *out = reinterpret_cast<void*>(t->t->stream()); });
}

int cagnet_trainer_free(cagnet_trainer_t t) {
  return guarded([&] { delete t; });
}

}  // extern "C"
