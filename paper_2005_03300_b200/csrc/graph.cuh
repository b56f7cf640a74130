// Device-resident CSR matrices and the CSR/block construction kernels
// (csr.cpp:59-218, dataset.cpp:76-118), all bit-exact in structure with the
// reference; values are the reference fp64 values rounded to fp32.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace cagnet {

struct DeviceCsr {
  int device = 0;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  DevBuf<int64_t> row_ptr;  // n_rows + 1
  DevBuf<int32_t> col_idx;  // nnz
  DevBuf<float> vals;       // nnz
  // Global row / column of local (0, 0) when this is a block of a dataset matrix
  // (extract_block); the packed SpMM stream checks its values against them.
  int64_t row_off = 0, col_off = 0;
};

// csr.cpp:195-218 — every ordered pair (u, v != u) consumes one draw of the
// seeded stream; row u starts at draw u*(n-1).
DeviceCsr er_generate_device(int64_t n, double degree, uint64_t seed, cudaStream_t s);
// O(nnz) ER-shaped generator: per-row independent streams, geometric gaps.
DeviceCsr er_skip_generate_device(int64_t n, double degree, uint64_t seed, cudaStream_t s);
// csr.cpp:94-116.  Optionally returns the row degrees of A+I.
DeviceCsr normalize_device(const DeviceCsr& raw, DevBuf<int32_t>* degree_out, cudaStream_t s);
// csr.cpp:118-138 (values moved, columns sorted).
DeviceCsr transpose_device(const DeviceCsr& a, cudaStream_t s);
// permute_csr, dataset.cpp:49-72: out[i][j] = in[perm[i]][perm[j]] — values
// moved (never recomputed), columns re-sorted per row.  perm / inv are device
// arrays of n = rows = cols entries.
DeviceCsr permute_csr_device(const DeviceCsr& a, const int64_t* perm, const int64_t* inv,
                             cudaStream_t s);
// csr.cpp:140-162.
DeviceCsr extract_block_device(const DeviceCsr& a, int64_t r0, int64_t r1, int64_t c0,
                               int64_t c1, cudaStream_t s);
// Rotated copy for the overlapped 1D stage (strategy_rows.cu): row r keeps its
// nonzeros but starts at the first column >= c0, so the columns in [c0, c1)
// (this rank's own vertex block) come first, then [c1, n), then [0, c0); the
// out CSR shares a's row_ptr, and mid[r] ends the [c0, c1) group.
struct RotatedCsr {
  DevBuf<int32_t> col_idx;
  DevBuf<float> vals;
  DevBuf<int64_t> mid;
};
RotatedCsr rotate_rows_device(const DeviceCsr& a, int64_t c0, int64_t c1, cudaStream_t s);
// Host arrays (int64 indices; fp64 values or NULL = unit) → device.
DeviceCsr upload_csr(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* vals, cudaStream_t s);
// dataset.cpp:92-98 — U[0,1) features, element (i, j) is draw i*f + j.
void random_features_device(int64_t n, int64_t f, uint64_t seed, float* out, int64_t ld,
                            cudaStream_t s);
// Host-side labels (dataset.cpp:100-108) — variable draws per label.
std::vector<int32_t> random_labels_host(int64_t n, int64_t classes, uint64_t seed);

}  // namespace cagnet
