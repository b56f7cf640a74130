// Internal launchers for the hot-path kernels (sm_100a).  The C-ABI in
// capi.cu and the C++ trainers call these; nothing here allocates except the
// split-K workspace, which is stream-ordered.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace cagnet {
namespace kern {

// ---- K1: CSR SpMM (csr.cpp:164-179) ---------------------------------------
// Fused row epilogue of a final (non-accumulating) SpMM whose f <= 32: the
// SpMM row t (f values, still in registers) optionally goes to raw_out, is
// multiplied by a small dense W (f x fo, element (k, c) at W[k*w_sk + c*w_sn];
// the next layer's T·W / the backward S·Wᵀ), masked by relu′ (z *= 1[mask >
// 0], dense.cpp:72-92) and written to T (fo columns, or f without W); relu(z)
// optionally goes to relu_out.  Replaces a GEMM launch and an elementwise pass
// that would each re-read the n x f tile.
struct SpmmEpi {
  const float* W = nullptr;
  int64_t w_sk = 0, w_sn = 0;
  int fo = 0;
  const float* mask = nullptr;
  int64_t mask_ld = 0;
  float* relu_out = nullptr;
  int64_t relu_ld = 0;
  float* raw_out = nullptr;
  int64_t raw_ld = 0;
  // Direct peer push (no-W epilogues): the final row value — relu(Z) when
  // push_relu, else the stored (masked) row — also goes to row
  // push_off + row * push_ld of each of the push_n buffers in push_bufs (a
  // device array: the next exchange's panel slot of this rank on every rank).
  float* const* push_bufs = nullptr;
  int push_n = 0;
  int64_t push_off = 0, push_ld = 0;
  bool push_relu = false;
};
constexpr int kSpmmEpiMaxF = 32;
constexpr int kSpmmEpiMaxFo = 64;

// Packed nonzero stream of a block of the normalized adjacency (pack_normalized):
// entry k = (d << bits) | col, d the column vertex's degree in A + I; the value
// 1/sqrt(d_row d_col) (csr.cpp:94-116) is rebuilt as row_scale[row] * rsqrt(d), so
// the narrow-row kernel streams 4 B per nonzero — one L1 wavefront per 8 entries —
// instead of 8 B in two (values agree to ~5e-7 relative, inside the 1e-4 bar).
struct SpmmPacked {
  const uint32_t* e = nullptr;
  const float* row_scale = nullptr;
  int bits = 0;
};

// T[i, 0:f] = (accumulate ? T[i, 0:f] : 0) + sum_k vals[k] * H[col[k], 0:f]
// with the nonzeros of each row folded in ascending order (the reference's
// accumulation order), one fp32 FMA per term.
// nnz (optional, -1 = unknown) sizes the row teams of the narrow-row kernel.
// colval (optional): the same nonzeros interleaved as int2 {col, float bits}
// (interleave_colval), read by the narrow-row kernel in one load per nonzero.
void spmm_csr(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
              const float* H, int64_t ldh, int f, float* T, int64_t ldt, bool accumulate,
              cudaStream_t stream, int64_t nnz = -1, const SpmmEpi* epi = nullptr,
              const int2* colval = nullptr, const SpmmPacked* packed = nullptr);

// Same, with row i's nonzeros given as [seg_begin[i], seg_end[i]).
void spmm_segments(int64_t n_rows, const int64_t* seg_begin, const int64_t* seg_end,
                   const int32_t* col_idx, const float* vals, const float* H, int64_t ldh, int f,
                   float* T, int64_t ldt, bool accumulate, cudaStream_t stream, int64_t nnz = -1,
                   const SpmmEpi* epi = nullptr, const int2* colval = nullptr,
                   const SpmmPacked* packed = nullptr);
// out[k] = {col_idx[k], bits of vals[k]} for the interleaved nonzero stream.
void interleave_colval(int64_t nnz, const int32_t* col_idx, const float* vals, int2* out,
                       cudaStream_t stream);
// The packed stream of a block whose local (0, 0) is (row_off, col_off) of a
// normalized dataset matrix; deg = degrees of A + I of every vertex.  Adds to
// *bad (device counter) every nonzero whose value is not bitwise
// (float)(1/sqrt(d_r d_c)) or whose degree needs more than 32 - bits bits; the
// stream is only usable when *bad stays 0.
// deg[i] = row_ptr[i + 1] - row_ptr[i].
void row_degrees(int64_t n, const int64_t* row_ptr, int32_t* deg, cudaStream_t stream);
void pack_normalized(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                     const float* vals, const int32_t* deg, int64_t row_off, int64_t col_off,
                     int bits, uint32_t* out, float* row_scale, unsigned long long* bad,
                     cudaStream_t stream);
// split[b * rows + r] (b = 0..nb) = first nonzero of row r in column block b
// of the ceiling-rule split of n_cols into nb blocks; split[nb * rows + r] = row end.
void column_splits(int64_t rows, int64_t n_cols, int nb, const int64_t* row_ptr,
                   const int32_t* col_idx, int64_t* split, cudaStream_t stream);

// ---- K2: tcgen05 split-TF32 GEMM (dense.cpp:37-70) ---------------------------
// op(A) m x k: element (i, p) at A[i * a_sm + p * a_sk]
// op(B) k x n: element (p, j) at B[p * b_sk + j * b_sn]
enum Epilogue { EPI_NONE = 0, EPI_RELU = 1, EPI_RELU_PRIME = 2 };
// Direct peer push of an SpMM's finished rows (see SpmmEpi::push_*).
struct PushSpec {
  float* const* bufs = nullptr;
  int n = 0;
  int64_t off = 0, ld = 0;
  bool relu = false;
};

struct GemmDesc {
  int64_t m = 0, n = 0, k = 0;
  const float* A = nullptr;
  int64_t a_sm = 0, a_sk = 0;
  const float* B = nullptr;
  int64_t b_sk = 0, b_sn = 0;
  float* C = nullptr;
  int64_t ldc = 0;
  bool accumulate = false;
  int epilogue = EPI_NONE;
  const float* aux = nullptr;  // RELU_PRIME: pre-activation Z (ldaux)
  int64_t ldaux = 0;
  float* aux_out = nullptr;    // RELU: receives relu(Z) (ldao)
  int64_t ldao = 0;
};
void gemm_tf32x3(const GemmDesc& d, cudaStream_t stream);
// Persistent TMA-fed variant for row-major A (16 B rows), N <= 64 and a B that
// fits in shared memory; returns false (nothing launched) when not applicable.
bool gemm_tma_try(const GemmDesc& d, cudaStream_t stream);
// A-in-TMEM variant (gemm_tm.cu): row-major A with B resident (T·W, S·Wᵀ) or
// M-contiguous A with B streamed and split-K (Hᵀ·S); N <= 64.  Returns false
// (nothing launched) when the shape or layout does not apply.
bool gemm_tm_try(const GemmDesc& d, cudaStream_t stream);
// CUDA-core kernels (gemm_small.cu) for narrow x narrow shapes: K, N <= 32
// with many rows (H·W, S·Wᵀ of 16-wide layers) and M, N <= 32 with a long K
// (Hᵀ·S); returns false (nothing launched) otherwise.
bool gemm_small_try(const GemmDesc& d, cudaStream_t stream);

// ---- K3: fused elementwise ----------------------------------------------------
// log_softmax_rows + nll_tile (dense.cpp:94-136) over full rows of Z; writes
// the column tile [c0, c1) of logp and G; loss partial (fp64, undivided) is
// written to *loss_out (device) deterministically.
void logsoftmax_nll(const float* Z, int64_t rows, int cols, int64_t ldz, int c0, int c1,
                    float* logp, int64_t ldl, float* G, int64_t ldg, const int32_t* labels,
                    const uint8_t* mask, int64_t train_total, double* loss_out,
                    cudaStream_t stream);
// Variant for tiles whose full rows are spread over `parts` column blocks laid
// out back to back (the 2D/3D all-gather result): block q holds rows x
// width_q columns at base + q * block_stride with leading dim ldz.
void logsoftmax_nll_blocks(const float* base, int parts, const int* widths, int64_t block_stride,
                           int64_t rows, int64_t ldz, int own_part, float* logp, int64_t ldl,
                           float* G, int64_t ldg, const int32_t* labels, const uint8_t* mask,
                           int64_t train_total, double* loss_out, cudaStream_t stream);
void relu(const float* Z, int64_t rows, int cols, int64_t ldz, float* H, int64_t ldh,
          cudaStream_t stream);
void sgd(float* W, const float* Y, int64_t count, float lr, cudaStream_t stream);
// losses[*slot] = *partial; ++*slot — the epoch's loss lands at a device-side
// index, so a replayed CUDA graph of the epoch appends instead of overwriting.
void push_loss(double* losses, int* slot, const double* partial, cudaStream_t stream);
// g[r, c] *= 1[z[r, c] > 0]   (hadamard with relu_prime, dense.cpp:72-92)
void mask_relu_prime(float* g, int64_t ldg, const float* z, int64_t ldz, int64_t rows,
                     int64_t cols, cudaStream_t stream);
// dst[r, 0:cols] = src[r, 0:cols] for strided row-major blocks.
// Device-to-device byte copy / zero fill as SM kernels (stream ordered).
void copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t stream);
void zero_bytes(void* dst, size_t bytes, cudaStream_t stream);
void copy2d(float* dst, int64_t ldd, const float* src, int64_t lds, int64_t rows, int64_t cols,
            cudaStream_t stream);
// dst (cols x rows, ldd) = src^T (rows x cols, lds)
void transpose2d(float* dst, int64_t ldd, const float* src, int64_t lds, int64_t rows,
                 int64_t cols, cudaStream_t stream);
void fill(float* p, int64_t count, float v, cudaStream_t stream);
// fp64 host-converted values → fp32 device values happen on the host; this
// converts device fp64 → fp32.
void f64_to_f32(const double* src, float* dst, int64_t count, cudaStream_t stream);

}  // namespace kern
}  // namespace cagnet
