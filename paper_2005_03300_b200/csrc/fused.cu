// K3 — fused elementwise kernels: log_softmax + NLL + gradient, ReLU, SGD and
// the small layout helpers the partition layer needs (strided copies,
// transposes).  All are HBM-streaming kernels.
#include "common.cuh"
#include <map>
#include <mutex>

#include "kernels.cuh"

namespace cagnet {
namespace kern {
namespace {

constexpr int kMaxParts = 8;

struct RowBlocks {
  const float* base;
  int64_t block_stride;  // elements between column blocks
  int64_t ld;
  int parts;
  int widths[kMaxParts];
  int offs[kMaxParts + 1];
};

__device__ __forceinline__ float load_col(const RowBlocks& b, int64_t r, int j) {
  int q = 0;
#pragma unroll
  for (int t = 1; t < kMaxParts; ++t)
    if (t < b.parts && j >= b.offs[t]) q = t;
  return b.base[q * b.block_stride + r * b.ld + (j - b.offs[q])];
}

// One warp per row.  Reference order: mx = max_j z; s = sum_j exp(z - mx);
// lse = log(s); logp = z - mx - lse (dense.cpp:94-107); grad on training rows
// = exp(logp) / |T| minus 1/|T| at the label; loss partial += -logp[y]
// (dense.cpp:109-136), accumulated in fp64.
__global__ void __launch_bounds__(256)
    logsoftmax_nll_kernel(const RowBlocks zb, int64_t rows, int c0, int c1, float* logp,
                          int64_t ldl, float* G, int64_t ldg, const int32_t* __restrict__ labels,
                          const uint8_t* __restrict__ mask, double inv_total,
                          double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int warps_per_block = blockDim.x >> 5;
  const int cols = zb.offs[zb.parts];
  double loss = 0.0;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps_per_block + (threadIdx.x >> 5);
       r < rows; r += static_cast<int64_t>(gridDim.x) * warps_per_block) {
    float mx = -INFINITY;
    for (int j = lane; j < cols; j += 32) mx = fmaxf(mx, load_col(zb, r, j));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float s = 0.f;
    for (int j = lane; j < cols; j += 32) s += expf(load_col(zb, r, j) - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float lse = logf(s);
    const bool train = mask == nullptr || mask[r] != 0;
    const int y = labels ? labels[r] : -1;
    const float inv = static_cast<float>(inv_total);
    for (int j = c0 + lane; j < c1; j += 32) {
      const float lp = (load_col(zb, r, j) - mx) - lse;
      if (logp) logp[r * ldl + (j - c0)] = lp;
      if (G) {
        float g = 0.f;
        if (train) {
          g = expf(lp) * inv;
          if (j == y) g -= inv;
        }
        G[r * ldg + (j - c0)] = g;
      }
      if (train && j == y) loss += -static_cast<double>(lp);
    }
  }
  // Deterministic block reduction in fp64.
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, o);
  if (lane == 0) red[threadIdx.x >> 5] = loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < warps_per_block; ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

// Row-team variant for the common case (cols <= TPR * NV): TPR lanes own a
// row, each keeps its NV columns in registers, so the row is read once and
// every reduction is a few xor shuffles; one warp covers 32 / TPR rows and
// the grid covers every row (no serial row loop per warp).
template <int TPR, int NV, bool SINGLE>
__global__ void __launch_bounds__(256)
    logsoftmax_nll_rows_kernel(const RowBlocks zb, int64_t rows, int c0, int c1, float* logp,
                               int64_t ldl, float* G, int64_t ldg,
                               const int32_t* __restrict__ labels,
                               const uint8_t* __restrict__ mask, double inv_total,
                               double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int sub = lane % TPR;
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / TPR;
  const int cols = zb.offs[zb.parts];
  const bool live = r < rows;
  float z[NV];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = sub + i * TPR;
    z[i] = -INFINITY;
    if (live && j < cols) z[i] = SINGLE ? zb.base[r * zb.ld + j] : load_col(zb, r, j);
    mx = fmaxf(mx, z[i]);
  }
#pragma unroll
  for (int o = TPR / 2; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (sub + i * TPR < cols) s += expf(z[i] - mx);
#pragma unroll
  for (int o = TPR / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  double loss = 0.0;
  if (live) {
    const float lse = logf(s);
    const bool train = mask == nullptr || mask[r] != 0;
    const int y = labels ? labels[r] : -1;
    const float inv = static_cast<float>(inv_total);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int j = sub + i * TPR;
      if (j >= c0 && j < c1) {
        const float lp = (z[i] - mx) - lse;
        if (logp) logp[r * ldl + (j - c0)] = lp;
        if (G) {
          float g = 0.f;
          if (train) {
            g = expf(lp) * inv;
            if (j == y) g -= inv;
          }
          G[r * ldg + (j - c0)] = g;
        }
        if (train && j == y) loss = -static_cast<double>(lp);
      }
    }
  }
  // Deterministic block reduction in fp64.
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, o);
  if (lane == 0) red[threadIdx.x >> 5] = loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int count,
                                    double* out) {
  __shared__ double red[256];
  double t = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) t += partials[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

template <int TPR>
void launch_lsm_rows(const RowBlocks& zb, int64_t rows, int c0, int c1, float* logp, int64_t ldl,
                     float* G, int64_t ldg, const int32_t* labels, const uint8_t* mask,
                     double inv, double* partials, int64_t blocks, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(blocks);
  if (zb.parts == 1)
    logsoftmax_nll_rows_kernel<TPR, 8, true><<<g, 256, 0, s>>>(zb, rows, c0, c1, logp, ldl, G, ldg,
                                                               labels, mask, inv, partials);
  else
    logsoftmax_nll_rows_kernel<TPR, 8, false><<<g, 256, 0, s>>>(zb, rows, c0, c1, logp, ldl, G, ldg,
                                                                labels, mask, inv, partials);
}

void launch_lsm(const RowBlocks& zb, int64_t rows, int c0, int c1, float* logp, int64_t ldl,
                float* G, int64_t ldg, const int32_t* labels, const uint8_t* mask,
                int64_t train_total, double* loss_out, cudaStream_t s) {
  const int cols = zb.offs[zb.parts];
  const double inv = train_total > 0 ? 1.0 / static_cast<double>(train_total) : 0.0;
  const int tpr = cols <= 64 ? 8 : 32;
  int64_t blocks;
  if (cols <= 8 * 32) {
    blocks = ceil_div64(rows > 0 ? rows : 1, 256 / tpr);
  } else {
    const int sms = num_sms(current_device());
    blocks = ceil_div64(rows > 0 ? rows : 1, 8);
    if (blocks > 4 * sms) blocks = 4 * sms;
  }
  double* partials = static_cast<double*>(stream_scratch(s, blocks * sizeof(double)));
  if (cols <= 8 * 32) {
    if (tpr == 8)
      launch_lsm_rows<8>(zb, rows, c0, c1, logp, ldl, G, ldg, labels, mask, inv, partials, blocks, s);
    else
      launch_lsm_rows<32>(zb, rows, c0, c1, logp, ldl, G, ldg, labels, mask, inv, partials, blocks, s);
  } else {
    logsoftmax_nll_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        zb, rows, c0, c1, logp, ldl, G, ldg, labels, mask, inv, partials);
  }
  CG_LAUNCH_CHECK();
  if (loss_out) {
    sum_partials_kernel<<<1, 256, 0, s>>>(partials, static_cast<int>(blocks), loss_out);
    CG_LAUNCH_CHECK();
  }
}

// (row, col) of flat element e; 32-bit division whenever the extent allows.
__device__ __forceinline__ void split_index(int64_t e, int64_t cols, int64_t total, int64_t& r,
                                            int64_t& c) {
  if (total < (int64_t{1} << 31)) {
    const uint32_t q = static_cast<uint32_t>(e) / static_cast<uint32_t>(cols);
    r = q;
    c = static_cast<uint32_t>(e) - q * static_cast<uint32_t>(cols);
  } else {
    r = e / cols;
    c = e % cols;
  }
}

__global__ void relu_kernel(const float* __restrict__ Z, int64_t rows, int cols, int64_t ldz,
                            float* __restrict__ H, int64_t ldh) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r, c;
    split_index(e, cols, total, r, c);
    const float z = Z[r * ldz + c];
    H[r * ldh + c] = z > 0.f ? z : 0.f;
  }
}

__global__ void sgd_kernel(float* __restrict__ W, const float* __restrict__ Y, int64_t count,
                           float lr) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    W[e] -= lr * Y[e];
}

__global__ void copy2d_kernel(float* __restrict__ dst, int64_t ldd, const float* __restrict__ src,
                              int64_t lds, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r, c;
    split_index(e, cols, total, r, c);
    dst[r * ldd + c] = src[r * lds + c];
  }
}

__global__ void transpose2d_kernel(float* __restrict__ dst, int64_t ldd,
                                   const float* __restrict__ src, int64_t lds, int64_t rows,
                                   int64_t cols) {
  __shared__ float tile[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][i];
  }
}

__global__ void mask_relu_prime_kernel(float* __restrict__ g, int64_t ldg,
                                       const float* __restrict__ z, int64_t ldz, int64_t rows,
                                       int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r, c;
    split_index(e, cols, total, r, c);
    const float x = g[r * ldg + c];
    g[r * ldg + c] = z[r * ldz + c] > 0.f ? x : x * 0.f;
  }
}

__global__ void fill_kernel(float* p, int64_t count, float v) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[e] = v;
}

__global__ void f64_to_f32_kernel(const double* __restrict__ s, float* __restrict__ d,
                                  int64_t count) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[e] = static_cast<float>(s[e]);
}

__global__ void push_loss_kernel(double* losses, int* slot, const double* partial) {
  losses[*slot] = *partial;
  *slot += 1;
}

unsigned grid_for(int64_t total) {
  const int sms = num_sms(current_device());
  int64_t b = ceil_div64(total > 0 ? total : 1, 256);
  if (b > 8 * sms) b = 8 * sms;
  return static_cast<unsigned>(b);
}

}  // namespace

void logsoftmax_nll(const float* Z, int64_t rows, int cols, int64_t ldz, int c0, int c1,
                    float* logp, int64_t ldl, float* G, int64_t ldg, const int32_t* labels,
                    const uint8_t* mask, int64_t train_total, double* loss_out,
                    cudaStream_t stream) {
  RowBlocks zb{};
  zb.base = Z;
  zb.block_stride = 0;
  zb.ld = ldz;
  zb.parts = 1;
  zb.widths[0] = cols;
  zb.offs[0] = 0;
  zb.offs[1] = cols;
  launch_lsm(zb, rows, c0, c1, logp, ldl, G, ldg, labels, mask, train_total, loss_out, stream);
}

void logsoftmax_nll_blocks(const float* base, int parts, const int* widths, int64_t block_stride,
                           int64_t rows, int64_t ldz, int own_part, float* logp, int64_t ldl,
                           float* G, int64_t ldg, const int32_t* labels, const uint8_t* mask,
                           int64_t train_total, double* loss_out, cudaStream_t stream) {
  require(parts >= 1 && parts <= kMaxParts, "logsoftmax_nll_blocks: 1..8 column blocks");
  RowBlocks zb{};
  zb.base = base;
  zb.block_stride = block_stride;
  zb.ld = ldz;
  zb.parts = parts;
  zb.offs[0] = 0;
  for (int q = 0; q < parts; ++q) {
    zb.widths[q] = widths[q];
    zb.offs[q + 1] = zb.offs[q] + widths[q];
  }
  for (int q = parts; q < kMaxParts; ++q) zb.offs[q + 1] = zb.offs[parts];
  launch_lsm(zb, rows, zb.offs[own_part], zb.offs[own_part + 1], logp, ldl, G, ldg, labels, mask,
             train_total, loss_out, stream);
}

void relu(const float* Z, int64_t rows, int cols, int64_t ldz, float* H, int64_t ldh,
          cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  relu_kernel<<<grid_for(rows * cols), 256, 0, stream>>>(Z, rows, cols, ldz, H, ldh);
  CG_LAUNCH_CHECK();
}

void sgd(float* W, const float* Y, int64_t count, float lr, cudaStream_t stream) {
  if (count <= 0) return;
  sgd_kernel<<<grid_for(count), 256, 0, stream>>>(W, Y, count, lr);
  CG_LAUNCH_CHECK();
}

void push_loss(double* losses, int* slot, const double* partial, cudaStream_t stream) {
  push_loss_kernel<<<1, 1, 0, stream>>>(losses, slot, partial);
  CG_LAUNCH_CHECK();
}

void mask_relu_prime(float* g, int64_t ldg, const float* z, int64_t ldz, int64_t rows,
                     int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  mask_relu_prime_kernel<<<grid_for(rows * cols), 256, 0, stream>>>(g, ldg, z, ldz, rows, cols);
  CG_LAUNCH_CHECK();
}

void copy2d(float* dst, int64_t ldd, const float* src, int64_t lds, int64_t rows, int64_t cols,
            cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  if (ldd == cols && lds == cols) {
    copy_bytes(dst, src, static_cast<size_t>(rows * cols) * sizeof(float), stream);
    return;
  }
  copy2d_kernel<<<grid_for(rows * cols), 256, 0, stream>>>(dst, ldd, src, lds, rows, cols);
  CG_LAUNCH_CHECK();
}

void transpose2d(float* dst, int64_t ldd, const float* src, int64_t lds, int64_t rows,
                 int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid(static_cast<unsigned>(ceil_div64(cols, 32)), static_cast<unsigned>(ceil_div64(rows, 32)));
  transpose2d_kernel<<<grid, dim3(32, 8), 0, stream>>>(dst, ldd, src, lds, rows, cols);
  CG_LAUNCH_CHECK();
}

namespace {
// Byte copies / zero fills as SM kernels, not copy-engine or runtime memset
// operations: on a GPU shared by several in-process ranks a copy-engine
// queue entry that waits for its stream can block other ranks' copies behind
// it (the waits of comm_local.cu would then never be satisfied).
__global__ void copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
__global__ void copy1_kernel(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
__global__ void zero16_kernel(uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = make_uint4(0, 0, 0, 0);
}
__global__ void zero1_kernel(unsigned char* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = 0;
}
unsigned copy_grid(size_t n) {
  const size_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 2048 ? (b ? b : 1) : 2048);
}
}  // namespace

void copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0 || dst == src) return;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) % 16 == 0) {
    copy16_kernel<<<copy_grid(bytes / 16), 256, 0, stream>>>(static_cast<uint4*>(dst),
                                                            static_cast<const uint4*>(src), bytes / 16);
  } else {
    copy1_kernel<<<copy_grid(bytes), 256, 0, stream>>>(static_cast<unsigned char*>(dst),
                                                       static_cast<const unsigned char*>(src), bytes);
  }
  CG_LAUNCH_CHECK();
}

void zero_bytes(void* dst, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return;
  if ((reinterpret_cast<uintptr_t>(dst) | bytes) % 16 == 0)
    zero16_kernel<<<copy_grid(bytes / 16), 256, 0, stream>>>(static_cast<uint4*>(dst), bytes / 16);
  else
    zero1_kernel<<<copy_grid(bytes), 256, 0, stream>>>(static_cast<unsigned char*>(dst), bytes);
  CG_LAUNCH_CHECK();
}

void fill(float* p, int64_t count, float v, cudaStream_t stream) {
  if (count <= 0) return;
  fill_kernel<<<grid_for(count), 256, 0, stream>>>(p, count, v);
  CG_LAUNCH_CHECK();
}

void f64_to_f32(const double* src, float* dst, int64_t count, cudaStream_t stream) {
  if (count <= 0) return;
  f64_to_f32_kernel<<<grid_for(count), 256, 0, stream>>>(src, dst, count);
  CG_LAUNCH_CHECK();
}

}  // namespace kern

void* stream_scratch(cudaStream_t s, size_t bytes) {
  struct Entry {
    void* p = nullptr;
    size_t bytes = 0;
  };
  static std::mutex mu;
  // Keyed by device too: a destroyed stream's handle can come back for a
  // stream of another device, and pool memory is not accessible across devices.
  static std::map<std::pair<int, cudaStream_t>, Entry> cache;
  int dev = 0;
  CG_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_pair(dev, s);
  {
    std::lock_guard<std::mutex> lk(mu);
    const Entry& e = cache[key];
    if (e.bytes >= bytes && e.p) return e.p;
  }
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CG_CUDA(cudaStreamIsCapturing(s, &st));
  if (st != cudaStreamCaptureStatusNone)
    throw std::logic_error("stream_scratch: workspace growth inside a graph capture");
  // Stream-ordered growth: the old workspace is released behind the work
  // already queued on s, and nothing here blocks the host.  (The previous
  // form synchronised s and cudaFree'd under the lock: with one host thread
  // per rank, a rank whose stream held a collective waiting for a peer kept
  // the lock while the peer's thread blocked on it before launching its side
  // of that collective — a deadlock on the first growth of an NCCL run.)
  const size_t want = bytes + bytes / 4 + 256;
  void* p = nullptr;
  CG_CUDA(cudaMallocAsync(&p, want, s));
  void* old = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    Entry& e = cache[key];
    old = e.p;
    e.p = p;
    e.bytes = want;
  }
  if (old) CG_CUDA(cudaFreeAsync(old, s));
  return p;
}

}  // namespace cagnet
