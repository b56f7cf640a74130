// K4 — CSR / block construction on the GPU, bit-exact in structure with the
// reference (csr.cpp, dataset.cpp).
//
// The reference Erdős–Rényi generator (csr.cpp:195-218) walks all n(n-1)
// ordered pairs with one sequential xoshiro256** draw each — 9 ns/pair on a
// CPU core, ≈8 minutes for the Reddit-shaped graph.  Row u always consumes
// exactly n-1 draws, so its sub-stream starts at draw u*(n-1).  The state
// update of xoshiro is linear over GF(2); the host builds the 256x256 jump
// matrix J = T^(n-1) and its powers J^(2^i), one thread per row applies the
// powers selected by the bits of u to the seed state and then replays the
// row's n-1 draws.  Accept/reject uses the exact integer form of
// next_double() < p:  (x >> 11) < ceil(p * 2^53).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "graph.cuh"
#include "rng.hpp"

namespace cagnet {
namespace {

struct DevXoshiro {
  uint64_t s0, s1, s2, s3;
  __device__ __forceinline__ uint64_t next() {
    const uint64_t x = s1 * 5;
    const uint64_t result = ((x << 7) | (x >> 57)) * 9;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = (s3 << 45) | (s3 >> 19);
    return result;
  }
};

// states[idx] = (J^idx) * s0 using the powers J^(2^i) (i < nbits), staged
// matrix by matrix through shared memory.
__global__ void __launch_bounds__(256)
    jump_states_kernel(const uint64_t* __restrict__ mats, int nbits, ulonglong4 s0,
                       int64_t count, uint64_t* __restrict__ states) {
  __shared__ uint64_t m[256 * 4];
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t x[4] = {s0.x, s0.y, s0.z, s0.w};
  for (int i = 0; i < nbits; ++i) {
    __syncthreads();
    for (int t = threadIdx.x; t < 1024; t += blockDim.x) m[t] = mats[static_cast<int64_t>(i) * 1024 + t];
    __syncthreads();
    if (idx < count && ((idx >> i) & 1)) {
      uint64_t y[4] = {0, 0, 0, 0};
#pragma unroll 4
      for (int r = 0; r < 256; ++r) {
        const int p = __popcll(m[r * 4 + 0] & x[0]) + __popcll(m[r * 4 + 1] & x[1]) +
                      __popcll(m[r * 4 + 2] & x[2]) + __popcll(m[r * 4 + 3] & x[3]);
        y[r >> 6] |= static_cast<uint64_t>(p & 1) << (r & 63);
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) x[w] = y[w];
    }
  }
  if (idx < count) {
#pragma unroll
    for (int w = 0; w < 4; ++w) states[idx * 4 + w] = x[w];
  }
}

int bit_length(uint64_t v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

// Device array of start states for `count` sub-streams of `step` draws each.
DevBuf<uint64_t> sub_stream_states(uint64_t seed, uint64_t step, int64_t count, cudaStream_t s) {
  const int nbits = count > 1 ? bit_length(static_cast<uint64_t>(count - 1)) : 0;
  std::vector<Gf2Mat> pw = jump_powers(step, nbits);
  DevBuf<uint64_t> mats(static_cast<size_t>(nbits > 0 ? nbits : 1) * 1024);
  std::vector<uint64_t> flat(static_cast<size_t>(nbits) * 1024);
  for (int i = 0; i < nbits; ++i) std::memcpy(&flat[static_cast<size_t>(i) * 1024], pw[i].rows, 8192);
  if (nbits > 0)
    CG_CUDA(cudaMemcpyAsync(mats.get(), flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, s));
  Xoshiro base(seed);
  DevBuf<uint64_t> states(static_cast<size_t>(count) * 4);
  const ulonglong4 s0 = make_ulonglong4(base.s[0], base.s[1], base.s[2], base.s[3]);
  const unsigned blocks = static_cast<unsigned>(ceil_div64(count, 256));
  jump_states_kernel<<<blocks, 256, 0, s>>>(mats.get(), nbits, s0, count, states.get());
  CG_LAUNCH_CHECK();
  // `flat` must outlive the async copy.
  CG_CUDA(cudaStreamSynchronize(s));
  return states;
}

// One thread per row u: n-1 draws, skipping v == u (no draw consumed).
template <bool FILL>
__global__ void __launch_bounds__(128)
    er_rows_kernel(int64_t n, uint64_t thresh, const uint64_t* __restrict__ states,
                   int64_t* __restrict__ counts, const int64_t* __restrict__ row_ptr,
                   int32_t* __restrict__ cols) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  DevXoshiro g{states[u * 4 + 0], states[u * 4 + 1], states[u * 4 + 2], states[u * 4 + 3]};
  int64_t cnt = 0;
  int64_t pos = FILL ? row_ptr[u] : 0;
  for (int64_t v = 0; v < n; ++v) {
    if (v == u) continue;
    const uint64_t r = g.next();
    if ((r >> 11) < thresh) {
      if (FILL) cols[pos++] = static_cast<int32_t>(v);
      ++cnt;
    }
  }
  if (!FILL) counts[u] = cnt;
}

// splitmix64 finaliser used to derive independent per-row seeds for the
// O(nnz) generator.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <bool FILL>
__global__ void __launch_bounds__(128)
    er_skip_kernel(int64_t n, double log1mp, uint64_t seed, int64_t* __restrict__ counts,
                   const int64_t* __restrict__ row_ptr, int32_t* __restrict__ cols) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  // Per-row xoshiro state from splitmix64(seed, u) (same expansion as Rng's ctor).
  uint64_t x = seed ^ (0x9e3779b97f4a7c15ULL * static_cast<uint64_t>(u + 1));
  DevXoshiro g;
  x += 0x9e3779b97f4a7c15ULL; g.s0 = mix64(x);
  x += 0x9e3779b97f4a7c15ULL; g.s1 = mix64(x);
  x += 0x9e3779b97f4a7c15ULL; g.s2 = mix64(x);
  x += 0x9e3779b97f4a7c15ULL; g.s3 = mix64(x);
  int64_t cnt = 0;
  int64_t pos = FILL ? row_ptr[u] : 0;
  int64_t t = -1;  // candidate index over the n-1 non-self columns
  for (;;) {
    const double uu = static_cast<double>(g.next() >> 11) * 0x1.0p-53;
    const double gap = floor(log1p(-uu) / log1mp);
    if (!(gap < static_cast<double>(n))) break;
    t += static_cast<int64_t>(gap) + 1;
    if (t >= n - 1) break;
    if (FILL) cols[pos++] = static_cast<int32_t>(t < u ? t : t + 1);
    ++cnt;
  }
  if (!FILL) counts[u] = cnt;
}

// row_ptr[0] = 0, row_ptr[i+1] = row_ptr[i] + counts[i].
void counts_to_row_ptr(const int64_t* counts, int64_t n, int64_t* row_ptr, cudaStream_t s) {
  CG_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int64_t), s));
  if (n == 0) return;
  size_t temp = 0;
  CG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, counts, row_ptr + 1, n, s));
  DevBuf<char> tmp(temp);
  CG_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), temp, counts, row_ptr + 1, n, s));
  CG_CUDA(cudaStreamSynchronize(s));
}

int64_t read_back_i64(const int64_t* p, cudaStream_t s) {
  int64_t v = 0;
  CG_CUDA(cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  return v;
}

__global__ void fill_ones_kernel(float* v, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[e] = 1.0f;
}

unsigned grid_for(int64_t total, int threads = 256) {
  int64_t b = ceil_div64(total > 0 ? total : 1, threads);
  const int64_t cap = 8LL * num_sms(current_device());
  return static_cast<unsigned>(b < cap ? b : cap);
}

// ---- normalize (csr.cpp:94-116) ------------------------------------------------
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t lo, int64_t hi,
                                                   int64_t key) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void norm_degree_kernel(int64_t n, const int64_t* __restrict__ rp,
                                   const int32_t* __restrict__ ci, int64_t* __restrict__ cnt,
                                   int32_t* __restrict__ deg) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t lb = lower_bound_i32(ci, rp[i], rp[i + 1], i);
  const bool has = lb < rp[i + 1] && ci[lb] == i;
  const int64_t d = rp[i + 1] - rp[i] + (has ? 0 : 1);
  cnt[i] = d;
  deg[i] = static_cast<int32_t>(d);
}

// Warp per row: merge the diagonal into the sorted row, values 1/sqrt(d_i d_j)
// in fp64 (IEEE sqrt and division, as on the host) rounded to fp32.
__global__ void norm_fill_kernel(int64_t n, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, const int32_t* __restrict__ deg,
                                 const int64_t* __restrict__ orp, int32_t* __restrict__ oci,
                                 float* __restrict__ ov) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int64_t beg = rp[i], end = rp[i + 1], obeg = orp[i];
  const bool has = (orp[i + 1] - obeg) == (end - beg);
  const double di = static_cast<double>(deg[i]);
  for (int64_t t = beg + lane; t < end; t += 32) {
    const int32_t c = ci[t];
    const int64_t pos = obeg + (t - beg) + ((!has && c > i) ? 1 : 0);
    oci[pos] = c;
    ov[pos] = static_cast<float>(1.0 / sqrt(di * static_cast<double>(deg[c])));
  }
  if (!has && lane == 0) {
    const int64_t lb = lower_bound_i32(ci, beg, end, i);
    oci[obeg + (lb - beg)] = static_cast<int32_t>(i);
    ov[obeg + (lb - beg)] = static_cast<float>(1.0 / sqrt(di * di));
  }
}

// ---- transpose ------------------------------------------------------------------
__global__ void iota_u32_kernel(uint32_t* p, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[e] = static_cast<uint32_t>(e);
}

// t_row_ptr[c] = first position of key >= c in the sorted keys.
__global__ void keys_to_row_ptr_kernel(const int32_t* __restrict__ keys, int64_t nnz,
                                       int64_t n_cols, int64_t* __restrict__ trp) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c > n_cols) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < c)
      lo = mid + 1;
    else
      hi = mid;
  }
  trp[c] = lo;
}

// Gathers the source row (upper_bound in row_ptr) and value of every permuted nonzero.
__global__ void transpose_gather_kernel(int64_t nnz, int64_t n_rows, const uint32_t* __restrict__ perm,
                                        const int64_t* __restrict__ rp, const float* __restrict__ v,
                                        int32_t* __restrict__ tci, float* __restrict__ tv) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t src = perm[e];
    int64_t lo = 0, hi = n_rows;  // find row r with rp[r] <= src < rp[r+1]
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= src)
        lo = mid;
      else
        hi = mid - 1;
    }
    tci[e] = static_cast<int32_t>(lo);
    tv[e] = v[src];
  }
}

// ---- extract_block -----------------------------------------------------------------
__global__ void block_count_kernel(int64_t r0, int64_t rows, int64_t c0, int64_t c1,
                                   const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                   int64_t* __restrict__ lo_out, int64_t* __restrict__ cnt) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t b = rp[r0 + r], e = rp[r0 + r + 1];
  const int64_t lo = lower_bound_i32(ci, b, e, c0);
  const int64_t hi = lower_bound_i32(ci, lo, e, c1);
  lo_out[r] = lo;
  cnt[r] = hi - lo;
}

__global__ void block_fill_kernel(int64_t rows, int64_t c0, const int64_t* __restrict__ lo_in,
                                  const int64_t* __restrict__ orp, const int32_t* __restrict__ ci,
                                  const float* __restrict__ v, int32_t* __restrict__ oci,
                                  float* __restrict__ ov) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const int64_t lo = lo_in[r], ob = orp[r], len = orp[r + 1] - ob;
  for (int64_t t = lane; t < len; t += 32) {
    oci[ob + t] = static_cast<int32_t>(ci[lo + t] - c0);
    ov[ob + t] = v[lo + t];
  }
}

__global__ void rotate_rows_kernel(int64_t rows, int32_t c0, int32_t c1, const int64_t* __restrict__ rp,
                                   const int32_t* __restrict__ ci, const float* __restrict__ v,
                                   int32_t* __restrict__ oci, float* __restrict__ ov,
                                   int64_t* __restrict__ mid) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const int64_t b = rp[r], e = rp[r + 1], len = e - b;
  const int64_t lo = lower_bound_i32(ci, b, e, c0);
  const int64_t hi = lower_bound_i32(ci, lo, e, c1);
  if (lane == 0) mid[r] = b + (hi - lo);
  for (int64_t t = lane; t < len; t += 32) {
    int64_t src = lo + t;
    if (src >= e) src -= len;
    oci[b + t] = ci[src];
    ov[b + t] = v[src];
  }
}

// ---- features ----------------------------------------------------------------------
constexpr int64_t kFeatChunk = 4096;

__global__ void __launch_bounds__(128)
    features_kernel(int64_t total, int64_t f, int64_t ld, const uint64_t* __restrict__ states,
                    int64_t chunks, float* __restrict__ out) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= chunks) return;
  DevXoshiro g{states[c * 4 + 0], states[c * 4 + 1], states[c * 4 + 2], states[c * 4 + 3]};
  const int64_t start = c * kFeatChunk;
  const int64_t end = start + kFeatChunk < total ? start + kFeatChunk : total;
  int64_t row = start / f, col = start % f;
  for (int64_t e = start; e < end; ++e) {
    const double d = static_cast<double>(g.next() >> 11) * 0x1.0p-53;
    out[row * ld + col] = static_cast<float>(d);
    if (++col == f) {
      col = 0;
      ++row;
    }
  }
}

}  // namespace

DeviceCsr er_generate_device(int64_t n, double degree, uint64_t seed, cudaStream_t s) {
  require(n > 0, "generate_erdos_renyi: n must be positive");
  const double p = degree / static_cast<double>(n);
  require(p >= 0.0 && p <= 1.0, "generate_erdos_renyi: edge probability " + std::to_string(p) +
                                    " outside [0, 1]");
  require(n < (1LL << 31), "generate_erdos_renyi: n must fit int32 column indices");
  uint64_t thresh;
  if (p >= 1.0)
    thresh = 1ULL << 53;
  else
    thresh = static_cast<uint64_t>(std::ceil(std::ldexp(p, 53)));

  DeviceCsr a;
  a.device = current_device();
  a.n_rows = a.n_cols = n;
  DevBuf<uint64_t> states = sub_stream_states(seed, static_cast<uint64_t>(n - 1), n, s);
  DevBuf<int64_t> counts(static_cast<size_t>(n));
  const unsigned blocks = static_cast<unsigned>(ceil_div64(n, 128));
  er_rows_kernel<false><<<blocks, 128, 0, s>>>(n, thresh, states.get(), counts.get(), nullptr, nullptr);
  CG_LAUNCH_CHECK();
  a.row_ptr.resize(static_cast<size_t>(n + 1));
  counts_to_row_ptr(counts.get(), n, a.row_ptr.get(), s);
  a.nnz = read_back_i64(a.row_ptr.get() + n, s);
  a.col_idx.resize(static_cast<size_t>(a.nnz));
  er_rows_kernel<true><<<blocks, 128, 0, s>>>(n, thresh, states.get(), nullptr, a.row_ptr.get(),
                                              a.col_idx.get());
  CG_LAUNCH_CHECK();
  a.vals.resize(static_cast<size_t>(a.nnz));
  fill_ones_kernel<<<grid_for(a.nnz), 256, 0, s>>>(a.vals.get(), a.nnz);
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
  return a;
}

DeviceCsr er_skip_generate_device(int64_t n, double degree, uint64_t seed, cudaStream_t s) {
  require(n > 1, "er_skip_generate: n must be > 1");
  const double p = degree / static_cast<double>(n);
  require(p > 0.0 && p < 1.0, "er_skip_generate: edge probability outside (0, 1)");
  require(n < (1LL << 31), "er_skip_generate: n must fit int32 column indices");
  DeviceCsr a;
  a.device = current_device();
  a.n_rows = a.n_cols = n;
  DevBuf<int64_t> counts(static_cast<size_t>(n));
  const double log1mp = std::log1p(-p);
  const unsigned blocks = static_cast<unsigned>(ceil_div64(n, 128));
  er_skip_kernel<false><<<blocks, 128, 0, s>>>(n, log1mp, seed, counts.get(), nullptr, nullptr);
  CG_LAUNCH_CHECK();
  a.row_ptr.resize(static_cast<size_t>(n + 1));
  counts_to_row_ptr(counts.get(), n, a.row_ptr.get(), s);
  a.nnz = read_back_i64(a.row_ptr.get() + n, s);
  a.col_idx.resize(static_cast<size_t>(a.nnz));
  er_skip_kernel<true><<<blocks, 128, 0, s>>>(n, log1mp, seed, nullptr, a.row_ptr.get(), a.col_idx.get());
  CG_LAUNCH_CHECK();
  a.vals.resize(static_cast<size_t>(a.nnz));
  fill_ones_kernel<<<grid_for(a.nnz), 256, 0, s>>>(a.vals.get(), a.nnz);
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
  return a;
}

DeviceCsr normalize_device(const DeviceCsr& raw, DevBuf<int32_t>* degree_out, cudaStream_t s) {
  require(raw.n_rows == raw.n_cols, "add_self_loops_and_normalize: matrix is " +
                                        std::to_string(raw.n_rows) + "x" +
                                        std::to_string(raw.n_cols) + ", expected square");
  const int64_t n = raw.n_rows;
  DeviceCsr out;
  out.device = current_device();
  out.n_rows = out.n_cols = n;
  DevBuf<int64_t> cnt(static_cast<size_t>(n));
  DevBuf<int32_t> deg(static_cast<size_t>(n));
  const unsigned b = static_cast<unsigned>(ceil_div64(n, 256));
  norm_degree_kernel<<<b, 256, 0, s>>>(n, raw.row_ptr.get(), raw.col_idx.get(), cnt.get(), deg.get());
  CG_LAUNCH_CHECK();
  out.row_ptr.resize(static_cast<size_t>(n + 1));
  counts_to_row_ptr(cnt.get(), n, out.row_ptr.get(), s);
  out.nnz = read_back_i64(out.row_ptr.get() + n, s);
  out.col_idx.resize(static_cast<size_t>(out.nnz));
  out.vals.resize(static_cast<size_t>(out.nnz));
  const unsigned wb = static_cast<unsigned>(ceil_div64(n * 32, 256));
  norm_fill_kernel<<<wb, 256, 0, s>>>(n, raw.row_ptr.get(), raw.col_idx.get(), deg.get(),
                                      out.row_ptr.get(), out.col_idx.get(), out.vals.get());
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
  if (degree_out) *degree_out = std::move(deg);
  return out;
}

DeviceCsr transpose_device(const DeviceCsr& a, cudaStream_t s) {
  require(a.nnz < (1LL << 32), "transpose: nnz must fit 32-bit positions");
  DeviceCsr t;
  t.device = current_device();
  t.n_rows = a.n_cols;
  t.n_cols = a.n_rows;
  t.nnz = a.nnz;
  t.row_ptr.resize(static_cast<size_t>(t.n_rows + 1));
  t.col_idx.resize(static_cast<size_t>(t.nnz));
  t.vals.resize(static_cast<size_t>(t.nnz));
  if (a.nnz == 0) {
    CG_CUDA(cudaMemsetAsync(t.row_ptr.get(), 0, (t.n_rows + 1) * sizeof(int64_t), s));
    CG_CUDA(cudaStreamSynchronize(s));
    return t;
  }
  // Stable LSD radix sort of (column, position) pairs: within a column the
  // positions stay ascending, i.e. source rows ascending (csr.cpp:130-136).
  DevBuf<int32_t> keys_out(static_cast<size_t>(a.nnz));
  DevBuf<uint32_t> pos_in(static_cast<size_t>(a.nnz)), pos_out(static_cast<size_t>(a.nnz));
  iota_u32_kernel<<<grid_for(a.nnz), 256, 0, s>>>(pos_in.get(), a.nnz);
  CG_LAUNCH_CHECK();
  const int end_bit = bit_length(static_cast<uint64_t>(a.n_cols > 1 ? a.n_cols - 1 : 1));
  size_t temp = 0;
  CG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, a.col_idx.get(), keys_out.get(),
                                          pos_in.get(), pos_out.get(), a.nnz, 0, end_bit, s));
  {
    DevBuf<char> tmp(temp);
    CG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), temp, a.col_idx.get(), keys_out.get(),
                                            pos_in.get(), pos_out.get(), a.nnz, 0, end_bit, s));
    CG_CUDA(cudaStreamSynchronize(s));
  }
  pos_in.release();
  keys_to_row_ptr_kernel<<<static_cast<unsigned>(ceil_div64(t.n_rows + 1, 256)), 256, 0, s>>>(
      keys_out.get(), a.nnz, t.n_rows, t.row_ptr.get());
  CG_LAUNCH_CHECK();
  transpose_gather_kernel<<<grid_for(a.nnz), 256, 0, s>>>(a.nnz, a.n_rows, pos_out.get(),
                                                          a.row_ptr.get(), a.vals.get(),
                                                          t.col_idx.get(), t.vals.get());
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
  return t;
}

__global__ void permuted_len_kernel(int64_t n, const int64_t* __restrict__ rp,
                                    const int64_t* __restrict__ perm, int64_t* __restrict__ len) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) len[i] = rp[perm[i] + 1] - rp[perm[i]];
}

// Warp per new row i: the entries of old row perm[i] with columns relabelled
// by inv, in old order (the segmented sort below orders them).
__global__ void permuted_fill_kernel(int64_t n, const int64_t* __restrict__ rp,
                                     const int32_t* __restrict__ ci, const float* __restrict__ v,
                                     const int64_t* __restrict__ perm, const int64_t* __restrict__ inv,
                                     const int64_t* __restrict__ new_rp, int32_t* __restrict__ keys,
                                     float* __restrict__ vals) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t r = perm[i], b = rp[r], e = rp[r + 1], o = new_rp[i];
  for (int64_t k = b + lane; k < e; k += 32) {
    keys[o + (k - b)] = static_cast<int32_t>(inv[ci[k]]);
    vals[o + (k - b)] = v[k];
  }
}

DeviceCsr permute_csr_device(const DeviceCsr& a, const int64_t* perm, const int64_t* inv,
                             cudaStream_t s) {
  require(a.n_rows == a.n_cols, "permute_random: square adjacency required");
  require(a.nnz < (1LL << 31), "permute_random: nnz must fit the segmented sort");
  DeviceCsr out;
  out.device = current_device();
  out.n_rows = a.n_rows;
  out.n_cols = a.n_cols;
  out.nnz = a.nnz;
  const int64_t n = a.n_rows;
  out.row_ptr.resize(static_cast<size_t>(n + 1));
  out.col_idx.resize(static_cast<size_t>(std::max<int64_t>(a.nnz, 1)));
  out.vals.resize(static_cast<size_t>(std::max<int64_t>(a.nnz, 1)));
  CG_CUDA(cudaMemsetAsync(out.row_ptr.get(), 0, sizeof(int64_t), s));
  if (n == 0) return out;
  DevBuf<int64_t> len(static_cast<size_t>(n));
  permuted_len_kernel<<<static_cast<unsigned>(ceil_div64(n, 256)), 256, 0, s>>>(n, a.row_ptr.get(), perm, len.get());
  CG_LAUNCH_CHECK();
  size_t temp = 0;
  CG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, len.get(), out.row_ptr.get() + 1, n, s));
  {
    DevBuf<char> tmp(temp);
    CG_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), temp, len.get(), out.row_ptr.get() + 1, n, s));
    CG_CUDA(cudaStreamSynchronize(s));
  }
  if (a.nnz == 0) return out;
  DevBuf<int32_t> keys(static_cast<size_t>(a.nnz));
  DevBuf<float> vals(static_cast<size_t>(a.nnz));
  permuted_fill_kernel<<<static_cast<unsigned>(ceil_div64(n * 32, 256)), 256, 0, s>>>(
      n, a.row_ptr.get(), a.col_idx.get(), a.vals.get(), perm, inv, out.row_ptr.get(), keys.get(),
      vals.get());
  CG_LAUNCH_CHECK();
  temp = 0;
  CG_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, temp, keys.get(), out.col_idx.get(), vals.get(),
                                              out.vals.get(), static_cast<int>(a.nnz), static_cast<int>(n),
                                              out.row_ptr.get(), out.row_ptr.get() + 1, s));
  {
    DevBuf<char> tmp(temp);
    CG_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp.get(), temp, keys.get(), out.col_idx.get(),
                                                vals.get(), out.vals.get(), static_cast<int>(a.nnz),
                                                static_cast<int>(n), out.row_ptr.get(),
                                                out.row_ptr.get() + 1, s));
    CG_CUDA(cudaStreamSynchronize(s));
  }
  return out;
}

DeviceCsr extract_block_device(const DeviceCsr& a, int64_t r0, int64_t r1, int64_t c0,
                               int64_t c1, cudaStream_t s) {
  if (r0 > r1 || r1 > a.n_rows || c0 > c1 || c1 > a.n_cols)
    throw std::invalid_argument("extract_block: range [" + std::to_string(r0) + "," +
                                std::to_string(r1) + ")x[" + std::to_string(c0) + "," +
                                std::to_string(c1) + ") outside " + std::to_string(a.n_rows) +
                                "x" + std::to_string(a.n_cols));
  DeviceCsr b;
  b.device = current_device();
  b.n_rows = r1 - r0;
  b.n_cols = c1 - c0;
  b.row_off = a.row_off + r0;
  b.col_off = a.col_off + c0;
  b.row_ptr.resize(static_cast<size_t>(b.n_rows + 1));
  if (b.n_rows == 0) {
    CG_CUDA(cudaMemsetAsync(b.row_ptr.get(), 0, sizeof(int64_t), s));
    CG_CUDA(cudaStreamSynchronize(s));
    b.col_idx.resize(0);
    b.vals.resize(0);
    return b;
  }
  DevBuf<int64_t> lo(static_cast<size_t>(b.n_rows)), cnt(static_cast<size_t>(b.n_rows));
  block_count_kernel<<<static_cast<unsigned>(ceil_div64(b.n_rows, 256)), 256, 0, s>>>(
      r0, b.n_rows, c0, c1, a.row_ptr.get(), a.col_idx.get(), lo.get(), cnt.get());
  CG_LAUNCH_CHECK();
  counts_to_row_ptr(cnt.get(), b.n_rows, b.row_ptr.get(), s);
  b.nnz = read_back_i64(b.row_ptr.get() + b.n_rows, s);
  b.col_idx.resize(static_cast<size_t>(b.nnz));
  b.vals.resize(static_cast<size_t>(b.nnz));
  block_fill_kernel<<<static_cast<unsigned>(ceil_div64(b.n_rows * 32, 256)), 256, 0, s>>>(
      b.n_rows, c0, lo.get(), b.row_ptr.get(), a.col_idx.get(), a.vals.get(), b.col_idx.get(),
      b.vals.get());
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
  return b;
}

RotatedCsr rotate_rows_device(const DeviceCsr& a, int64_t c0, int64_t c1, cudaStream_t s) {
  require(0 <= c0 && c0 <= c1 && c1 <= a.n_cols, "rotate_rows: column range outside the matrix");
  RotatedCsr o;
  o.col_idx.resize(static_cast<size_t>(std::max<int64_t>(a.nnz, 1)));
  o.vals.resize(static_cast<size_t>(std::max<int64_t>(a.nnz, 1)));
  o.mid.resize(static_cast<size_t>(std::max<int64_t>(a.n_rows, 1)));
  if (a.n_rows > 0) {
    rotate_rows_kernel<<<static_cast<unsigned>(ceil_div64(a.n_rows * 32, 256)), 256, 0, s>>>(
        a.n_rows, static_cast<int32_t>(c0), static_cast<int32_t>(c1), a.row_ptr.get(), a.col_idx.get(),
        a.vals.get(), o.col_idx.get(), o.vals.get(), o.mid.get());
    CG_LAUNCH_CHECK();
  }
  CG_CUDA(cudaStreamSynchronize(s));
  return o;
}

DeviceCsr upload_csr(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* vals, cudaStream_t s) {
  require(n_rows >= 0 && n_cols >= 0, "csr_upload: negative shape");
  require(n_cols < (1LL << 31), "csr_upload: n_cols must fit int32 column indices");
  DeviceCsr a;
  a.device = current_device();
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.nnz = row_ptr[n_rows];
  std::vector<int32_t> ci(static_cast<size_t>(a.nnz));
  std::vector<float> v(static_cast<size_t>(a.nnz));
  for (int64_t k = 0; k < a.nnz; ++k) {
    require(col_idx[k] >= 0 && col_idx[k] < n_cols, "csr_upload: column index out of range");
    ci[k] = static_cast<int32_t>(col_idx[k]);
    v[k] = vals ? static_cast<float>(vals[k]) : 1.0f;
  }
  a.row_ptr.resize(static_cast<size_t>(n_rows + 1));
  a.col_idx.resize(static_cast<size_t>(a.nnz));
  a.vals.resize(static_cast<size_t>(a.nnz));
  CG_CUDA(cudaMemcpyAsync(a.row_ptr.get(), row_ptr, (n_rows + 1) * sizeof(int64_t),
                          cudaMemcpyHostToDevice, s));
  if (a.nnz) {
    CG_CUDA(cudaMemcpyAsync(a.col_idx.get(), ci.data(), a.nnz * sizeof(int32_t),
                            cudaMemcpyHostToDevice, s));
    CG_CUDA(cudaMemcpyAsync(a.vals.get(), v.data(), a.nnz * sizeof(float), cudaMemcpyHostToDevice, s));
  }
  CG_CUDA(cudaStreamSynchronize(s));
  return a;
}

void random_features_device(int64_t n, int64_t f, uint64_t seed, float* out, int64_t ld,
                            cudaStream_t s) {
  const int64_t total = n * f;
  if (total == 0) return;
  const int64_t chunks = ceil_div64(total, kFeatChunk);
  DevBuf<uint64_t> states = sub_stream_states(seed, static_cast<uint64_t>(kFeatChunk), chunks, s);
  features_kernel<<<static_cast<unsigned>(ceil_div64(chunks, 128)), 128, 0, s>>>(
      total, f, ld, states.get(), chunks, out);
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
}

std::vector<int32_t> random_labels_host(int64_t n, int64_t classes, uint64_t seed) {
  require(classes > 0, "random_labels: need at least one class");
  Xoshiro rng(seed);
  std::vector<int32_t> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<int32_t>(rng.bounded(static_cast<uint64_t>(classes)));
  return out;
}

}  // namespace cagnet
