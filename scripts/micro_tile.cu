// Microbenchmark: f = 16 SpMM on a random 233K x 233K matrix (494 nnz/row), row-parallel
// gathers (the product kernel's shape) vs a persistent row-chunk kernel that walks column
// tiles so the H slice of a tile is reused from L1 (L1 variant) or from shared memory
// staged by cp.async (SMEM variant).  Accumulators: K rows per 4-lane quad in registers.
// Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_tile micro_tile.cu
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void fma4(float4& a, float w, const float4& h) {
  a.x = fmaf(w, h.x, a.x); a.y = fmaf(w, h.y, a.y); a.z = fmaf(w, h.z, a.z); a.w = fmaf(w, h.w, a.w);
}

template <int LV, int QPR, int U, int THREADS>
__global__ void __launch_bounds__(THREADS) k_row(int n, const int64_t* __restrict__ rp, const int* __restrict__ ci,
                                                 const float* __restrict__ v, const float* __restrict__ H, float* __restrict__ T) {
  constexpr int TEAM = LV * QPR, RPW = 32 / TEAM;
  const int lane = threadIdx.x & 31, sub = lane % LV, q = (lane % TEAM) / LV;
  const int64_t row = ((int64_t)blockIdx.x * THREADS + threadIdx.x) / 32 * RPW + lane / TEAM;
  int64_t p = 0, e = 0;
  if (row < n) { p = rp[row] + q; e = rp[row + 1]; }
  float4 acc = make_float4(0, 0, 0, 0);
  for (; p + (U - 1) * QPR < e; p += U * QPR) {
    float4 h[U]; float w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = __ldg(ci + p + u * QPR);
      w[u] = __ldg(v + p + u * QPR);
      h[u] = __ldg(reinterpret_cast<const float4*>(H + (int64_t)c * 16) + sub);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) fma4(acc, w[u], h[u]);
  }
  for (; p < e; p += QPR)
    fma4(acc, __ldg(v + p), __ldg(reinterpret_cast<const float4*>(H + (int64_t)__ldg(ci + p) * 16) + sub));
#pragma unroll
  for (int o = LV; o < TEAM; o <<= 1) {
    acc.x += __shfl_xor_sync(~0u, acc.x, o); acc.y += __shfl_xor_sync(~0u, acc.y, o);
    acc.z += __shfl_xor_sync(~0u, acc.z, o); acc.w += __shfl_xor_sync(~0u, acc.w, o);
  }
  if (row < n && q == 0) reinterpret_cast<float4*>(T + row * 16)[sub] = acc;
}

__device__ __forceinline__ void cp16(void* s, const void* g) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Persistent row chunk per CTA; quad (4 lanes, float4 each) owns K consecutive rows;
// every CTA walks column tiles of CW columns in order.
template <int K, int U, bool SMEM, int CW, int NT>
__global__ void __launch_bounds__(NT, 1) k_tile(int n, const int64_t* __restrict__ rp, const int* __restrict__ ci,
                                                const float* __restrict__ v, const float* __restrict__ H,
                                                float* __restrict__ T, int rows_per_cta) {
  extern __shared__ float4 hs[];
  const int tid = threadIdx.x, quad = tid >> 2, lv = tid & 3;
  const int rbase = blockIdx.x * rows_per_cta;
  unsigned cur[K], end[K];
  float4 acc[K];
  const int64_t nzbase = rp[min(rbase, n)];
  ci += nzbase;
  v += nzbase;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int lr = quad * K + j, row = rbase + lr;
    cur[j] = end[j] = 0;
    if (lr < rows_per_cta && row < n) { cur[j] = unsigned(rp[row] - nzbase); end[j] = unsigned(rp[row + 1] - nzbase); }
    acc[j] = make_float4(0, 0, 0, 0);
  }
  const int ntiles = (n + CW - 1) / CW;
  auto stage = [&](int t) {
    const int c0 = t * CW;
    const int rows = min(CW, n - c0);
    float4* dst = hs + (t & 1) * CW * 4;
    const float4* src = reinterpret_cast<const float4*>(H) + (int64_t)c0 * 4;
    for (int i = tid; i < rows * 4; i += NT) cp16(dst + i, src + i);
    cp_commit();
  };
  if (SMEM) stage(0);
  for (int t = 0; t < ntiles; ++t) {
    if (SMEM) {
      if (t + 1 < ntiles) { stage(t + 1); cp_wait<1>(); } else cp_wait<0>();
      __syncthreads();
    }
    const int cend = min((t + 1) * CW, n);
    const float4* hb = hs + (t & 1) * CW * 4 - (int64_t)t * CW * 4 + lv;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      while (true) {
        int c[U]; float w[U]; float4 h[U];
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const unsigned p = cur[j] + u;
          c[u] = p < end[j] ? __ldg(ci + p) : INT_MAX;
          const bool ok = c[u] < cend;
          cnt += ok;
          w[u] = ok ? __ldg(v + p) : 0.f;
          if (SMEM) h[u] = ok ? hb[c[u] * 4] : make_float4(0, 0, 0, 0);
          else h[u] = ok ? __ldg(reinterpret_cast<const float4*>(H + (int64_t)c[u] * 16) + lv) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) fma4(acc[j], w[u], h[u]);
        cur[j] += cnt;
        if (cnt < U) break;
      }
    }
    if (SMEM) __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int lr = quad * K + j, row = rbase + lr;
    if (lr < rows_per_cta && row < n) reinterpret_cast<float4*>(T + (int64_t)row * 16)[lv] = acc[j];
  }
}

// Sub-team q of a row (QPR = 8 sub-teams of 4 lanes) loads entries [base + 4q, base + 4q + 4) of
// every 32-entry window as one int4 / float4 (one 128 B wavefront per window for the warp's row);
// dead slots (before the row start or past its end) skip the gather.
template <bool VALS, int WIN>
__global__ void __launch_bounds__(128) k_vec(int n, const int64_t* __restrict__ rp, const int* __restrict__ ci,
                                             const float* __restrict__ v, const float* __restrict__ H, float* __restrict__ T) {
  const int lane = threadIdx.x & 31, sub = lane & 3, q = lane >> 2;
  const int64_t row = ((int64_t)blockIdx.x * 128 + threadIdx.x) >> 5;
  if (row >= n) return;
  const int64_t b = rp[row], e = rp[row + 1];
  float4 acc = make_float4(0, 0, 0, 0);
  const char* hb = reinterpret_cast<const char*>(H) + sub * 16;
  for (int64_t base = b & ~int64_t(3); base < e; base += 32 * WIN) {
    int4 c[WIN]; float4 w[WIN];
#pragma unroll
    for (int u = 0; u < WIN; ++u) {
      const int64_t p = base + 32 * u + 4 * q;
      c[u] = p < e ? __ldg(reinterpret_cast<const int4*>(ci + p)) : make_int4(0, 0, 0, 0);
      if (VALS) w[u] = p < e ? __ldg(reinterpret_cast<const float4*>(v + p)) : make_float4(0, 0, 0, 0);
      else w[u] = make_float4(1e-3f, 1e-3f, 1e-3f, 1e-3f);
    }
#pragma unroll
    for (int u = 0; u < WIN; ++u) {
      const int64_t p = base + 32 * u + 4 * q;
      const int cc[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
      const float ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
      float4 h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool live = p + i >= b && p + i < e;
        h[i] = live ? __ldg(reinterpret_cast<const float4*>(hb + (uint64_t)(uint32_t)cc[i] * 64u)) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) fma4(acc, (p + i >= b && p + i < e) ? ww[i] : 0.f, h[i]);
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(~0u, acc.x, o); acc.y += __shfl_xor_sync(~0u, acc.y, o);
    acc.z += __shfl_xor_sync(~0u, acc.z, o); acc.w += __shfl_xor_sync(~0u, acc.w, o);
  }
  if (q == 0) reinterpret_cast<float4*>(T + row * 16)[sub] = acc;
}

int main() {
  const int n = 232965, deg = 494;
  const int64_t nnz = (int64_t)n * deg;
  std::vector<int64_t> rp(n + 1);
  std::vector<int> ci(nnz);
  std::vector<float> vv(nnz);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i <= n; ++i) rp[i] = (int64_t)i * deg;
  for (int64_t k = 0; k < nnz; ++k) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; ci[k] = (int)(s % n); vv[k] = 1e-3f * (1 + (s >> 40) % 7); }
  for (int i = 0; i < n; ++i) std::sort(ci.begin() + rp[i], ci.begin() + rp[i + 1]);
  int64_t* d_rp; int* d_ci; float *d_v, *d_H, *d_T;
  CK(cudaMalloc(&d_rp, (n + 1) * 8)); CK(cudaMalloc(&d_ci, nnz * 4)); CK(cudaMalloc(&d_v, nnz * 4));
  CK(cudaMalloc(&d_H, (size_t)n * 64)); CK(cudaMalloc(&d_T, (size_t)n * 64));
  CK(cudaMemcpy(d_rp, rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_v, vv.data(), nnz * 4, cudaMemcpyHostToDevice));
  std::vector<float> hh((size_t)n * 16);
  for (auto& x : hh) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = (s % 1000) * 1e-3f; }
  CK(cudaMemcpy(d_H, hh.data(), hh.size() * 4, cudaMemcpyHostToDevice));
  std::vector<float> ref((size_t)n * 16), got((size_t)n * 16);
  bool have_ref = false;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    CK(cudaMemset(d_T, 0, (size_t)n * 64));
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    CK(cudaMemcpy(got.data(), d_T, got.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0;
    if (!have_ref) { ref = got; have_ref = true; }
    for (size_t i = 0; i < got.size(); ++i) err = std::max(err, (double)std::abs(got[i] - ref[i]) / (1e-3 + std::abs(ref[i])));
    printf("%-44s %8.3f ms  gather %6.2f TB/s  maxrel %.2e\n", name, ms, nnz * 64.0 / ms / 1e9, err);
  };
  {
    const int rpb = 128 / 32;
    const int grid = (n + rpb - 1) / rpb;
    timeit("row LV4 QPR8 U4 T128 (product shape)", [&] { k_row<4, 8, 4, 128><<<grid, 128>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  }
  {
    const int grid = (n + 3) / 4;
    timeit("vec int4/float4 CSR loads WIN=1", [&] { k_vec<true, 1><<<grid, 128>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
    timeit("vec int4/float4 CSR loads WIN=2", [&] { k_vec<true, 2><<<grid, 128>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
    timeit("vec no vals WIN=1 (diff expected)", [&] { k_vec<false, 1><<<grid, 128>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
    timeit("vec no vals WIN=2 (diff expected)", [&] { k_vec<false, 2><<<grid, 128>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  }
  return 0;
}
