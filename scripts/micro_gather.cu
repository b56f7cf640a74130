// Microbenchmark: gather-bound SpMM variants for narrow f (16) on a random
// (ER-like) 233K x 233K matrix with 494 nnz/row.  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_gather micro_gather.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ float4 ld_na(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// (a)/(b): 4 lanes per row, one float4 per lane, col/val broadcast by shuffle.
template <bool NA, int UNR>
__global__ void __launch_bounds__(256) k_lpr4(int n, const int64_t* rp, const int* ci, const float* v, const float4* H, float4* T) {
  int lane = threadIdx.x & 31, sub = lane & 3, grp = lane >> 2;
  int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) / 32 * 8 + grp;
  int64_t b = 0, len = 0;
  if (row < n) { b = rp[row]; len = rp[row + 1] - b; }
  int64_t mx = len;
  for (int o = 16; o >= 4; o >>= 1) { int64_t t = __shfl_xor_sync(~0u, mx, o); mx = t > mx ? t : mx; }
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = 0; base < mx; base += 4) {
    int c = 0; float vv = 0;
    if (base + sub < len) { c = ci[b + base + sub]; vv = v[b + base + sub]; }
    float4 h[4]; float w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int cc = __shfl_sync(~0u, c, grp * 4 + t); w[t] = __shfl_sync(~0u, vv, grp * 4 + t);
      const float4* p = H + (int64_t)cc * 4 + sub;
      h[t] = NA ? ld_na(p) : __ldg(p);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) { acc.x += w[t] * h[t].x; acc.y += w[t] * h[t].y; acc.z += w[t] * h[t].z; acc.w += w[t] * h[t].w; }
  }
  if (row < n) T[row * 4 + sub] = acc;
}

// (a'): 4 lanes per row; U chunks of 4 nonzeros per iteration, all loads issued
// before the FMAs, predicated (not branched) on the row length.
template <int U>
__global__ void __launch_bounds__(256) k_lpr4u(int n, const int64_t* rp, const int* ci, const float* v, const float4* H, float4* T) {
  int lane = threadIdx.x & 31, sub = lane & 3, grp = lane >> 2;
  int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) / 32 * 8 + grp;
  int64_t b = 0, len = 0;
  if (row < n) { b = rp[row]; len = rp[row + 1] - b; }
  int64_t mx = len;
  for (int o = 16; o >= 4; o >>= 1) { int64_t t = __shfl_xor_sync(~0u, mx, o); mx = t > mx ? t : mx; }
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = 0; base < mx; base += 4 * U) {
    int c[U]; float vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = base + 4 * u + sub;
      c[u] = q < len ? ci[b + q] : 0;
      vv[u] = q < len ? v[b + q] : 0.f;
    }
    float4 h[4 * U]; float w[4 * U];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int cc = __shfl_sync(~0u, c[u], grp * 4 + t);
        w[4 * u + t] = __shfl_sync(~0u, vv[u], grp * 4 + t);
        const bool ok = base + 4 * u + t < len;
        h[4 * u + t] = ok ? __ldg(H + (int64_t)cc * 4 + sub) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
    for (int t = 0; t < 4 * U; ++t) { acc.x = fmaf(w[t], h[t].x, acc.x); acc.y = fmaf(w[t], h[t].y, acc.y); acc.z = fmaf(w[t], h[t].z, acc.z); acc.w = fmaf(w[t], h[t].w, acc.w); }
  }
  if (row < n) T[row * 4 + sub] = acc;
}

// (g): QPR quads (4 lanes) per row, each quad strides over the row's nonzeros
// (no shuffles in the loop), U independent gathers per lane in flight,
// quad partial sums reduced with xor shuffles at the end.
template <int QPR, int U>
__global__ void __launch_bounds__(256) k_qpr(int n, const int64_t* rp, const int* ci, const float* v, const float4* H, float4* T) {
  constexpr int LPR = 4 * QPR, RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, sub = lane & 3, q = (lane % LPR) >> 2, grp = lane / LPR;
  const int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) / 32 * RPW + grp;
  int64_t b = 0, e = 0;
  if (row < n) { b = rp[row]; e = rp[row + 1]; }
  float4 acc = make_float4(0, 0, 0, 0);
  int64_t p = b + q;
  for (; p + (U - 1) * QPR < e; p += U * QPR) {
    float4 h[U]; float w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { const int c = __ldg(ci + p + u * QPR); w[u] = __ldg(v + p + u * QPR); h[u] = __ldg(H + (int64_t)c * 4 + sub); }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x = fmaf(w[u], h[u].x, acc.x); acc.y = fmaf(w[u], h[u].y, acc.y); acc.z = fmaf(w[u], h[u].z, acc.z); acc.w = fmaf(w[u], h[u].w, acc.w); }
  }
  for (; p < e; p += QPR) { const int c = __ldg(ci + p); const float w = __ldg(v + p); const float4 h = __ldg(H + (int64_t)c * 4 + sub);
    acc.x = fmaf(w, h.x, acc.x); acc.y = fmaf(w, h.y, acc.y); acc.z = fmaf(w, h.z, acc.z); acc.w = fmaf(w, h.w, acc.w); }
#pragma unroll
  for (int o = 4; o < LPR; o <<= 1) {
    acc.x += __shfl_xor_sync(~0u, acc.x, o); acc.y += __shfl_xor_sync(~0u, acc.y, o);
    acc.z += __shfl_xor_sync(~0u, acc.z, o); acc.w += __shfl_xor_sync(~0u, acc.w, o);
  }
  if (row < n && q == 0) T[row * 4 + sub] = acc;
}

// (c): warp per row, lane per nonzero, 4 x float4 per lane, butterfly reduce.
template <bool NA>
__global__ void __launch_bounds__(256) k_lane_nnz(int n, const int64_t* rp, const int* ci, const float* v, const float4* H, float4* T) {
  int lane = threadIdx.x & 31;
  int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) / 32;
  if (row >= n) return;
  int64_t b = rp[row], e = rp[row + 1];
  float a[16] = {0};
  for (int64_t p = b + lane; p < e; p += 32) {
    int c = ci[p]; float w = v[p];
    const float4* q = H + (int64_t)c * 4;
    float4 h0 = NA ? ld_na(q) : __ldg(q), h1 = NA ? ld_na(q + 1) : __ldg(q + 1), h2 = NA ? ld_na(q + 2) : __ldg(q + 2), h3 = NA ? ld_na(q + 3) : __ldg(q + 3);
    a[0] += w * h0.x; a[1] += w * h0.y; a[2] += w * h0.z; a[3] += w * h0.w;
    a[4] += w * h1.x; a[5] += w * h1.y; a[6] += w * h1.z; a[7] += w * h1.w;
    a[8] += w * h2.x; a[9] += w * h2.y; a[10] += w * h2.z; a[11] += w * h2.w;
    a[12] += w * h3.x; a[13] += w * h3.y; a[14] += w * h3.z; a[15] += w * h3.w;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i)
    for (int o = 16; o; o >>= 1) a[i] += __shfl_xor_sync(~0u, a[i], o);
  if (lane < 4) T[row * 4 + lane] = make_float4(a[4 * lane], a[4 * lane + 1], a[4 * lane + 2], a[4 * lane + 3]);
}

// (f): 2 lanes per row, 2 float4 (32 B sector) per lane.
template <bool NA>
__global__ void __launch_bounds__(256) k_lpr2(int n, const int64_t* rp, const int* ci, const float* v, const float4* H, float4* T) {
  int lane = threadIdx.x & 31, sub = lane & 1, grp = lane >> 1;
  int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) / 32 * 16 + grp;
  int64_t b = 0, len = 0;
  if (row < n) { b = rp[row]; len = rp[row + 1] - b; }
  int64_t mx = len;
  for (int o = 16; o >= 2; o >>= 1) { int64_t t = __shfl_xor_sync(~0u, mx, o); mx = t > mx ? t : mx; }
  float4 a0 = make_float4(0, 0, 0, 0), a1 = a0;
  for (int64_t base = 0; base < mx; base += 2) {
    int c = 0; float vv = 0;
    if (base + sub < len) { c = ci[b + base + sub]; vv = v[b + base + sub]; }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      int cc = __shfl_sync(~0u, c, grp * 2 + t); float w = __shfl_sync(~0u, vv, grp * 2 + t);
      const float4* p = H + (int64_t)cc * 4 + sub * 2;
      float4 h0 = NA ? ld_na(p) : __ldg(p), h1 = NA ? ld_na(p + 1) : __ldg(p + 1);
      a0.x += w * h0.x; a0.y += w * h0.y; a0.z += w * h0.z; a0.w += w * h0.w;
      a1.x += w * h1.x; a1.y += w * h1.y; a1.z += w * h1.z; a1.w += w * h1.w;
    }
  }
  if (row < n) { T[row * 4 + sub * 2] = a0; T[row * 4 + sub * 2 + 1] = a1; }
}

// Pure streaming of col/val (lower bound on A traffic).
__global__ void k_stream(int64_t nnz, const int* ci, const float* v, float* out) {
  float s = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) s += ci[p] * v[p];
  if (s == 12345.f) out[0] = s;
}

int main() {
  const int n = 232965, deg = 494;
  const int64_t nnz = (int64_t)n * deg;
  std::vector<int64_t> rp(n + 1);
  std::vector<int> ci(nnz);
  std::vector<float> vv(nnz, 0.001f);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i <= n; ++i) rp[i] = (int64_t)i * deg;
  for (int64_t k = 0; k < nnz; ++k) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; ci[k] = (int)(s % n); }
  for (int i = 0; i < n; ++i) std::sort(ci.begin() + rp[i], ci.begin() + rp[i + 1]);
  int64_t* d_rp; int* d_ci; float* d_v; float4 *d_H, *d_T; float* d_o;
  CK(cudaMalloc(&d_rp, (n + 1) * 8)); CK(cudaMalloc(&d_ci, nnz * 4)); CK(cudaMalloc(&d_v, nnz * 4));
  CK(cudaMalloc(&d_H, (size_t)n * 64)); CK(cudaMalloc(&d_T, (size_t)n * 64)); CK(cudaMalloc(&d_o, 4));
  CK(cudaMemcpy(d_rp, rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_v, vv.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_H, 0, (size_t)n * 64));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-28s %8.3f ms  gather %6.2f TB/s  compulsory %6.2f TB/s\n", name, ms, nnz * 64.0 / ms / 1e9, (nnz * 8.0 + n * 128.0) / ms / 1e9);
  };
  int b4 = (n + 63) / 64, b1 = (n + 7) / 8, b2 = (n + 127) / 128;
  run("stream col/val", [&] { k_stream<<<148 * 8, 256>>>(nnz, d_ci, d_v, d_o); });
  run("lpr4 ldg", [&] { k_lpr4<false, 4><<<b4, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lpr4 L1::no_allocate", [&] { k_lpr4<true, 4><<<b4, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("qpr8 U=2", [&] { k_qpr<8, 2><<<(n + 7) / 8, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("qpr8 U=4", [&] { k_qpr<8, 4><<<(n + 7) / 8, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("qpr8 U=8", [&] { k_qpr<8, 8><<<(n + 7) / 8, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("qpr4 U=4", [&] { k_qpr<4, 4><<<(n + 15) / 16, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("qpr2 U=4", [&] { k_qpr<2, 4><<<(n + 31) / 32, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lpr4u U=1", [&] { k_lpr4u<1><<<b4, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lpr4u U=2", [&] { k_lpr4u<2><<<b4, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lpr4u U=4", [&] { k_lpr4u<4><<<b4, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lane-per-nnz ldg", [&] { k_lane_nnz<false><<<b1, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lane-per-nnz no_alloc", [&] { k_lane_nnz<true><<<b1, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lpr2 ldg", [&] { k_lpr2<false><<<b2, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  run("lpr2 no_alloc", [&] { k_lpr2<true><<<b2, 256>>>(n, d_rp, d_ci, d_v, d_H, d_T); });
  return 0;
}
