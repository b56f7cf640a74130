// Microbenchmark: narrow-f (16) SpMM gathers with 128-bit vs 256-bit loads on a random
// 233K x 233K matrix, 494 nnz/row (sorted).  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_v8 micro_v8.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct F8 { float v[8]; };
template <int NA>
__device__ __forceinline__ F8 ld8(const float* p) {
  F8 r;
  if (NA == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(r.v[0]),"=f"(r.v[1]),"=f"(r.v[2]),"=f"(r.v[3]),"=f"(r.v[4]),"=f"(r.v[5]),"=f"(r.v[6]),"=f"(r.v[7]) : "l"(p));
  else
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(r.v[0]),"=f"(r.v[1]),"=f"(r.v[2]),"=f"(r.v[3]),"=f"(r.v[4]),"=f"(r.v[5]),"=f"(r.v[6]),"=f"(r.v[7]) : "l"(p));
  return r;
}

// LV lanes cover one 16-float row (LV=4: float4 each; LV=2: 8 floats each via v8;
// LV=1: 16 floats via 2 x v8); QPR sub-teams stride over the row's nonzeros.
template <int LV, int QPR, int U, int NA, int THREADS>
__global__ void __launch_bounds__(THREADS) k_row(int n, const int64_t* __restrict__ rp, const int* __restrict__ ci,
                                                 const float* __restrict__ v, const float* __restrict__ H, float* __restrict__ T) {
  constexpr int TEAM = LV * QPR, RPW = 32 / TEAM, W = 16 / LV;
  const int lane = threadIdx.x & 31, sub = lane % LV, q = (lane % TEAM) / LV;
  const int64_t row = ((int64_t)blockIdx.x * THREADS + threadIdx.x) / 32 * RPW + lane / TEAM;
  int64_t p = 0, e = 0;
  if (row < n) { p = rp[row] + q; e = rp[row + 1]; }
  float acc[W];
#pragma unroll
  for (int i = 0; i < W; ++i) acc[i] = 0.f;
  auto gather = [&](int c, float* h) {
    const float* src = H + (int64_t)c * 16 + sub * W;
    if constexpr (W == 4) {
      float4 t = __ldg(reinterpret_cast<const float4*>(src));
      h[0] = t.x; h[1] = t.y; h[2] = t.z; h[3] = t.w;
    } else {
#pragma unroll
      for (int k = 0; k < W / 8; ++k) {
        F8 t = ld8<NA>(src + 8 * k);
#pragma unroll
        for (int j = 0; j < 8; ++j) h[8 * k + j] = t.v[j];
      }
    }
  };
  for (; p + (U - 1) * QPR < e; p += U * QPR) {
    float h[U][W], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = __ldg(ci + p + u * QPR);
      w[u] = __ldg(v + p + u * QPR);
      gather(c, h[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = fmaf(w[u], h[u][i], acc[i]);
  }
  for (; p < e; p += QPR) {
    float h[W];
    gather(__ldg(ci + p), h);
    const float w = __ldg(v + p);
#pragma unroll
    for (int i = 0; i < W; ++i) acc[i] = fmaf(w, h[i], acc[i]);
  }
#pragma unroll
  for (int o = LV; o < TEAM; o <<= 1)
#pragma unroll
    for (int i = 0; i < W; ++i) acc[i] += __shfl_xor_sync(~0u, acc[i], o);
  if (row < n && q == 0) {
#pragma unroll
    for (int i = 0; i < W; i += 4)
      *reinterpret_cast<float4*>(T + row * 16 + sub * W + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
  }
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
  if (FILE* fp = fopen("/tmp/csr_rp.bin", "rb")) {  // product graph dumped by tune_dump.py
    int64_t m = 0;
    fread(rp.data(), 8, n + 1, fp); fclose(fp);
    m = rp[n];
    ci.resize(m); vv.resize(m);
    fp = fopen("/tmp/csr_ci.bin", "rb"); fread(ci.data(), 4, m, fp); fclose(fp);
    fp = fopen("/tmp/csr_v.bin", "rb"); fread(vv.data(), 4, m, fp); fclose(fp);
    printf("loaded product CSR nnz=%lld\n", (long long)m);
  }
  const int64_t nnz_used = rp[n];
  int64_t* d_rp; int* d_ci; float *d_v, *d_H, *d_T;
  CK(cudaMalloc(&d_rp, (n + 1) * 8)); CK(cudaMalloc(&d_ci, nnz_used * 4)); CK(cudaMalloc(&d_v, nnz_used * 4));
  CK(cudaMalloc(&d_H, (size_t)n * 64)); CK(cudaMalloc(&d_T, (size_t)n * 64));
  CK(cudaMemcpy(d_rp, rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci.data(), nnz_used * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_v, vv.data(), nnz_used * 4, cudaMemcpyHostToDevice));
  std::vector<float> hh((size_t)n * 16);
  for (auto& x : hh) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = (s % 1000) * 1e-3f; }
  CK(cudaMemcpy(d_H, hh.data(), hh.size() * 4, cudaMemcpyHostToDevice));
  std::vector<float> ref((size_t)n * 16), got((size_t)n * 16);
  bool have_ref = false;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, int rows_per_block, int threads, auto kern) {
    const int grid = (n + rows_per_block - 1) / rows_per_block;
    for (int i = 0; i < 2; ++i) kern<<<grid, threads>>>(n, d_rp, d_ci, d_v, d_H, d_T);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) kern<<<grid, threads>>>(n, d_rp, d_ci, d_v, d_H, d_T);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    CK(cudaMemcpy(got.data(), d_T, got.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0;
    if (!have_ref) { ref = got; have_ref = true; }
    for (size_t i = 0; i < got.size(); ++i) err = std::max(err, (double)std::abs(got[i] - ref[i]));
    printf("%-34s %8.3f ms  gather %6.2f TB/s  maxdiff %.2e\n", name, ms, nnz * 64.0 / ms / 1e9, err);
  };
#define RUN(LV, QPR, U, NA, TH) run(#LV " lanes QPR=" #QPR " U=" #U " NA=" #NA " T=" #TH, TH / 32 * (32 / (LV * QPR)), TH, k_row<LV, QPR, U, NA, TH>)
  RUN(4, 8, 4, 0, 256);
  RUN(4, 8, 2, 0, 256);
  RUN(4, 8, 4, 0, 128);
  RUN(4, 4, 4, 0, 256);
  RUN(2, 16, 4, 0, 256);
  RUN(2, 16, 2, 0, 256);
  RUN(2, 16, 4, 1, 256);
  RUN(2, 8, 4, 0, 256);
  RUN(2, 16, 8, 0, 256);
  RUN(1, 32, 2, 0, 256);
  RUN(1, 32, 4, 0, 256);
  RUN(1, 16, 4, 0, 256);
  RUN(1, 32, 2, 1, 256);
  return 0;
}
