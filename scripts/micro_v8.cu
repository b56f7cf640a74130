// Microbenchmark: narrow-f (16) SpMM gathers with 128-bit vs 256-bit loads on a random
// 233K x 233K matrix, 494 nnz/row (sorted).  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_v8 micro_v8.cu
#include <algorithm>
#include <cmath>
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
      float4 t;
      if constexpr (NA == 0) t = __ldg(reinterpret_cast<const float4*>(src));
      else if constexpr (NA == 1)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x),"=f"(t.y),"=f"(t.z),"=f"(t.w) : "l"(src));
      else if constexpr (NA == 2)
        asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x),"=f"(t.y),"=f"(t.z),"=f"(t.w) : "l"(src));
      else if constexpr (NA == 3)
        asm volatile("ld.global.nc.L1::evict_first.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x),"=f"(t.y),"=f"(t.z),"=f"(t.w) : "l"(src));
      else if constexpr (NA == 4)
        asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x),"=f"(t.y),"=f"(t.z),"=f"(t.w) : "l"(src));
      else
        asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x),"=f"(t.y),"=f"(t.z),"=f"(t.w) : "l"(src));
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


// The product's stream form: interleaved {col, val} int2 entries; PEEL = walk from the
// QPR-aligned entry at or below the row start (the head group range-predicated).
template <int PEEL, int THREADS>
__global__ void __launch_bounds__(THREADS, 2048 / THREADS) k_row_cv(int n, const int64_t* __restrict__ rp, const int2* __restrict__ cv,
                                                   const float* __restrict__ H, float* __restrict__ T) {
  constexpr int LV = 4, QPR = 8, U = 4;
  const int lane = threadIdx.x & 31, vec = lane % LV, q = lane / LV;
  const int64_t row = ((int64_t)blockIdx.x * THREADS + threadIdx.x) / 32;
  int64_t b = 0, e = 0;
  if (row < n) { b = rp[row]; e = rp[row + 1]; }
  const char* hbase = reinterpret_cast<const char*>(H) + vec * 16;
  auto gather = [&](int c) { return __ldg(reinterpret_cast<const float4*>(hbase + (uint64_t)(uint32_t)c * 64u)); };
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  auto fma4 = [&](float w, float4 h) { acc.x = fmaf(w, h.x, acc.x); acc.y = fmaf(w, h.y, acc.y); acc.z = fmaf(w, h.z, acc.z); acc.w = fmaf(w, h.w, acc.w); };
  const int2* pe = cv + e;
  const int2* p = cv + b + q;
  if (PEEL) {
    const int64_t head = b & ~(int64_t)(QPR - 1);
    if (head != b) {
      const int2* hp = cv + head + q;
      if (hp >= cv + b && hp < pe) { const int2 x = __ldg(hp); fma4(__int_as_float(x.y), gather(x.x)); }
      p = hp + QPR;
    }
  }
  for (; p + (U - 1) * QPR < pe; p += U * QPR) {
    float4 h[U]; float w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { const int2 x = __ldg(p + u * QPR); w[u] = __int_as_float(x.y); h[u] = gather(x.x); }
#pragma unroll
    for (int u = 0; u < U; ++u) fma4(w[u], h[u]);
  }
  for (; p < pe; p += QPR) { const int2 x = __ldg(p); fma4(__int_as_float(x.y), gather(x.x)); }
#pragma unroll
  for (int o = LV; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(~0u, acc.x, o); acc.y += __shfl_xor_sync(~0u, acc.y, o);
    acc.z += __shfl_xor_sync(~0u, acc.z, o); acc.w += __shfl_xor_sync(~0u, acc.w, o);
  }
  if (row < n && q == 0) *reinterpret_cast<float4*>(T + row * 16 + vec * 4) = acc;
}

// Packed entries: u32 = (degree of the column vertex << CB) | column; the value is
// rebuilt as s_row * rsqrt(d_col) (the normalized adjacency's 1/sqrt(d_r d_c)).
template <int THREADS>
__global__ void __launch_bounds__(THREADS, 2048 / THREADS) k_row_pk(int n, const int64_t* __restrict__ rp, const uint32_t* __restrict__ pk,
                                                   const float* __restrict__ rs, int cb, const float* __restrict__ H, float* __restrict__ T) {
  constexpr int LV = 4, QPR = 8, U = 4;
  const int lane = threadIdx.x & 31, vec = lane % LV, q = lane / LV;
  const int64_t row = ((int64_t)blockIdx.x * THREADS + threadIdx.x) / 32;
  int64_t b = 0, e = 0;
  if (row < n) { b = rp[row]; e = rp[row + 1]; }
  const char* hbase = reinterpret_cast<const char*>(H) + vec * 16;
  const uint32_t cmask = (1u << cb) - 1u;
  auto gather = [&](uint32_t c) { return __ldg(reinterpret_cast<const float4*>(hbase + (uint64_t)c * 64u)); };
  auto weight = [&](uint32_t x) { return rsqrtf(static_cast<float>(x >> cb)); };
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  auto fma4 = [&](float w, float4 h) { acc.x = fmaf(w, h.x, acc.x); acc.y = fmaf(w, h.y, acc.y); acc.z = fmaf(w, h.z, acc.z); acc.w = fmaf(w, h.w, acc.w); };
  const uint32_t* pe = pk + e;
  const uint32_t* p = pk + b + q;
  const int64_t head = b & ~(int64_t)(QPR - 1);
  if (head != b) {
    const uint32_t* hp = pk + head + q;
    if (hp >= pk + b && hp < pe) { const uint32_t x = __ldg(hp); fma4(weight(x), gather(x & cmask)); }
    p = hp + QPR;
  }
  for (; p + (U - 1) * QPR < pe; p += U * QPR) {
    float4 h[U]; float w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { const uint32_t x = __ldg(p + u * QPR); w[u] = weight(x); h[u] = gather(x & cmask); }
#pragma unroll
    for (int u = 0; u < U; ++u) fma4(w[u], h[u]);
  }
  for (; p < pe; p += QPR) { const uint32_t x = __ldg(p); fma4(weight(x), gather(x & cmask)); }
#pragma unroll
  for (int o = LV; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(~0u, acc.x, o); acc.y += __shfl_xor_sync(~0u, acc.y, o);
    acc.z += __shfl_xor_sync(~0u, acc.z, o); acc.w += __shfl_xor_sync(~0u, acc.w, o);
  }
  if (row < n && q == 0) {
    const float sr = rs[row];
    *reinterpret_cast<float4*>(T + row * 16 + vec * 4) = make_float4(sr * acc.x, sr * acc.y, sr * acc.z, sr * acc.w);
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
  std::vector<int> degv(n);
  for (int i = 0; i < n; ++i) degv[i] = (int)(rp[i + 1] - rp[i]);
  for (int i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) vv[k] = (float)(1.0 / sqrt((double)degv[i] * (double)degv[ci[k]]));
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
  {
    std::vector<int2> cvh(nnz_used);
    for (int64_t k = 0; k < nnz_used; ++k) cvh[k] = make_int2(ci[k], *reinterpret_cast<int*>(&vv[k]));
    int2* d_cv; CK(cudaMalloc(&d_cv, nnz_used * 8));
    CK(cudaMemcpy(d_cv, cvh.data(), nnz_used * 8, cudaMemcpyHostToDevice));
    auto cvrun = [&](const char* name, auto kern) {
      auto wrap = [&](int n_, const int64_t* rp_, const int*, const float*, const float* H_, float* T_) {};
      (void)wrap;
      const int grid = (n + 3) / 4;
      for (int i = 0; i < 2; ++i) kern<<<grid, 128>>>(n, d_rp, d_cv, d_H, d_T);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) kern<<<grid, 128>>>(n, d_rp, d_cv, d_H, d_T);
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      printf("%-34s %8.3f ms  gather %6.2f TB/s\n", name, ms, nnz * 64.0 / ms / 1e9);
    };
    cvrun("cv stream, head peel", k_row_cv<1, 128>);
    std::vector<float> ref_cv((size_t)n * 16);
    CK(cudaMemcpy(ref_cv.data(), d_T, ref_cv.size() * 4, cudaMemcpyDeviceToHost));
    {
      int cb = 1; while ((1 << cb) < n) ++cb;
      std::vector<uint32_t> pkh(nnz_used); std::vector<float> rsh(n);
      for (int i = 0; i < n; ++i) rsh[i] = (float)(1.0 / sqrt((double)degv[i]));
      for (int64_t k = 0; k < nnz_used; ++k) pkh[k] = ((uint32_t)degv[ci[k]] << cb) | (uint32_t)ci[k];
      uint32_t* d_pk; float* d_rs;
      CK(cudaMalloc(&d_pk, nnz_used * 4)); CK(cudaMalloc(&d_rs, n * 4));
      CK(cudaMemcpy(d_pk, pkh.data(), nnz_used * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(d_rs, rsh.data(), n * 4, cudaMemcpyHostToDevice));
      const int grid = (n + 3) / 4;
      for (int i = 0; i < 2; ++i) k_row_pk<128><<<grid, 128>>>(n, d_rp, d_pk, d_rs, cb, d_H, d_T);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) k_row_pk<128><<<grid, 128>>>(n, d_rp, d_pk, d_rs, cb, d_H, d_T);
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      std::vector<float> got_pk((size_t)n * 16);
      CK(cudaMemcpy(got_pk.data(), d_T, got_pk.size() * 4, cudaMemcpyDeviceToHost));
      double rel = 0;
      for (size_t i = 0; i < got_pk.size(); ++i) rel = std::max(rel, (double)std::abs(got_pk[i] - ref_cv[i]) / (std::abs(ref_cv[i]) + 1e-3));
      printf("%-34s %8.3f ms  gather %6.2f TB/s  max rel diff vs cv %.2e (cb=%d)\n", "packed u32 + row scale", ms, nnz * 64.0 / ms / 1e9, rel, cb);
    }
    cvrun("cv stream, no peel", k_row_cv<0, 128>);
  }
  RUN(4, 8, 4, 0, 128);
  RUN(4, 8, 4, 1, 128);
  RUN(4, 8, 4, 2, 128);
  RUN(4, 8, 4, 3, 128);
  RUN(4, 8, 4, 4, 128);
  RUN(4, 8, 4, 5, 128);
  RUN(4, 8, 4, 0, 128);
  return 0;
}
