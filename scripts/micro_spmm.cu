// Microbenchmark of the production SpMM (spmm.cu) on a random 233K x 233K
// matrix with 494 nnz/row (Reddit-shaped), for several feature widths.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2005_03300_b200/csrc \
//      -o micro_spmm micro_spmm.cu ../paper_2005_03300_b200/csrc/spmm.cu
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

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


int main(int argc, char** argv) {
  const int n = 232965, deg = 494;
  const int64_t nnz = static_cast<int64_t>(n) * deg;
  std::vector<int64_t> rp(n + 1);
  std::vector<int> ci(nnz);
  std::vector<float> vv(nnz, 0.001f);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i <= n; ++i) rp[i] = static_cast<int64_t>(i) * deg;
  for (int64_t k = 0; k < nnz; ++k) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    ci[k] = static_cast<int>(s % n);
  }
  for (int i = 0; i < n; ++i) std::sort(ci.begin() + rp[i], ci.begin() + rp[i + 1]);
  cagnet::DevBuf<int64_t> d_rp(n + 1);
  cagnet::DevBuf<int32_t> d_ci(nnz);
  cagnet::DevBuf<float> d_v(nnz);
  CG_CUDA(cudaMemcpy(d_rp.get(), rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CG_CUDA(cudaMemcpy(d_ci.get(), ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CG_CUDA(cudaMemcpy(d_v.get(), vv.data(), nnz * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int f : {16, 41, 602}) {
    const int64_t ld = cagnet::padded_ld(f);
    cagnet::DevBuf<float> H(static_cast<size_t>(n) * ld), T(static_cast<size_t>(n) * ld);
    CG_CUDA(cudaMemset(H.get(), 0, static_cast<size_t>(n) * ld * 4));
    auto launch = [&] {
      cagnet::kern::spmm_csr(n, d_rp.get(), d_ci.get(), d_v.get(), H.get(), ld, f, T.get(), ld, false, 0, nnz);
    };
    launch();
    CG_CUDA(cudaDeviceSynchronize());
    const int reps = f > 100 ? 3 : 20;
    if (f == 16) {
      auto l2 = [&] { k_lpr4u<2><<<(n + 63) / 64, 256>>>(n, d_rp.get(), d_ci.get(), d_v.get(), (const float4*)H.get(), (float4*)T.get()); };
      for (int i = 0; i < 3; ++i) l2();
      cudaEventRecord(a);
      for (int i = 0; i < reps; ++i) l2();
      cudaEventRecord(b);
      CG_CUDA(cudaEventSynchronize(b));
      float ms2;
      cudaEventElapsedTime(&ms2, a, b);
      printf("micro lpr4u<2> f=16 %8.3f ms\n", ms2 / reps);
    }
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    CG_CUDA(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("%s f=%4d  %8.3f ms  gather %6.2f TB/s\n", argc > 1 ? argv[1] : "", f, ms,
           nnz * 4.0 * ld / ms / 1e9);
  }
  return 0;
}
