// Micro-benchmark: shared-memory column-tiled SpMM vs the L1-gather SpMM for
// the Reddit shape (n = 232,965 rows, 494 nonzeros per row, f = 16).
//
// Tiled: CTA b owns a block of rows (quads of 4 lanes, RQ rows per quad) and
// sweeps the columns in tiles of Wc rows of H that TMA bulk-copies into shared
// memory (double-buffered); each quad walks its precomputed entry stream for
// the tile ({row_in_quad << 16 | local col, value}) gathering from shared
// memory.  The L2 then serves one 64 B row of H per (CTA, tile) instead of one
// per nonzero.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_tiled micro_tiled.cu
#include <cuda_runtime.h>
#include <thrust/binary_search.h>
#include <thrust/device_vector.h>
#include <thrust/sort.h>
#include <thrust/sequence.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fma4(float4& a, float w, const float4& h) {
  a.x = fmaf(w, h.x, a.x);
  a.y = fmaf(w, h.y, a.y);
  a.z = fmaf(w, h.z, a.z);
  a.w = fmaf(w, h.w, a.w);
}

// ---- tiled kernel -----------------------------------------------------------------
template <int RQ>
__global__ void __launch_bounds__(1024, 1)
    tiled_kernel(const int2* __restrict__ ent, const uint32_t* __restrict__ desc, const float* __restrict__ H,
                 int64_t n_cols, int T, int Wc, int QPC, int64_t n_rows, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  float4* tile0 = reinterpret_cast<float4*>(sm + 128);
  const int lane = threadIdx.x & 31, l4 = lane & 3;
  const int qid = threadIdx.x >> 2;  // quad in CTA
  const unsigned qmask = 0xFu << (lane & ~3);
  const int64_t gquad = static_cast<int64_t>(blockIdx.x) * QPC + qid;
  const bool live = qid < QPC;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int t0 = static_cast<int>((static_cast<int64_t>(blockIdx.x) * T) / gridDim.x);
  auto stage = [&](int tt) {
    const int t = (tt + t0) % T;
    const int64_t c0 = static_cast<int64_t>(t) * Wc;
    const int64_t rows = n_cols - c0 < Wc ? n_cols - c0 : Wc;
    float4* dst = tile0 + static_cast<size_t>(tt & 1) * Wc * 4;
    mbar_expect(&bar[tt & 1], static_cast<uint32_t>(rows * 64));
    bulk_load(dst, H + c0 * 16, static_cast<uint32_t>(rows * 64), &bar[tt & 1]);
  };
  if (threadIdx.x == 0) stage(0);
  float4 acc[RQ];
#pragma unroll
  for (int r = 0; r < RQ; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int t = 0; t < T; ++t) {
    if (threadIdx.x == 0 && t + 1 < T) stage(t + 1);
    mbar_wait(&bar[t & 1], (t >> 1) & 1);
    const float4* tile = tile0 + static_cast<size_t>(t & 1) * Wc * 4;
    if (live) {
      const size_t d = (static_cast<size_t>(blockIdx.x) * T + (t + t0) % T) * QPC + qid;
      const uint32_t s = desc[d], e = desc[d + 1];
      int cur = 0;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t b = s; b < e; b += 4) {
        int2 my = make_int2(-1, 0);
        if (b + l4 < e) my = __ldg(&ent[b + l4]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int x = __shfl_sync(qmask, my.x, (lane & ~3) | k);
          const float v = __int_as_float(__shfl_sync(qmask, my.y, (lane & ~3) | k));
          if (x >= 0) {
            const int row = x >> 16;
            if (row != cur) {
#pragma unroll
              for (int r = 0; r < RQ; ++r)
                if (r == cur) {
                  acc[r].x += a.x;
                  acc[r].y += a.y;
                  acc[r].z += a.z;
                  acc[r].w += a.w;
                }
              a = make_float4(0.f, 0.f, 0.f, 0.f);
              cur = row;
            }
            fma4(a, v, tile[(x & 0xFFFF) * 4 + l4]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RQ; ++r)
        if (r == cur) {
          acc[r].x += a.x;
          acc[r].y += a.y;
          acc[r].z += a.z;
          acc[r].w += a.w;
        }
    }
    __syncthreads();
  }
  if (live) {
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      const int64_t row = gquad * RQ + r;
      if (row < n_rows) reinterpret_cast<float4*>(out + row * 16)[l4] = acc[r];
    }
  }
}

// ---- tiled kernel with the CTA's entry block and descriptors staged by TMA too ----------
constexpr int kECap = 4608;  // entries per buffer (40 KB)
template <int RQ>
__global__ void __launch_bounds__(1024, 1)
    staged_kernel(const int2* __restrict__ ent, const uint32_t* __restrict__ desc, const float* __restrict__ H,
                  int64_t n_cols, int T, int Wc, int QPC, int64_t n_rows, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  const size_t hbytes = static_cast<size_t>(Wc) * 64;
  const size_t dwords = static_cast<size_t>(QPC) + 8;
  const size_t bufbytes = hbytes + kECap * 8 + 16 + dwords * 4;
  unsigned char* base = sm + 128;
  __shared__ uint32_t ebase_s[2], dbase_s[2];
  __shared__ int over_s[2];
  const int lane = threadIdx.x & 31, l4 = lane & 3;
  const int qid = threadIdx.x >> 2;
  const unsigned qmask = 0xFu << (lane & ~3);
  const int64_t gquad = static_cast<int64_t>(blockIdx.x) * QPC + qid;
  const bool live = qid < QPC;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // CTAs sweep the tiles from staggered starting points, so the SMs do not
  // all pull the same H rows from the same L2 lines at the same moment.
  const int t0 = static_cast<int>((static_cast<int64_t>(blockIdx.x) * T) / gridDim.x);
  auto stage = [&](int tt) {
    const int k = tt & 1;
    const int t = (tt + t0) % T;
    unsigned char* buf = base + k * bufbytes;
    const int64_t c0 = static_cast<int64_t>(t) * Wc;
    const int64_t rows = n_cols - c0 < Wc ? n_cols - c0 : Wc;
    const size_t d0 = (static_cast<size_t>(blockIdx.x) * T + t) * QPC;
    const uint32_t s = desc[d0], e = desc[d0 + QPC];
    const uint32_t ea = s & ~1u, eb = (e + 1) & ~1u;
    const size_t da = d0 & ~static_cast<size_t>(3), db = (d0 + QPC + 1 + 3) & ~static_cast<size_t>(3);
    const bool over = eb - ea > static_cast<uint32_t>(kECap);
    ebase_s[k] = ea;
    dbase_s[k] = static_cast<uint32_t>(d0 - da);
    over_s[k] = over;
    const uint32_t bytes = static_cast<uint32_t>(rows * 64 + (over ? 0 : (eb - ea) * 8) + (db - da) * 4);
    mbar_expect(&bar[k], bytes);
    bulk_load(buf, H + c0 * 16, static_cast<uint32_t>(rows * 64), &bar[k]);
    if (!over && eb > ea) bulk_load(buf + hbytes, ent + ea, (eb - ea) * 8, &bar[k]);
    bulk_load(buf + hbytes + kECap * 8 + 16, desc + da, static_cast<uint32_t>((db - da) * 4), &bar[k]);
  };
  if (threadIdx.x == 0) stage(0);
  float4 acc[RQ];
#pragma unroll
  for (int r = 0; r < RQ; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int t = 0; t < T; ++t) {
    const int k = t & 1;
    if (threadIdx.x == 0 && t + 1 < T) stage(t + 1);
    mbar_wait(&bar[k], (t >> 1) & 1);
    unsigned char* buf = base + k * bufbytes;
    const float4* tile = reinterpret_cast<const float4*>(buf);
    const int2* sent = reinterpret_cast<const int2*>(buf + hbytes);
    const uint32_t* sdesc = reinterpret_cast<const uint32_t*>(buf + hbytes + kECap * 8 + 16) + dbase_s[k];
    const uint32_t eb0 = ebase_s[k];
    const bool over = over_s[k];
    {
      // Warp-uniform trip count: every quad runs the warp's longest stream,
      // predicated, so shuffles use the full mask and quads never diverge.
      uint32_t s = 0, e = 0;
      if (live) {
        s = sdesc[qid];
        e = sdesc[qid + 1];
      }
      uint32_t len = e - s, mx = len;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      int cur = 0;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t j = 0; j < mx; j += 4) {
        const uint32_t b = s + j;
        int2 my = make_int2(-1, 0);
        if (j + l4 < len) my = over ? __ldg(&ent[b + l4]) : sent[b + l4 - eb0];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int x = __shfl_sync(0xffffffffu, my.x, (lane & ~3) | kk);
          const float v = __int_as_float(__shfl_sync(0xffffffffu, my.y, (lane & ~3) | kk));
          const int row = x >> 16;
          if (x >= 0 && row != cur) {
#pragma unroll
            for (int r = 0; r < RQ; ++r)
              if (r == cur) {
                acc[r].x += a.x;
                acc[r].y += a.y;
                acc[r].z += a.z;
                acc[r].w += a.w;
              }
            a = make_float4(0.f, 0.f, 0.f, 0.f);
            cur = row;
          }
          const float4 h = tile[(x >= 0 ? (x & 0xFFFF) : 0) * 4 + l4];
          fma4(a, x >= 0 ? v : 0.f, h);
        }
      }
#pragma unroll
      for (int r = 0; r < RQ; ++r)
        if (r == cur) {
          acc[r].x += a.x;
          acc[r].y += a.y;
          acc[r].z += a.z;
          acc[r].w += a.w;
        }
    }
    __syncthreads();
  }
  if (live) {
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      const int64_t row = gquad * RQ + r;
      if (row < n_rows) reinterpret_cast<float4*>(out + row * 16)[l4] = acc[r];
    }
  }
}

// ---- L1-gather baseline (warp per row, 8 sub-teams of 4 lanes, 4 in flight) --------
__global__ void __launch_bounds__(128) csr_kernel(const int2* __restrict__ cv, int deg, const float* __restrict__ H,
                                                  int64_t n_rows, float* __restrict__ out) {
  const int lane = threadIdx.x & 31, l4 = lane & 3, q = lane >> 2;
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * 128 + threadIdx.x) >> 5;
  if (row >= n_rows) return;
  const int2* p = cv + row * deg + q;
  const int2* pe = cv + (row + 1) * deg;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (; p + 24 < pe; p += 32) {
    int2 x[4];
    float4 h[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldg(p + u * 8);
#pragma unroll
    for (int u = 0; u < 4; ++u) h[u] = __ldg(reinterpret_cast<const float4*>(H + static_cast<int64_t>(x[u].x) * 16) + l4);
#pragma unroll
    for (int u = 0; u < 4; ++u) fma4(acc, __int_as_float(x[u].y), h[u]);
  }
  for (; p < pe; p += 8) {
    const int2 x = __ldg(p);
    fma4(acc, __int_as_float(x.y), __ldg(reinterpret_cast<const float4*>(H + static_cast<int64_t>(x.x) * 16) + l4));
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (q == 0) reinterpret_cast<float4*>(out + row * 16)[l4] = acc;
}

// ---- data ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
__global__ void gen_csr(int64_t nnz, int deg, int64_t n, int2* cv, int parity_rq) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix(static_cast<uint64_t>(k) + 12345);
    int c = static_cast<int>(h % static_cast<uint64_t>(n));
    // Idealised pairing: quad q only touches columns of parity q & 1, so the
    // two quads of a quarter-warp never collide on a shared-memory bank half.
    if (parity_rq) c = (c & ~1) | static_cast<int>(((k / deg) / parity_rq) & 1);
    if (c >= n) c -= 2;
    cv[k] = make_int2(c, __float_as_int(0.001f * static_cast<float>(1 + (h >> 40) % 1000)));
  }
}
__global__ void gen_keys(int64_t nnz, int deg, const int2* cv, int RQ, int QPC, int T, int Wc, uint64_t* keys,
                         int2* ent) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / deg;
    const int c = cv[k].x;
    const int64_t quad = r / RQ;
    const int64_t b = quad / QPC, q = quad % QPC;
    const int t = c / Wc;
    keys[k] = ((static_cast<uint64_t>(b) * T + t) * QPC + q) * 8 + static_cast<uint64_t>(r % RQ);
    ent[k] = make_int2(static_cast<int>((r % RQ) << 16) | (c % Wc), cv[k].y);
  }
}
__global__ void fill_h(int64_t n, float* H) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 16; i += (int64_t)gridDim.x * blockDim.x)
    H[i] = static_cast<float>((mix(i) >> 41) % 1000) * 1e-3f - 0.5f;
}

template <int RQ>
float run_tiled(const int2* cv, int64_t n, int deg, int NW, int Wc, const float* H, float* out, int reps,
                bool staged) {
  const int QPC = NW * 8;
  const int64_t rows_per_cta = static_cast<int64_t>(QPC) * RQ;
  const int B = static_cast<int>((n + rows_per_cta - 1) / rows_per_cta);
  const int T = static_cast<int>((n + Wc - 1) / Wc);
  const int64_t nnz = n * deg;
  thrust::device_vector<uint64_t> keys(nnz);
  thrust::device_vector<int2> ent(nnz);
  gen_keys<<<2048, 256>>>(nnz, deg, cv, RQ, QPC, T, Wc, thrust::raw_pointer_cast(keys.data()),
                          thrust::raw_pointer_cast(ent.data()));
  CK(cudaGetLastError());
  thrust::stable_sort_by_key(keys.begin(), keys.end(), ent.begin());
  const int64_t nd = static_cast<int64_t>(B) * T * QPC + 1;
  thrust::device_vector<uint64_t> probes(nd);
  thrust::sequence(probes.begin(), probes.end(), 0ull, 8ull);
  thrust::device_vector<uint32_t> desc(nd);
  thrust::lower_bound(keys.begin(), keys.end(), probes.begin(), probes.end(), desc.begin());
  const size_t smem = staged ? 128 + 2 * (static_cast<size_t>(Wc) * 64 + kECap * 8 + 16 + (QPC + 8) * 4)
                             : 128 + 2ull * Wc * 64;
  auto kern = staged ? staged_kernel<RQ> : tiled_kernel<RQ>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i)
    kern<<<B, NW * 32, smem>>>(thrust::raw_pointer_cast(ent.data()), thrust::raw_pointer_cast(desc.data()),
                                           H, n, T, Wc, QPC, n, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i)
    kern<<<B, NW * 32, smem>>>(thrust::raw_pointer_cast(ent.data()), thrust::raw_pointer_cast(desc.data()),
                                           H, n, T, Wc, QPC, n, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("%s RQ=%d NW=%d Wc=%d CTAs=%d tiles=%d smem=%zu: %.4f ms\n", staged ? "staged" : "tiled", RQ, NW, Wc, B,
         T, smem, ms / reps);
  return ms / reps;
}

int main() {
  for (int parity = 0; parity < 2; ++parity) {
  printf("=== %s column parities ===\n", parity ? "paired (ideal)" : "random");
  const int64_t n = 232965;
  const int deg = 494;
  const int64_t nnz = n * deg;
  int2* cv;
  float *H, *o1, *o2;
  CK(cudaMalloc(&cv, nnz * sizeof(int2)));
  CK(cudaMalloc(&H, n * 16 * sizeof(float)));
  CK(cudaMalloc(&o1, n * 16 * sizeof(float)));
  CK(cudaMalloc(&o2, n * 16 * sizeof(float)));
  gen_csr<<<2048, 256>>>(nnz, deg, n, cv, parity ? 7 : 0);
  fill_h<<<2048, 256>>>(n, H);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 20;
  const unsigned g = static_cast<unsigned>((n * 32 + 127) / 128);
  csr_kernel<<<g, 128>>>(cv, deg, H, n, o1);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) csr_kernel<<<g, 128>>>(cv, deg, H, n, o1);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("L1-gather CSR: %.4f ms\n", ms / reps);
  std::vector<float> h1(n * 16), h2(n * 16);
  CK(cudaMemcpy(h1.data(), o1, n * 64, cudaMemcpyDeviceToHost));
  struct Cfg { int rq, nw, wc; bool st; };
  for (Cfg c : {Cfg{7, 29, 1536, false}, Cfg{7, 29, 1024, true}, Cfg{7, 29, 1792, false}}) {
    CK(cudaMemset(o2, 0, n * 64));
    switch (c.rq) {
      case 7: run_tiled<7>(cv, n, deg, c.nw, c.wc, H, o2, reps, c.st); break;
    }
    CK(cudaMemcpy(h2.data(), o2, n * 64, cudaMemcpyDeviceToHost));
    double err = 0, nrm = 0;
    for (int64_t i = 0; i < n * 16; ++i) {
      err += (h1[i] - h2[i]) * (double)(h1[i] - h2[i]);
      nrm += h1[i] * (double)h1[i];
    }
    printf("   rel err vs CSR = %.3e\n", std::sqrt(err / nrm));
  }
  cudaFree(cv); cudaFree(H); cudaFree(o1); cudaFree(o2);
  }
  return 0;
}
