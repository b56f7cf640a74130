// Microbenchmark: TMA tile::gather4 throughput for random 64 B rows (f=16 fp32)
// vs the LDG gather path.  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_tma_gather micro_tma_gather.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void gather4(void* smem, const CUtensorMap* map, uint64_t* bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               :: "r"(smem_u32(smem)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}

// Each CTA: 1 warp.  Lanes 0..G-1 each issue one gather4 per batch (4 rows of 64 B),
// STAGES batches in flight; after a batch lands, lane 0 re-arms it for the next one.
template <int STAGES, int G>
__global__ void __launch_bounds__(32) k_tma(const __grid_constant__ CUtensorMap map, const int* __restrict__ ci, int64_t nnz, float* out) {
  __shared__ __align__(128) float buf[STAGES][G * 4 * 16];
  __shared__ uint64_t bar[STAGES];
  const int lane = threadIdx.x;
  if (lane == 0) for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t per_batch = 4 * G;
  const int64_t nb = nnz / per_batch;
  float sink = 0.f;
  int64_t b = blockIdx.x;
  const int64_t stride = gridDim.x;
  // prologue
  for (int s = 0; s < STAGES; ++s) {
    const int64_t bb = b + s * stride;
    if (bb < nb) {
      if (lane == 0) mbar_expect_tx(&bar[s], G * 4 * 64);
      __syncwarp();
      if (lane < G) {
        const int* c = ci + bb * per_batch + lane * 4;
        gather4(&buf[s][lane * 64], &map, &bar[s], 0, c[0], c[1], c[2], c[3]);
      }
    }
  }
  uint32_t phase[STAGES] = {0};
  for (int64_t it = 0;; ++it) {
    const int s = it % STAGES;
    const int64_t bb = b + it * stride;
    if (bb >= nb) break;
    mbar_wait(&bar[s], phase[s]);
    phase[s] ^= 1;
    sink += buf[s][lane];
    __syncwarp();
    const int64_t nx = bb + STAGES * stride;
    if (nx < nb) {
      if (lane == 0) mbar_expect_tx(&bar[s], G * 4 * 64);
      __syncwarp();
      if (lane < G) {
        const int* c = ci + nx * per_batch + lane * 4;
        gather4(&buf[s][lane * 64], &map, &bar[s], 0, c[0], c[1], c[2], c[3]);
      }
    }
  }
  if (sink == 12345.f) out[0] = sink;
}

__global__ void k_ldg(const float4* __restrict__ H, const int* __restrict__ ci, int64_t nnz, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const int lane = threadIdx.x & 3;
  for (int64_t p = (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) / 4; p < nnz; p += (int64_t)gridDim.x * blockDim.x / 4) {
    float4 h = __ldg(H + (int64_t)ci[p] * 4 + lane);
    acc.x += h.x; acc.y += h.y; acc.z += h.z; acc.w += h.w;
  }
  if (acc.x == 12345.f) out[0] = acc.y;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 232965;
  const int64_t nnz = (int64_t)n * 494;
  std::vector<int> ci(nnz);
  uint64_t s = 88172645463325252ull;
  for (int64_t k = 0; k < nnz; ++k) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; ci[k] = (int)(s % n); }
  int* d_ci; float* d_H; float* d_o;
  CK(cudaMalloc(&d_ci, nnz * 4)); CK(cudaMalloc(&d_H, (size_t)n * 64)); CK(cudaMalloc(&d_o, 4));
  CK(cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_H, 0, (size_t)n * 64));
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {16, (cuuint64_t)n};
  cuuint64_t strides[1] = {64};
  cuuint32_t box[2] = {16, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d_H, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-26s %8.3f ms  gather %6.2f TB/s\n", name, ms, nnz * 64.0 / ms / 1e9);
  };
  run("ldg 4 lanes/row", [&] { k_ldg<<<148 * 16, 256>>>((const float4*)d_H, d_ci, nnz, d_o); });
  run("tma gather4 S=8 G=8 x16", [&] { k_tma<8, 8><<<148 * 16, 32>>>(map, d_ci, nnz, d_o); });
  run("tma gather4 S=8 G=8 x32", [&] { k_tma<8, 8><<<148 * 32, 32>>>(map, d_ci, nnz, d_o); });
  run("tma gather4 S=16 G=8 x16", [&] { k_tma<16, 8><<<148 * 16, 32>>>(map, d_ci, nnz, d_o); });
  run("tma gather4 S=4 G=32 x16", [&] { k_tma<4, 32><<<148 * 16, 32>>>(map, d_ci, nnz, d_o); });
  run("tma gather4 S=8 G=16 x32", [&] { k_tma<8, 16><<<148 * 32, 32>>>(map, d_ci, nnz, d_o); });
  CK(cudaGetLastError());
  return 0;
}
