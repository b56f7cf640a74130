// Microbenchmark: the 1D stage exchange on N GPUs of one box (single process, peer access):
// every GPU pushes its panel slot (rows x 16 floats) into every peer's buffer at once.
// Variants: the product publish kernel shape, destination-major grids, grid sizes,
// copy-engine peer copies, and (when supported) an NVLS multicast store through a
// multicast object.  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_push micro_push.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1);} } while (0)
#define CU(x) do { CUresult e = (x); if (e != CUDA_SUCCESS) { const char* m; cuGetErrorString(e, &m); printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, m); return false;} } while (0)

constexpr int MAXG = 8;
struct Dst { float4* p[MAXG]; };

// Product shape: element loop, every element stored to all destinations.
__global__ void push_all(Dst d, int P, int self, const float4* __restrict__ src, int64_t n4, int64_t off4) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[e];
#pragma unroll 4
    for (int k = 1; k < P; ++k) d.p[(self + k) % P][off4 + e] = v;
  }
}
// Destination-major: blockIdx.y picks the peer.
__global__ void push_dst(Dst d, int P, int self, const float4* __restrict__ src, int64_t n4, int64_t off4) {
  float4* dst = d.p[(self + 1 + blockIdx.y) % P] + off4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}
// Destination-major with 4 independent 16 B stores per thread per iteration.
__global__ void push_dst4(Dst d, int P, int self, const float4* __restrict__ src, int64_t n4, int64_t off4) {
  float4* dst = d.p[(self + 1 + blockIdx.y) % P] + off4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; e + 3 * stride < n4; e += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = src[e + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[e + u * stride] = v[u];
  }
  for (; e < n4; e += stride) dst[e] = src[e];
}
// NVLS: one multimem store reaches every GPU bound to the multicast object.
__global__ void push_mc(float4* mc, const float4* __restrict__ src, int64_t n4, int64_t off4) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[e];
    float4* p = mc + off4 + e;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
}

int G = 0;
int64_t rows = 0;
float4* buf[MAXG];
float4* src[MAXG];
cudaStream_t st[MAXG][MAXG];
cudaEvent_t e0[MAXG], e1[MAXG];

template <typename F>
void timeit(const char* name, F launch_on) {
  for (int it = 0; it < 3; ++it) {
    for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); launch_on(g); }
    for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
  }
  const int reps = 20;
  for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaEventRecord(e0[g], st[g][0])); }
  for (int r = 0; r < reps; ++r)
    for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); launch_on(g); }
  float worst = 0;
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(e1[g], st[g][0]));
    CK(cudaEventSynchronize(e1[g]));
    float ms; CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
    worst = ms > worst ? ms : worst;
  }
  const double us = worst / reps * 1e3;
  const double egress = (double)rows * 64 * (G - 1);
  printf("%-44s %7.1f us  egress/GPU %6.1f GB/s\n", name, us, egress / us / 1e3);
}

bool setup_mc(size_t bytes, float4** mc_ptr, float4** uc) {
  CU(cuInit(0));
  int sup = 0;
  CUdevice dev0; CU(cuDeviceGet(&dev0, 0));
  CU(cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev0));
  printf("multicast supported: %d\n", sup);
  if (!sup) return false;
  CUmulticastObjectProp mp = {};
  mp.numDevices = G;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  bytes = (bytes + gran - 1) / gran * gran;
  mp.size = bytes;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int g = 0; g < G; ++g) { CUdevice d; CU(cuDeviceGet(&d, g)); CU(cuMulticastAddDevice(mc, d)); }
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle h;
    CU(cuMemCreate(&h, bytes, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, h, 0, bytes, 0));
    CUdeviceptr va;
    CU(cuMemAddressReserve(&va, bytes, gran, 0, 0));
    CU(cuMemMap(va, bytes, 0, h, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = g;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(va, bytes, &ad, 1));
    uc[g] = reinterpret_cast<float4*>(va);
    CUdeviceptr mva;
    CU(cuMemAddressReserve(&mva, bytes, gran, 0, 0));
    CU(cuMemMap(mva, bytes, 0, mc, 0));
    CU(cuMemSetAccess(mva, bytes, &ad, 1));
    mc_ptr[g] = reinterpret_cast<float4*>(mva);
  }
  return true;
}

int main(int argc, char** argv) {
  CK(cudaGetDeviceCount(&G));
  if (G > MAXG) G = MAXG;
  // argv[1]: graph rows multiplier (1 = Reddit: a 16-float panel of 232,965 rows).
  const int64_t n = 232965LL * (argc > 1 ? atoi(argv[1]) : 1);
  rows = (n + G - 1) / G;
  const int64_t n4 = rows * 4;  // 16 floats per row
  printf("GPUs %d, rows per slot %lld (%.2f MB)\n", G, (long long)rows, rows * 64 / 1e6);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int q = 0; q < G; ++q) if (q != g) { cudaDeviceEnablePeerAccess(q, 0); cudaGetLastError(); }
    CK(cudaMalloc(&buf[g], G * n4 * 16));
    CK(cudaMalloc(&src[g], n4 * 16));
    CK(cudaMemset(src[g], 1, n4 * 16));
    for (int k = 0; k < G; ++k) CK(cudaStreamCreateWithFlags(&st[g][k], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g])); CK(cudaEventCreate(&e1[g]));
  }
  Dst d;
  for (int g = 0; g < G; ++g) d.p[g] = buf[g];
  int sms = 148;
  for (int mult : {2, 4, 8}) {
    char name[64];
    snprintf(name, sizeof name, "push_all grid %dx148 x256 (product)", mult);
    timeit(name, [&](int g) { push_all<<<mult * sms, 256, 0, st[g][0]>>>(d, G, g, src[g], n4, g * n4); });
  }
  for (int per : {1, 2, 4}) {
    char name[64];
    snprintf(name, sizeof name, "push_dst grid %dx148/(P-1) per peer", per);
    timeit(name, [&](int g) { push_dst<<<dim3(per * sms / (G - 1) + 1, G - 1), 256, 0, st[g][0]>>>(d, G, g, src[g], n4, g * n4); });
    snprintf(name, sizeof name, "push_dst4 grid %dx148/(P-1) per peer", per);
    timeit(name, [&](int g) { push_dst4<<<dim3(per * sms / (G - 1) + 1, G - 1), 256, 0, st[g][0]>>>(d, G, g, src[g], n4, g * n4); });
  }
  timeit("copy engine: cudaMemcpyAsync per peer (1 stream)", [&](int g) {
    for (int k = 1; k < G; ++k) { const int q = (g + k) % G; CK(cudaMemcpyAsync(buf[q] + g * n4, src[g], n4 * 16, cudaMemcpyDeviceToDevice, st[g][0])); }
  });
  timeit("copy engine: per peer on its own stream", [&](int g) {
    for (int k = 1; k < G; ++k) { const int q = (g + k) % G; CK(cudaMemcpyAsync(buf[q] + g * n4, src[g], n4 * 16, cudaMemcpyDeviceToDevice, st[g][k])); }
    for (int k = 1; k < G; ++k) { cudaEvent_t ev; CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)); CK(cudaEventRecord(ev, st[g][k])); CK(cudaStreamWaitEvent(st[g][0], ev, 0)); CK(cudaEventDestroy(ev)); }
  });
  float4* mc[MAXG];
  float4* uc[MAXG];
  if (setup_mc(G * n4 * 16, mc, uc)) {
    for (int mult : {1, 2, 4}) {
      char name[64];
      snprintf(name, sizeof name, "multimem.st grid %dx148 (NVLS multicast)", mult);
      timeit(name, [&](int g) { push_mc<<<mult * sms, 256, 0, st[g][0]>>>(mc[g], src[g], n4, g * n4); });
    }
    // check: every GPU's unicast view holds every slot
    std::vector<float> h(4);
    CK(cudaSetDevice(G - 1));
    CK(cudaMemcpy(h.data(), uc[G - 1], 16, cudaMemcpyDeviceToHost));
    printf("mc check %g\n", h[0]);
  }
  return 0;
}
