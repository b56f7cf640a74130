// K2b — persistent, warp-specialised tcgen05 split-TF32 GEMM with a TMA-fed
// A operand, for the tall-skinny products T·W / H·W / S·Wᵀ (M = rows of a
// tile, K = f_in up to ~700, N <= 64): C (+)= A · op(B), A row-major with
// 16 B-aligned rows.
//
// Roles (one CTA per SM, static round-robin over 128-row M tiles):
//   warp 0  TMA producer  streams A k-blocks (128 x 32 fp32, SWIZZLE_128B)
//                         into a shared-memory ring, gated by `empty`;
//   warp 1  MMA issuer    one elected lane issues the 3 x 4 kind::tf32 MMAs
//                         of a k-block (hi·hi, hi·lo, lo·hi) into one of four
//                         TMEM accumulator chains, commits `empty` and, at a
//                         tile's end, `tmem_full`;
//   warps 2-5 converters  split each landed tile in place (hi) plus a lo copy
//                         (same swizzled position), arrive on `conv`; at a
//                         tile's end they drain TMEM (tcgen05.ld) through the
//                         fused epilogue and release the accumulator set.
// Two TMEM accumulator sets let the MMAs of tile t+1 overlap the epilogue of
// tile t.  All of B (hi + lo) stays resident in shared memory.
#include <cuda.h>

#include <atomic>

#include "common.cuh"
#include "kernels.cuh"
#include "tc.cuh"

namespace cagnet {
namespace kern {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int kMaxStages = 8;
constexpr int kChains = 4;             // independent accumulators per tile
constexpr int kLo = 2;                 // lo buffers
constexpr int kConvThreads = 128;      // 4 converter / epilogue warps
constexpr int kThreads = 64 + kConvThreads;
constexpr uint32_t A_TILE = BM * BK * 4;  // 16 KB
constexpr int kMaxBBytes = 96 * 1024;     // resident B (hi + lo)

struct TmaParams {
  int64_t m, n, k;
  const float* B;
  int64_t b_sk, b_sn;
  float* C;
  int64_t ldc;
  int accumulate;
  int epilogue;
  const float* aux;
  int64_t ldaux;
  float* aux_out;
  int64_t ldao;
  int nkb;      // k-blocks per tile
  int m_tiles;
};

// UMMA shared-memory descriptor, K-major SWIZZLE_128B (cute make_umma_desc:
// LBO = 16 B (unused for swizzled K-major), SBO = 1024 B between 8-row groups).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;          // LBO = 16 B
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO = 1024 B
  d |= static_cast<uint64_t>(1) << 46;          // version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;          // SWIZZLE_128B
  return d;
}

// Byte offset of element (row, k) of a [rows x 32] fp32 tile in the
// SWIZZLE_128B layout (1024 B-aligned base): 16 B chunks XOR row % 8.
__device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return static_cast<uint32_t>(row * 128 + ((((k >> 2) ^ (row & 7))) << 4) + (k & 3) * 4);
}

__device__ __forceinline__ void tma_load_2d(uint32_t smem, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float epilogue_value(const TmaParams& p, int64_t r, int64_t c, float v) {
  if (p.accumulate) v += p.C[r * p.ldc + c];
  if (p.epilogue == EPI_RELU) {
    if (p.aux_out) p.aux_out[r * p.ldao + c] = v > 0.f ? v : 0.f;
  } else if (p.epilogue == EPI_RELU_PRIME) {
    v = p.aux[r * p.ldaux + c] > 0.f ? v : v * 0.f;
  }
  return v;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap amap, const TmaParams p, int ns) {
  constexpr uint32_t B_TILE = BN * BK * 4;       // one k-block of B (hi or lo)
  constexpr uint32_t SET_COLS = kChains * BN;    // one accumulator set
  constexpr uint32_t TMEM_COLS = 2 * SET_COLS <= 32 ? 32 : 2 * SET_COLS <= 64 ? 64
                                 : 2 * SET_COLS <= 128 ? 128 : 2 * SET_COLS <= 256 ? 256 : 512;
  constexpr uint32_t IDESC = tc::idesc_tf32(BM, BN, 0, 0);

  extern __shared__ char smem_raw[];
  // Offset arithmetic on the __shared__ array keeps the compiler on LDS/STS;
  // SWIZZLE_128B tiles need 1024 B alignment.
  char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  char* a_hi = smem;                   // ns x 16 KB ring (TMA target, split in place)
  char* a_lo = a_hi + ns * A_TILE;     // kLo x 16 KB
  char* b_hi = a_lo + kLo * A_TILE;    // nkb x B_TILE, resident
  char* b_lo = b_hi + p.nkb * B_TILE;  // nkb x B_TILE, resident
  uint64_t* full = reinterpret_cast<uint64_t*>(b_lo + p.nkb * B_TILE);
  uint64_t* empty = full + kMaxStages;
  uint64_t* conv = empty + kMaxStages;
  uint64_t* tfull = conv + kMaxStages;  // [2] accumulator set ready
  uint64_t* tempty = tfull + 2;         // [2] accumulator set drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&conv[s], kConvThreads / 32);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], kConvThreads / 32);
    }
    tc::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);

  // Resident B: element (kk, j) of op(B) at B[kk * b_sk + j * b_sn] → row j,
  // column kk of the K-major [BN x 32] tile of k-block kk / 32.
  for (int e = tid; e < p.nkb * BN * BK; e += kThreads) {
    const int kb = e / (BN * BK);
    const int rem = e % (BN * BK);
    const int j = rem / BK, kk = rem % BK;
    const int64_t gk = static_cast<int64_t>(kb) * BK + kk;
    const float x = (gk < p.k && j < p.n) ? __ldg(p.B + gk * p.b_sk + static_cast<int64_t>(j) * p.b_sn) : 0.f;
    const float h = tc::to_tf32(x);
    const uint32_t off = kb * B_TILE + sw128_off(j, kk);
    *reinterpret_cast<float*>(b_hi + off) = h;
    *reinterpret_cast<float*>(b_lo + off) = x - h;
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int my_tiles = p.m_tiles > static_cast<int>(blockIdx.x)
                           ? (p.m_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                           : 0;
  const int64_t total = static_cast<int64_t>(my_tiles) * p.nkb;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      for (int64_t g = 0; g < total; ++g) {
        const int s = static_cast<int>(g % ns);
        if (g >= ns) tc::mbar_wait(&empty[s], static_cast<uint32_t>(((g / ns) - 1) & 1));
        const int t = static_cast<int>(g / p.nkb), kb = static_cast<int>(g % p.nkb);
        const int m_tile = static_cast<int>(blockIdx.x) + t * static_cast<int>(gridDim.x);
        tc::mbar_arrive_expect_tx(&full[s], A_TILE);
        tma_load_2d(tc::smem_u32(a_hi + s * A_TILE), &amap, tc::smem_u32(&full[s]), kb * BK, m_tile * BM);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    for (int64_t g = 0; g < total; ++g) {
      const int s = static_cast<int>(g % ns);
      const int t = static_cast<int>(g / p.nkb), kb = static_cast<int>(g % p.nkb);
      const int set = t & 1;
      if (kb == 0 && t >= 2) tc::mbar_wait(&tempty[set], static_cast<uint32_t>(((t >> 1) - 1) & 1));
      tc::mbar_wait(&conv[s], static_cast<uint32_t>((g / ns) & 1));
      tc::tc_fence_after();
      if (elect_one()) {
        const uint32_t ahs = tc::smem_u32(a_hi + s * A_TILE);
        const uint32_t als = tc::smem_u32(a_lo + (g % kLo) * A_TILE);
        const uint32_t bhs = tc::smem_u32(b_hi + kb * B_TILE), bls = tc::smem_u32(b_lo + kb * B_TILE);
        const uint32_t acc = tmem + set * SET_COLS + static_cast<uint32_t>((kb % kChains) * BN);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t dah = sw128_desc(ahs + kk * 32), dal = sw128_desc(als + kk * 32);
          const uint64_t dbh = sw128_desc(bhs + kk * 32), dbl = sw128_desc(bls + kk * 32);
          tc::mma_tf32(acc, dah, dbh, IDESC, (kb >= kChains) || kk != 0);
          tc::mma_tf32(acc, dah, dbl, IDESC, 1);
          tc::mma_tf32(acc, dal, dbh, IDESC, 1);
        }
        tc::mma_commit(&empty[s]);
        if (kb == p.nkb - 1) tc::mma_commit(&tfull[set]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- converters + epilogue ----------------
    const int ct = tid - 64;          // 0..127
    const int ew = warp - 2;          // epilogue warp → TMEM lanes [32 ew, 32 ew + 32)
    // tcgen05.ld lane quarter is fixed by warp id % 4.
    const int lane_q = warp & 3;
    for (int64_t g = 0; g < total; ++g) {
      const int s = static_cast<int>(g % ns);
      const int t = static_cast<int>(g / p.nkb), kb = static_cast<int>(g % p.nkb);
      // lo buffer g % kLo was read by MMA g - kLo.
      if (g >= kLo) tc::mbar_wait(&empty[(g - kLo) % ns], static_cast<uint32_t>(((g - kLo) / ns) & 1));
      tc::mbar_wait(&full[s], static_cast<uint32_t>((g / ns) & 1));
      char* ah = a_hi + s * A_TILE;
      char* al = a_lo + (g % kLo) * A_TILE;
#pragma unroll
      for (int i = 0; i < static_cast<int>(A_TILE / 16 / kConvThreads); ++i) {
        const uint32_t off = static_cast<uint32_t>((i * kConvThreads + ct) * 16);
        const float4 v = *reinterpret_cast<const float4*>(ah + off);
        float4 h, l;
        h.x = tc::to_tf32(v.x);
        h.y = tc::to_tf32(v.y);
        h.z = tc::to_tf32(v.z);
        h.w = tc::to_tf32(v.w);
        l.x = v.x - h.x;
        l.y = v.y - h.y;
        l.z = v.z - h.z;
        l.w = v.w - h.w;
        *reinterpret_cast<float4*>(ah + off) = h;
        *reinterpret_cast<float4*>(al + off) = l;
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&conv[s]);

      if (kb == p.nkb - 1) {
        // Tile finished: drain the accumulator set through the epilogue.
        const int set = t & 1;
        tc::mbar_wait(&tfull[set], static_cast<uint32_t>((t >> 1) & 1));
        tc::tc_fence_after();
        const int64_t m0 = static_cast<int64_t>(static_cast<int>(blockIdx.x) + t * static_cast<int>(gridDim.x)) * BM;
        const int64_t r = m0 + lane_q * 32 + (tid & 31);
        const uint32_t base = tmem + (static_cast<uint32_t>(lane_q * 32) << 16) + set * SET_COLS;
        const int chains = p.nkb < kChains ? p.nkb : kChains;
#pragma unroll 1
        for (int cb = 0; cb < BN / 16; ++cb) {
          float v[16];
          tc::tmem_ld16(base + cb * 16, v);
          for (int c = 1; c < chains; ++c) {
            float w[16];
            tc::tmem_ld16(base + c * BN + cb * 16, w);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += w[j];
          }
          if (r < p.m) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int64_t c = cb * 16 + j;
              if (c < p.n) p.C[r * p.ldc + c] = epilogue_value(p, r, c, v[j]);
            }
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&tempty[set]);
        (void)ew;
      }
    }
  }

  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

template <int BN>
void launch(const CUtensorMap& map, const TmaParams& p, cudaStream_t s) {
  // Ring depth from the shared-memory budget left after resident B and lo.
  const size_t fixed = 1024 + kLo * A_TILE + 2 * static_cast<size_t>(p.nkb) * BN * BK * 4 + 512;
  int ns = static_cast<int>((227 * 1024 - fixed) / A_TILE);
  if (ns > kMaxStages) ns = kMaxStages;
  const size_t smem = fixed + static_cast<size_t>(ns) * A_TILE;
  auto kfn = gemm_tma_kernel<BN>;
  static std::atomic<uint64_t> configured{0};
  const uint64_t bit = 1ull << (current_device() & 63);
  if (!(configured.load() & bit)) {
    CG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured.fetch_or(bit);
  }
  const int sms = num_sms(current_device());
  const unsigned grid = static_cast<unsigned>(p.m_tiles < sms ? p.m_tiles : sms);
  kfn<<<grid, kThreads, smem, s>>>(map, p, ns);
  CG_LAUNCH_CHECK();
}

}  // namespace

bool gemm_tma_try(const GemmDesc& d, cudaStream_t stream) {
  // A must be row-major with 16 B-aligned rows (TMA), N <= 64, and all of B
  // (hi + lo) must fit in shared memory next to a ring of >= 4 A tiles.
  if (d.a_sk != 1 || d.a_sm % 4 != 0 || reinterpret_cast<uintptr_t>(d.A) % 16 != 0) return false;
  if (d.n > 64 || d.k <= 0 || d.m < BM) return false;
  const int bn = d.n <= 16 ? 16 : d.n <= 32 ? 32 : d.n <= 48 ? 48 : 64;
  const int nkb = static_cast<int>(ceil_div64(d.k, BK));
  if (2 * static_cast<int64_t>(nkb) * bn * BK * 4 > kMaxBBytes) return false;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;

  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.k), static_cast<cuuint64_t>(d.m)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.a_sm) * 4};
  const cuuint32_t box[2] = {BK, BM};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(d.A), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;

  TmaParams p{};
  p.m = d.m;
  p.n = d.n;
  p.k = d.k;
  p.B = d.B;
  p.b_sk = d.b_sk;
  p.b_sn = d.b_sn;
  p.C = d.C;
  p.ldc = d.ldc;
  p.accumulate = d.accumulate ? 1 : 0;
  p.epilogue = d.epilogue;
  p.aux = d.aux;
  p.ldaux = d.ldaux;
  p.aux_out = d.aux_out;
  p.ldao = d.ldao;
  p.nkb = nkb;
  p.m_tiles = static_cast<int>(ceil_div64(d.m, BM));
  switch (bn) {
    case 16: launch<16>(map, p, stream); break;
    case 32: launch<32>(map, p, stream); break;
    case 48: launch<48>(map, p, stream); break;
    default: launch<64>(map, p, stream); break;
  }
  return true;
}

}  // namespace kern
}  // namespace cagnet
