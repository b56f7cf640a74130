// K2c — persistent, warp-specialised tcgen05 split-TF32 GEMM whose A operand
// is staged in TENSOR MEMORY, for the GCN's tall-skinny contractions
// (gemm_add, dense.cpp:37-70):
//   T·W / H·W / S·Wᵀ : A = rows of a dense tile (K contiguous), B = W resident
//   Hᵀ·S             : A = Hᵀ (M contiguous in memory, K = graph rows),
//                      B = S streamed alongside A, split-K across CTAs.
//
// Why TMEM: with N <= 64 the kernel moves ~16 KB of A per 4 K-steps of tiny
// MMAs, so shared-memory traffic, not the tensor pipe, was the ceiling of the
// smem-operand kernel (TMA write + read + hi/lo write-back + three MMA reads
// of A ≈ 7x the tile).  Here the TMA tile is read once by the converter warps
// (thread = TMEM lane = output row), split into hi = tf32_rn(x) and
// lo = x - hi in registers, and written to TMEM with tcgen05.st; the MMAs read
// A from TMEM ("TS" form).  The reading thread picks the element order, so the
// M-contiguous Hᵀ tile is transposed for free (tf32 smem operands must be
// K-major).  B is stacked as [B_hi; B_lo] (2·BN rows, K-major SWIZZLE_128B),
// so one N = 2·BN MMA gives A_hi·B_hi and A_hi·B_lo side by side and one
// N = BN MMA adds A_lo·B_hi onto the second half:
//   C = D[:, 0:BN] + D[:, BN:2BN]      (split-TF32, error ~2^-21 relative).
//
// Roles (one CTA per SM):
//   warp 0      TMA producer: A tile (+ S tile when streamed) per k-block;
//   warp 1      MMA issuer (one elected lane), TMEM allocator;
//   warps 2-5   converters (TMA smem → hi/lo → TMEM; streamed B → [hi; lo]
//               smem tile);
//   warps 6-9   epilogue of each finished tile: tcgen05.ld of the accumulator
//               chains → a staged smem tile → coalesced row-major stores with
//               the fused ReLU / ⊙relu′ / accumulate (or the split-K partial),
//               so conversion of tile t+1 never waits for tile t's stores.
// Accumulator chains (k-step kk → chain kk % CH) keep several independent
// MMAs in flight; two accumulator sets overlap tile t's epilogue with tile
// t+1's MMAs when TMEM allows.
#include <cuda.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"
#include "tc.cuh"

namespace cagnet {
namespace kern {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int kConv = 128;                // converter threads per group
constexpr int kConvGroups = 2;            // groups take alternate k-blocks (warps 2-5, 6-9)
constexpr int kEpi = 128;                 // epilogue threads (warps 10-13)
constexpr int kEpiWarp0 = 2 + kConvGroups * kConv / 32;
constexpr int kThreads = 64 + kConvGroups * kConv + kEpi;
constexpr uint32_t A_TILE = BM * BK * 4;  // 16 KB
constexpr int kMaxStages = 8;
constexpr int kMaxTmemStages = 8;         // A (hi + lo) stages in TMEM (upper bound)
constexpr int kMaxResidentB = 96 * 1024;  // bytes of resident [B_hi; B_lo]
// BN <= 16: accumulator chains and sets (build-time A/B knobs; TMEM left over
// after the accumulators holds the A stages).
#ifndef CAGNET_TM_CH16
#define CAGNET_TM_CH16 4
#endif
#ifndef CAGNET_TM_SETS16
#define CAGNET_TM_SETS16 2
#endif

// TMEM budget (512 columns): accumulator sets x chains x 2 BN, the rest holds
// A stages of 64 columns (hi + lo).  The split-K Hᵀ·S kernel has one tile per
// CTA, so one accumulator set and deeper A staging (the MMA-completion round
// trip, not bandwidth, bounds a shallow ring).
template <int BN, bool BSTREAM>
struct Cfg {
  static constexpr int CH = BN <= 16 ? CAGNET_TM_CH16 : BN <= 48 ? 2 : 1;  // accumulator chains
  static constexpr int SETS = (BSTREAM || BN == 48) ? 1 : BN <= 16 ? CAGNET_TM_SETS16 : 2;  // sets
  static constexpr uint32_t SET_COLS = CH * 2 * BN;
  static constexpr int TS_FIT = (512 - SETS * SET_COLS) / (2 * BK);
  static constexpr int TSTAGES = TS_FIT > kMaxTmemStages ? kMaxTmemStages : TS_FIT;
  static constexpr uint32_t A_COLS = TSTAGES * 2 * BK;             // hi + lo per stage
  static constexpr uint32_t D_BASE = A_COLS;
  static constexpr uint32_t COLS = A_COLS + SETS * SET_COLS;
  static_assert(COLS <= 512 && TSTAGES >= 2, "TMEM budget");
  static constexpr uint32_t B_TILE = 2 * BN * BK * 4;              // [hi; lo] k-block
  static constexpr uint32_t S_TILE = BN * BK * 4;                  // raw streamed S k-block
  static constexpr int EP_LD = BN;                                 // staged output row (floats)
  static constexpr uint32_t EP_BYTES = BM * EP_LD * 4;             // one [BM][BN] TMA box
};

struct TmParams {
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
  float* partial;   // split-K workspace [splits][m][n]; nullptr = direct epilogue
  int64_t k_chunk;  // K per split (multiple of BK)
  int nkb_res;      // k-blocks of resident B (0 when streamed)
  int m_tiles;
  int chains;       // accumulator chains in use (1 for short K: nothing to overlap)
  int dbg;          // timing experiments only (CAGNET_GEMM_DBG): 1 skip st, 2 skip mma, 4 skip epi stores
  // Contiguous operands move as ONE bulk copy per k-block instead of a tensor
  // box of many narrow rows (64 B rows cost the TMA one request each):
  const float* A;
  int64_t a_ld;     // row stride of A in memory (elements)
  int a_bulk;       // AMODE 0: tile = 128 x a_ld (a_ld <= 32); AMODE 1: k-block = 32 x a_ld (m <= 128)
  int s_bulk;       // streamed S k-block = 32 x b_sk contiguous floats (b_sk <= BN)
  int tstore;       // epilogue through TMA tensor stores (C / aux_out / partial maps)
  int64_t pld;      // row stride of the split-K partial rows (multiple of 4)
  int64_t mpad;     // rows per split in the partial buffer (m rounded up to BM)
  unsigned long long* trace;  // dev timing trace of CTA 0 (CAGNET_GEMM_TRACE), else null
};

// Timing trace (development only): slot = event * 64 + g for g < 64.
__device__ __forceinline__ void trace_at(const TmParams& p, int ev, int64_t g) {
  if (p.trace != nullptr && blockIdx.x == 0 && g < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[ev * 64 + g] = t;
  }
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;          // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO = 8 rows x 128 B
  d |= static_cast<uint64_t>(1) << 46;          // sm_100 descriptor version
  d |= static_cast<uint64_t>(2) << 61;          // SWIZZLE_128B
  return d;
}

// Byte offset of (row, k) in a [rows x 32] fp32 SWIZZLE_128B tile.
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

// 1D bulk copy global → shared, completing on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(uint32_t smem, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

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

// D[tmem] (+)= A[tmem] * B[smem].
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ float epilogue_value(const TmParams& p, int64_t r, int64_t c, float v) {
  if (p.accumulate) v += p.C[r * p.ldc + c];
  if (p.epilogue == EPI_RELU) {
    if (p.aux_out) p.aux_out[r * p.ldao + c] = v > 0.f ? v : 0.f;
  } else if (p.epilogue == EPI_RELU_PRIME) {
    v = p.aux[r * p.ldaux + c] > 0.f ? v : v * 0.f;
  }
  return v;
}

// AMODE 0: A tile = 128 rows x 32 k, K contiguous (TMA SWIZZLE_128B).
// AMODE 1: A tile = 32 k x 128 m, M contiguous (TMA, no swizzle) — Hᵀ.
// BSTREAM: B (k x n, n contiguous) arrives by TMA with every k-block.
template <int BN, int AMODE, bool BSTREAM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                   const __grid_constant__ CUtensorMap cmap, const __grid_constant__ CUtensorMap xmap,
                   const TmParams p, int ns) {
  using K = Cfg<BN, BSTREAM>;
  constexpr int kTmemStages = K::TSTAGES;
  constexpr uint32_t IDESC_HL = tc::idesc_tf32(BM, 2 * BN, 0, 0);  // A_hi · [B_hi; B_lo]
  constexpr uint32_t IDESC_L = tc::idesc_tf32(BM, BN, 0, 0);       // A_lo · B_hi
  constexpr int SB = kTmemStages;  // streamed [hi; lo] B stages (recycled with the TMEM stage)

  extern __shared__ char smem_raw[];
  char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  char* a_ring = smem;                                  // ns x 16 KB
  char* s_ring = a_ring + ns * A_TILE;                  // ns x S_TILE (streamed B raw)
  char* b_cat = s_ring + (BSTREAM ? ns * K::S_TILE : 0);  // resident nkb or SB stages
  const int b_slots = BSTREAM ? SB : p.nkb_res;
  float* ep = reinterpret_cast<float*>(b_cat + b_slots * K::B_TILE);  // [BM][BN] output tile
  float* ep2 = ep + BM * K::EP_LD;  // relu output / loaded relu′ mask (second box)
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(ep) + 2 * K::EP_BYTES);
  uint64_t* sempty = full + kMaxStages;       // smem stage read by the converters
  uint64_t* conv = sempty + kMaxStages;       // [kTmemStages] TMEM A stage written
  uint64_t* tempty = conv + kTmemStages;      // [kTmemStages] TMEM A stage consumed by MMA
  uint64_t* afull = tempty + kTmemStages;     // [2] accumulator set complete
  uint64_t* aempty = afull + 2;               // [2] accumulator set drained
  uint64_t* eload = aempty + 2;               // epilogue's C / mask tile loads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eload + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&sempty[s], kConv / 32);
    }
    for (int s = 0; s < kTmemStages; ++s) {
      tc::mbar_init(&conv[s], kConv / 32);
      tc::mbar_init(&tempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&afull[i], 1);
      tc::mbar_init(&aempty[i], kEpi / 32);
    }
    tc::mbar_init(eload, 1);
    tc::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
    if (BSTREAM)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);

  if (!BSTREAM) {
    // Resident [B_hi; B_lo]: element (kk, j) of op(B) → rows j and BN + j,
    // column kk % 32 of k-block kk / 32.
    for (int e = tid; e < p.nkb_res * BN * BK; e += kThreads) {
      const int kb = e / (BN * BK);
      const int rem = e % (BN * BK);
      const int j = rem / BK, kk = rem % BK;
      const int64_t gk = static_cast<int64_t>(kb) * BK + kk;
      const float x =
          (gk < p.k && j < p.n) ? __ldg(p.B + gk * p.b_sk + static_cast<int64_t>(j) * p.b_sn) : 0.f;
      const float h = tc::to_tf32(x);
      char* t = b_cat + kb * K::B_TILE;
      *reinterpret_cast<float*>(t + sw128_off(j, kk)) = h;
      *reinterpret_cast<float*>(t + sw128_off(BN + j, kk)) = x - h;
    }
    tc::fence_proxy_async_smem();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Work list: tiles (m_tile, split) strided over the grid.
  const int splits = static_cast<int>((p.k + p.k_chunk - 1) / p.k_chunk);
  const int tiles = p.m_tiles * splits;
  const int my_tiles = tiles > static_cast<int>(blockIdx.x)
                           ? (tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                           : 0;
  auto tile_of = [&](int t, int& m_tile, int& split, int& nkb) {
    const int id = static_cast<int>(blockIdx.x) + t * static_cast<int>(gridDim.x);
    m_tile = id % p.m_tiles;
    split = id / p.m_tiles;
    const int64_t k0 = static_cast<int64_t>(split) * p.k_chunk;
    const int64_t k1 = k0 + p.k_chunk < p.k ? k0 + p.k_chunk : p.k;
    nkb = static_cast<int>((k1 - k0 + BK - 1) / BK);
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int64_t g = 0;
      for (int t = 0; t < my_tiles; ++t) {
        int m_tile, split, nkb;
        tile_of(t, m_tile, split, nkb);
        const int64_t kb0 = static_cast<int64_t>(split) * (p.k_chunk / BK);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = static_cast<int>(g % ns);
          if (g >= ns) tc::mbar_wait(&sempty[s], static_cast<uint32_t>(((g / ns) - 1) & 1));
          const int64_t kg = (kb0 + kb) * BK;
          const int kcoord = static_cast<int>(kg);
          const int kval = static_cast<int>(p.k - kg < BK ? p.k - kg : BK);
          uint32_t a_bytes = A_TILE, s_bytes = BSTREAM ? K::S_TILE : 0;
          if (p.a_bulk) {
            if (AMODE == 0) {
              const int64_t r0 = static_cast<int64_t>(m_tile) * BM;
              const int rows = static_cast<int>(p.m - r0 < BM ? p.m - r0 : BM);
              a_bytes = static_cast<uint32_t>(rows * p.a_ld * 4);
            } else {
              a_bytes = static_cast<uint32_t>(kval * p.a_ld * 4);
            }
          }
          if (BSTREAM && p.s_bulk) s_bytes = static_cast<uint32_t>(kval * p.b_sk * 4);
          trace_at(p, 0, g);
          tc::mbar_arrive_expect_tx(&full[s], a_bytes + s_bytes);
          const uint32_t a_dst = tc::smem_u32(a_ring + s * A_TILE);
          if (p.a_bulk) {
            const float* src = AMODE == 0 ? p.A + static_cast<int64_t>(m_tile) * BM * p.a_ld
                                          : p.A + kg * p.a_ld;
            bulk_load(a_dst, src, a_bytes, tc::smem_u32(&full[s]));
          } else if (AMODE == 0) {
            tma_load_2d(a_dst, &amap, tc::smem_u32(&full[s]), kcoord, m_tile * BM);
          } else {
            tma_load_2d(a_dst, &amap, tc::smem_u32(&full[s]), m_tile * BM, kcoord);
          }
          if (BSTREAM) {
            const uint32_t s_dst = tc::smem_u32(s_ring + s * K::S_TILE);
            if (p.s_bulk)
              bulk_load(s_dst, p.B + kg * p.b_sk, s_bytes, tc::smem_u32(&full[s]));
            else
              tma_load_2d(s_dst, &bmap, tc::smem_u32(&full[s]), 0, kcoord);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int64_t g = 0;
    for (int t = 0; t < my_tiles; ++t) {
      int m_tile, split, nkb;
      tile_of(t, m_tile, split, nkb);
      const int set = K::SETS == 2 ? (t & 1) : 0;
      const int use = K::SETS == 2 ? (t >> 1) : t;  // how often this set was used before
      if (use >= 1) tc::mbar_wait(&aempty[set], static_cast<uint32_t>((use - 1) & 1));
      const uint32_t dset = tmem + K::D_BASE + set * K::SET_COLS;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int ts = static_cast<int>(g % kTmemStages);
        tc::mbar_wait(&conv[ts], static_cast<uint32_t>((g / kTmemStages) & 1));
        tc::tc_fence_after();
        if (elect_one()) {
          const uint32_t a_hi = tmem + ts * 2 * BK;
          const uint32_t a_lo = a_hi + BK;
          const uint32_t bt = tc::smem_u32(b_cat + (BSTREAM ? ts : kb) * K::B_TILE);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            if (p.dbg & 2) break;
            const int ch = kk % p.chains;
            const uint32_t d = dset + ch * 2 * BN;
            const uint64_t bdesc = sw128_desc(bt + kk * 32);
            mma_tf32_ts(d, a_hi + kk * 8, bdesc, IDESC_HL, (kb > 0) || (kk >= p.chains));
            mma_tf32_ts(d + BN, a_lo + kk * 8, bdesc, IDESC_L, 1);
          }
          trace_at(p, 3, g);
          tc::mma_commit(&tempty[ts]);
          if (kb == nkb - 1) {
            tc::mma_commit(&afull[set]);
            trace_at(p, 5, t);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp < kEpiWarp0) {
    // ---------------- converters ----------------
    // kConvGroups groups of 4 warps convert alternate k-blocks, so one group's
    // TMEM-store / proxy-fence latency overlaps the other group's work.
    const int grp = (warp - 2) / 4;
    const int ct = (tid - 64) % kConv;  // 0..127 within the group
    const int lane_q = warp & 3;   // TMEM lane quarter of this warp
    const int row = lane_q * 32 + (tid & 31);  // tile row = TMEM lane
    const uint32_t lane_bits = static_cast<uint32_t>(lane_q * 32) << 16;
    int64_t g = 0;
    for (int t = 0; t < my_tiles; ++t) {
      int m_tile, split, nkb;
      tile_of(t, m_tile, split, nkb);
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        if (static_cast<int>(g % kConvGroups) != grp) continue;
        const int s = static_cast<int>(g % ns);
        const int ts = static_cast<int>(g % kTmemStages);
        tc::mbar_wait(&full[s], static_cast<uint32_t>((g / ns) & 1));
        if (ct == 0) trace_at(p, 1, g);
        const char* at = a_ring + s * A_TILE;
        const int64_t kg = (static_cast<int64_t>(split) * (p.k_chunk / BK) + kb) * BK;
        const int kval = static_cast<int>(p.k - kg < BK ? p.k - kg : BK);
        // The TMEM stage (and the streamed-B slot) was consumed by MMA g - stages.
        if (g >= kTmemStages)
          tc::mbar_wait(&tempty[ts], static_cast<uint32_t>(((g / kTmemStages) - 1) & 1));
        tc::tc_fence_after();
        const uint32_t a_hi = tmem + lane_bits + ts * 2 * BK;
        // Two halves of 16 k-columns keep the register footprint at 32 + 32.
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t hi[BK / 2], lo[BK / 2];
          if (p.a_bulk) {
            // Dense rows of stride a_ld; bytes past the copied extent are stale.
            const int lda = static_cast<int>(p.a_ld);
            const float* af = reinterpret_cast<const float*>(at);
            const bool live = AMODE == 0 ? static_cast<int64_t>(m_tile) * BM + row < p.m : row < p.m;
#pragma unroll
            for (int i = 0; i < BK / 2; ++i) {
              const int kk = half * (BK / 2) + i;
              const float x = (live && kk < kval) ? (AMODE == 0 ? af[row * lda + kk] : af[kk * lda + row]) : 0.f;
              const float h = tc::to_tf32(x);
              hi[i] = __float_as_uint(h);
              lo[i] = __float_as_uint(x - h);
            }
          } else if (AMODE == 0) {
#pragma unroll
            for (int c = 0; c < BK / 8; ++c) {
              const int cc = half * (BK / 8) + c;
              const float4 v = *reinterpret_cast<const float4*>(at + row * 128 + ((cc ^ (row & 7)) << 4));
              const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float h = tc::to_tf32(x[j]);
                hi[4 * c + j] = __float_as_uint(h);
                lo[4 * c + j] = __float_as_uint(x[j] - h);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < BK / 2; ++i) {
              const int kk = half * (BK / 2) + i;
              const float x = *reinterpret_cast<const float*>(at + kk * (BM * 4) + row * 4);
              const float h = tc::to_tf32(x);
              hi[i] = __float_as_uint(h);
              lo[i] = __float_as_uint(x - h);
            }
          }
          if (!(p.dbg & 1)) {
            tmem_st16(a_hi + half * (BK / 2), hi);
            tmem_st16(a_hi + BK + half * (BK / 2), lo);
          }
        }
        if (BSTREAM) {
          // Raw S k-block [32 k][BN j] → K-major [B_hi; B_lo] rows j / BN + j.
          const char* st = s_ring + s * K::S_TILE;
          char* bt = b_cat + ts * K::B_TILE;
          const int sld = p.s_bulk ? static_cast<int>(p.b_sk) : BN;
#pragma unroll
          for (int i = 0; i < (BN * BK) / kConv; ++i) {
            const int e = i * kConv + ct;
            const int kk = e / BN, j = e % BN;
            const float x = (!p.s_bulk || (kk < kval && j < p.n))
                                ? *reinterpret_cast<const float*>(st + (kk * sld + j) * 4)
                                : 0.f;
            const float h = tc::to_tf32(x);
            *reinterpret_cast<float*>(bt + sw128_off(j, kk)) = h;
            *reinterpret_cast<float*>(bt + sw128_off(BN + j, kk)) = x - h;
          }
          tc::fence_proxy_async_smem();
        }
        if (!(p.dbg & 1)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc::tc_fence_before();
        __syncwarp();
        if ((tid & 31) == 0) {
          mbar_arrive(&sempty[s]);
          mbar_arrive(&conv[ts]);
          if (ct == 0) trace_at(p, 2, g);
        }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int et = tid - 64 - kConvGroups * kConv;  // 0..127
    const bool leader = et == 0;
    const int lane_q = warp & 3;
    const int row = lane_q * 32 + (tid & 31);
    const uint32_t lane_bits = static_cast<uint32_t>(lane_q * 32) << 16;
    const int n = static_cast<int>(p.n);
    const int rpp = kEpi / n;          // STG path: rows per pass (n <= 64)
    const int er = et / n, ec = et - er * n;
    const bool ec_ok = er < rpp;
    constexpr int NCH = BN / 4;        // float4 chunks per staged row
    const bool load_c = p.tstore && p.accumulate && !p.partial;
    const bool load_x = p.tstore && p.epilogue == EPI_RELU_PRIME && !p.partial;
    const bool relu_out = p.epilogue == EPI_RELU && p.aux_out != nullptr && !p.partial;
    for (int t = 0; t < my_tiles; ++t) {
      int m_tile, split, nkb;
      tile_of(t, m_tile, split, nkb);
      const int64_t r0 = static_cast<int64_t>(m_tile) * BM;
      if (leader && (load_c || load_x)) {
        tc::mbar_arrive_expect_tx(eload, (load_c ? K::EP_BYTES : 0) + (load_x ? K::EP_BYTES : 0));
        if (load_c) tma_load_2d(tc::smem_u32(ep), &cmap, tc::smem_u32(eload), 0, static_cast<int>(r0));
        if (load_x) tma_load_2d(tc::smem_u32(ep2), &xmap, tc::smem_u32(eload), 0, static_cast<int>(r0));
      }
      const int set = K::SETS == 2 ? (t & 1) : 0;
      const int use = K::SETS == 2 ? (t >> 1) : t;
      tc::mbar_wait(&afull[set], static_cast<uint32_t>(use & 1));
      if (et == 0) trace_at(p, 4, t);
      tc::tc_fence_after();
      const uint32_t base = tmem + lane_bits + K::D_BASE + set * K::SET_COLS;
      float v[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) v[j] = 0.f;
#pragma unroll 1
      for (int c = 0; c < p.chains; ++c) {
#pragma unroll
        for (int cb = 0; cb < BN / 16; ++cb) {
          uint32_t w[16], u[16];
          tc::tmem_ld16_nowait(base + c * 2 * BN + cb * 16, w);
          tc::tmem_ld16_nowait(base + c * 2 * BN + BN + cb * 16, u);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[cb * 16 + j] += __uint_as_float(w[j]) + __uint_as_float(u[j]);
        }
      }
      // The accumulator set is free once it sits in registers.
      tc::tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&aempty[set]);
      if (load_c || load_x) tc::mbar_wait(eload, static_cast<uint32_t>(t & 1));
      float4* e4 = reinterpret_cast<float4*>(ep + row * K::EP_LD);
      float4* x4 = reinterpret_cast<float4*>(ep2 + row * K::EP_LD);
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const int q = i;
        float4 z = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (load_c) {
          const float4 o = e4[q];
          z.x += o.x;
          z.y += o.y;
          z.z += o.z;
          z.w += o.w;
        }
        if (load_x) {
          const float4 m = x4[q];
          z.x = m.x > 0.f ? z.x : z.x * 0.f;
          z.y = m.y > 0.f ? z.y : z.y * 0.f;
          z.z = m.z > 0.f ? z.z : z.z * 0.f;
          z.w = m.w > 0.f ? z.w : z.w * 0.f;
        }
        e4[q] = z;
        if (p.tstore && relu_out)
          x4[q] = make_float4(fmaxf(z.x, 0.f), fmaxf(z.y, 0.f), fmaxf(z.z, 0.f), fmaxf(z.w, 0.f));
      }
      if (p.tstore) {
        tc::fence_proxy_async_smem();
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        if (leader && !(p.dbg & 4)) {
          if (p.partial) {
            tma_store_2d(&cmap, tc::smem_u32(ep), 0, static_cast<int>(static_cast<int64_t>(split) * p.mpad + r0));
          } else {
            tma_store_2d(&cmap, tc::smem_u32(ep), 0, static_cast<int>(r0));
            if (relu_out) tma_store_2d(&xmap, tc::smem_u32(ep2), 0, static_cast<int>(r0));
          }
          bulk_commit();
          bulk_wait_read0();  // staging tiles reusable
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        continue;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
      // Fallback: coalesced row-major stores, thread et owns column ec of rows
      // er, er + rpp, ...; loads of each batch of 4 rows precede their stores.
      const int rows = static_cast<int>(p.m - r0 < BM ? p.m - r0 : BM);
      if (ec_ok && !(p.dbg & 4)) {
        if (p.partial) {
          float* dst = p.partial + (static_cast<int64_t>(split) * p.mpad + r0) * p.pld + ec;
          for (int r = er; r < rows; r += rpp) dst[static_cast<int64_t>(r) * p.pld] = ep[r * K::EP_LD + ec];
        } else {
          for (int rb = er; rb < rows; rb += 4 * rpp) {
            float x[4], cold[4], ax[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = rb + i * rpp;
              const int64_t gr = r0 + r;
              const bool ok = r < rows;
              x[i] = ok ? ep[r * K::EP_LD + ec] : 0.f;
              cold[i] = (ok && p.accumulate) ? p.C[gr * p.ldc + ec] : 0.f;
              ax[i] = (ok && p.epilogue == EPI_RELU_PRIME) ? p.aux[gr * p.ldaux + ec] : 1.f;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = rb + i * rpp;
              if (r >= rows) break;
              const int64_t gr = r0 + r;
              float y = x[i] + cold[i];
              if (p.epilogue == EPI_RELU) {
                if (p.aux_out) p.aux_out[gr * p.ldao + ec] = y > 0.f ? y : 0.f;
              } else if (p.epilogue == EPI_RELU_PRIME) {
                y = ax[i] > 0.f ? y : y * 0.f;
              }
              p.C[gr * p.ldc + ec] = y;
            }
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
    }
    if (leader) bulk_wait0();  // stores globally visible before the CTA retires
  }

  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// Deterministic split-K fold: C = epilogue((acc ? C : 0) + sum_s partial[s]).
// One warp per output element: lane i sums splits i, i + 32, ... in order,
// then a fixed xor tree — the same order on every run.
__global__ void tm_reduce_kernel(const TmParams p, int splits) {
  const int64_t total = p.m * p.n;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t e = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; e < total;
       e += warps) {
    double s = 0.0;  // fp64 fold of the split partials (fixed order: deterministic)
    const int64_t r = e / p.n, c = e % p.n;
    for (int z = lane; z < splits; z += 32)
      s += static_cast<double>(p.partial[(static_cast<int64_t>(z) * p.mpad + r) * p.pld + c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      p.C[r * p.ldc + c] = epilogue_value(p, r, c, static_cast<float>(s));
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) != cudaSuccess ||
        r != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(q);
  }();
  return fn;
}

bool encode_2d(CUtensorMap* map, const float* base, uint64_t inner, uint64_t outer,
               uint64_t stride_elems, uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {stride_elems * 4};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int AMODE, bool BSTREAM>
void launch_tm(const CUtensorMap& amap, const CUtensorMap& bmap, const CUtensorMap& cmap,
               const CUtensorMap& xmap, const TmParams& p, int grid, cudaStream_t s) {
  using K = Cfg<BN, BSTREAM>;
  constexpr int kTmemStages = K::TSTAGES;
  const size_t fixed = 1024 + static_cast<size_t>(BSTREAM ? kTmemStages : p.nkb_res) * K::B_TILE +
                       2 * K::EP_BYTES + (3 * kMaxStages + 4 * kTmemStages + 10) * 8;
  const size_t per_stage = A_TILE + (BSTREAM ? K::S_TILE : 0);
  int ns = static_cast<int>((227 * 1024 - fixed) / per_stage);
  if (ns > kMaxStages) ns = kMaxStages;
  const size_t smem = fixed + static_cast<size_t>(ns) * per_stage;
  auto kfn = gemm_tm_kernel<BN, AMODE, BSTREAM>;
  static std::atomic<uint64_t> configured{0};
  const uint64_t bit = 1ull << (current_device() & 63);
  if (!(configured.load() & bit)) {
    CG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured.fetch_or(bit);
  }
  kfn<<<static_cast<unsigned>(grid), kThreads, smem, s>>>(amap, bmap, cmap, xmap, p, ns);
  CG_LAUNCH_CHECK();
}

struct Maps {
  CUtensorMap a, b, c, x;
};

template <int AMODE, bool BSTREAM>
void launch_bn(int bn, const Maps& m, const TmParams& p, int grid, cudaStream_t s) {
  switch (bn) {
    case 16: return launch_tm<16, AMODE, BSTREAM>(m.a, m.b, m.c, m.x, p, grid, s);
    case 32: return launch_tm<32, AMODE, BSTREAM>(m.a, m.b, m.c, m.x, p, grid, s);
    case 48: return launch_tm<48, AMODE, BSTREAM>(m.a, m.b, m.c, m.x, p, grid, s);
    default: return launch_tm<64, AMODE, BSTREAM>(m.a, m.b, m.c, m.x, p, grid, s);
  }
}

bool aligned16(const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; }

// Development trace: event times of CTA 0 relative to the first producer issue.
void dump_trace(const TmParams& p, cudaStream_t s, const char* what) {
  if (!p.trace) return;
  CG_CUDA(cudaStreamSynchronize(s));
  unsigned long long tr[8 * 64];
  CG_CUDA(cudaMemcpy(tr, p.trace, sizeof(tr), cudaMemcpyDeviceToHost));
  const unsigned long long t0 = tr[0];
  std::fprintf(stderr, "[gemm_tm trace %s m=%lld n=%lld k=%lld] g: issue full conv mma (ns)\n", what,
               static_cast<long long>(p.m), static_cast<long long>(p.n), static_cast<long long>(p.k));
  for (int g = 0; g < 24; ++g)
    std::fprintf(stderr, "  %2d: %8lld %8lld %8lld %8lld   epi[t=%d] %8lld commit %8lld\n", g,
                 static_cast<long long>(tr[g] - t0), static_cast<long long>(tr[64 + g] - t0),
                 static_cast<long long>(tr[128 + g] - t0), static_cast<long long>(tr[192 + g] - t0), g,
                 static_cast<long long>(tr[256 + g] - t0), static_cast<long long>(tr[320 + g] - t0));
}

}  // namespace

bool gemm_tm_try(const GemmDesc& d, cudaStream_t stream);

// N > 64 (e.g. Protein's 256 classes): column tiles of 64, each a full
// gemm_tm launch on the matching B / C / aux column slices (A is re-read
// once per tile; the output stream dominates these shapes).
bool gemm_tm_wide(const GemmDesc& d, cudaStream_t stream) {
  for (int64_t c0 = 0; c0 < d.n; c0 += 64) {
    GemmDesc t = d;
    t.n = d.n - c0 < 64 ? d.n - c0 : 64;
    t.B = d.B + c0 * d.b_sn;
    t.C = d.C + c0;
    if (d.aux) t.aux = d.aux + c0;
    if (d.aux_out) t.aux_out = d.aux_out + c0;
    // Every slice must take the tensor-core path; check the first one.
    if (!gemm_tm_try(t, stream)) {
      if (c0 == 0) return false;
      throw std::logic_error("gemm_tm: column tile rejected after the first");
    }
  }
  return true;
}

bool gemm_tm_try(const GemmDesc& d, cudaStream_t stream) {
  if (d.m <= 0 || d.n <= 0 || d.k <= 0) return false;
  if (d.n > 64) return gemm_tm_wide(d, stream);
  if (!aligned16(d.A)) return false;
  const int bn = d.n <= 16 ? 16 : d.n <= 32 ? 32 : d.n <= 48 ? 48 : 64;
  const int sms = num_sms(current_device());
  const int64_t m_tiles = ceil_div64(d.m, BM);

  TmParams p{};
  static const int dbg = [] {
    const char* e = std::getenv("CAGNET_GEMM_DBG");
    return e ? std::atoi(e) : 0;
  }();
  p.dbg = dbg;
  p.m = d.m;
  p.n = d.n;
  p.k = d.k;
  p.A = d.A;
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
  p.m_tiles = static_cast<int>(m_tiles);
  p.pld = round_up(d.n, 4);
  p.mpad = m_tiles * BM;
  static unsigned long long* trace = [] {
    unsigned long long* t = nullptr;
    if (std::getenv("CAGNET_GEMM_TRACE")) {
      CG_CUDA(cudaMalloc(&t, 8 * 64 * sizeof(unsigned long long)));
      CG_CUDA(cudaMemset(t, 0, 8 * 64 * sizeof(unsigned long long)));
    }
    return t;
  }();
  p.trace = trace;

  Maps maps;
  std::memset(&maps, 0, sizeof(maps));
  const bool a_k = d.a_sk == 1 && d.a_sm % 4 == 0 && d.a_sm >= d.k;
  const bool a_m = d.a_sm == 1 && d.a_sk % 4 == 0 && d.a_sk >= d.m;
  const bool b_stream_ok = d.b_sn == 1 && d.b_sk % 4 == 0 && aligned16(d.B) && d.b_sk >= d.n;
  // Epilogue through TMA tensor stores when every output matrix is a
  // 16 B-aligned row-major tile (the layout the trainers use).
  auto ok_mat = [](const void* q, int64_t ld) { return q != nullptr && aligned16(q) && ld % 4 == 0; };
  static const bool tstore_on = [] {
    const char* e = std::getenv("CAGNET_GEMM_TSTORE");
    return !(e && e[0] == '0');
  }();
  auto epi_maps = [&](bool split) -> bool {
    if (!tstore_on) return false;
    if (split) return true;  // partial map set by the caller
    if (!ok_mat(d.C, d.ldc)) return false;
    if (d.epilogue == EPI_RELU && d.aux_out && !ok_mat(d.aux_out, d.ldao)) return false;
    if (d.epilogue == EPI_RELU_PRIME && !ok_mat(d.aux, d.ldaux)) return false;
    if (!encode_2d(&maps.c, d.C, static_cast<uint64_t>(d.n), static_cast<uint64_t>(d.m),
                   static_cast<uint64_t>(d.ldc), static_cast<uint32_t>(bn), BM, false))
      return false;
    if (d.epilogue == EPI_RELU && d.aux_out)
      return encode_2d(&maps.x, d.aux_out, static_cast<uint64_t>(d.n), static_cast<uint64_t>(d.m),
                       static_cast<uint64_t>(d.ldao), static_cast<uint32_t>(bn), BM, false);
    if (d.epilogue == EPI_RELU_PRIME)
      return encode_2d(&maps.x, d.aux, static_cast<uint64_t>(d.n), static_cast<uint64_t>(d.m),
                       static_cast<uint64_t>(d.ldaux), static_cast<uint32_t>(bn), BM, false);
    return true;
  };

  if (a_k) {
    // T·W / S·Wᵀ: W resident, no split (K is a feature width).
    const int nkb = static_cast<int>(ceil_div64(d.k, BK));
    if (static_cast<int64_t>(nkb) * 2 * bn * BK * 4 > kMaxResidentB) return false;
    p.a_ld = d.a_sm;
    // (A 128-row tile with a_ld <= 32 is one contiguous range, but reading its
    // 64 B rows thread-per-row is 16-way bank-conflicted; the SWIZZLE_128B
    // tensor box reads conflict-free, so bulk stays off for AMODE 0.)
    p.a_bulk = 0;
    if (!p.a_bulk && !encode_2d(&maps.a, d.A, static_cast<uint64_t>(d.k), static_cast<uint64_t>(d.m),
                                static_cast<uint64_t>(d.a_sm), BK, BM, true))
      return false;
    p.nkb_res = nkb;
    p.k_chunk = static_cast<int64_t>(nkb) * BK;
    p.chains = nkb >= 2 ? (bn <= 16 ? CAGNET_TM_CH16 : bn <= 48 ? 2 : 1) : 1;
    p.tstore = epi_maps(false) ? 1 : 0;
    const int grid = static_cast<int>(m_tiles < sms ? m_tiles : sms);
    launch_bn<0, false>(bn, maps, p, grid, stream);
    dump_trace(p, stream, "aw");
    return true;
  }
  if (a_m && b_stream_ok) {
    // Hᵀ·S: K = graph rows, split across CTAs, S streamed with H.
    p.a_ld = d.a_sk;
    static const bool bulk_on = [] {
      const char* e = std::getenv("CAGNET_GEMM_BULK");
      return e && e[0] == '1';
    }();
    p.a_bulk = (bulk_on && m_tiles == 1 && d.a_sk <= BM) ? 1 : 0;  // a 32-row k-block is contiguous
    p.s_bulk = (bulk_on && d.b_sk <= bn) ? 1 : 0;
    if (!p.a_bulk && !encode_2d(&maps.a, d.A, static_cast<uint64_t>(d.m), static_cast<uint64_t>(d.k),
                                static_cast<uint64_t>(d.a_sk), BM, BK, false))
      return false;
    if (!p.s_bulk && !encode_2d(&maps.b, d.B, static_cast<uint64_t>(d.n), static_cast<uint64_t>(d.k),
                                static_cast<uint64_t>(d.b_sk), static_cast<uint32_t>(bn), BK, false))
      return false;
    const int64_t kblocks = ceil_div64(d.k, BK);
    // One tile per CTA, no second wave: floor(SMs / M tiles) splits — but no
    // split longer than kMaxChunkRows: the tensor cores' fp32 accumulation
    // over a long K loses accuracy (measured on Amazon-shaped H0ᵀ S, 96 K+ rows
    // per split: 4.7e-4 relative to fp64), so long reductions take more,
    // shorter splits (persistent CTAs walk several) folded in fp64.
    static const int64_t kMaxChunkRows = [] {
      const char* e = std::getenv("CAGNET_HTS_CHUNK_ROWS");
      return e ? std::atoll(e) : 8192LL;
    }();
    int64_t splits = sms / m_tiles;
    const int64_t min_splits = ceil_div64(kblocks, std::max<int64_t>(kMaxChunkRows / BK, 1));
    if (splits < min_splits) splits = min_splits;
    if (splits > kblocks) splits = kblocks;
    if (splits < 1) splits = 1;
    p.k_chunk = ceil_div64(kblocks, splits) * BK;
    splits = ceil_div64(d.k, p.k_chunk);
    p.chains = p.k_chunk / BK >= 2 ? (bn <= 16 ? CAGNET_TM_CH16 : bn <= 48 ? 2 : 1) : 1;
    float* work = nullptr;
    if (splits > 1) {
      work = static_cast<float*>(
          stream_scratch(stream, static_cast<size_t>(splits) * p.mpad * p.pld * sizeof(float)));
      p.partial = work;
      p.tstore = encode_2d(&maps.c, work, static_cast<uint64_t>(d.n),
                           static_cast<uint64_t>(splits * p.mpad), static_cast<uint64_t>(p.pld),
                           static_cast<uint32_t>(bn), BM, false)
                     ? 1
                     : 0;
    } else {
      p.tstore = epi_maps(false) ? 1 : 0;
    }
    const int64_t tiles = m_tiles * splits;
    const int grid = static_cast<int>(tiles < sms ? tiles : sms);
    launch_bn<1, true>(bn, maps, p, grid, stream);
    dump_trace(p, stream, "hts");
    if (splits > 1) {
      const int64_t total = d.m * d.n;  // one warp per element
      const int blocks = static_cast<int>(ceil_div64(total, 8) < 8 * sms ? ceil_div64(total, 8) : 8 * sms);
      tm_reduce_kernel<<<blocks, 256, 0, stream>>>(p, static_cast<int>(splits));
      CG_LAUNCH_CHECK();
    }
    return true;
  }
  return false;
}

}  // namespace kern
}  // namespace cagnet
