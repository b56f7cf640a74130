// K2 — dense GEMM on 5th-generation tensor cores (tcgen05, sm_100a), split-TF32.
//
// Reference: gemm_add / gemm, dense.cpp:37-70 (fp64, k ascending).  The GCN
// contractions are T·W (n x f_in · f_in x f_out), Hᵀ·S (f_in x n · n x f_out,
// split-K) and S·Wᵀ (n x f_out · f_out x f_in).  Operands are fp32; each is
// split on the fly into hi = tf32_rn(x) and lo = tf32_rn(x - hi) and the
// product is accumulated in TMEM as hi·hi + hi·lo + lo·hi (three
// kind::tf32 MMAs per k-step), which keeps the relative error near 2^-21 —
// well inside the 1e-4 fp32 parity budget — while the tensor pipe does the
// math.  Every shape here is skinny (N <= 64), so the kernel is an HBM
// streaming kernel: 128 threads stage a 128 x 32 tile of A (and BN x 32 of B)
// from global memory into a 2-stage shared-memory ring in the UMMA canonical
// SWIZZLE_NONE layout (K-major or MN-major, whichever makes the global loads
// coalesced), one elected thread issues the MMAs, tcgen05.commit on an
// mbarrier releases the stage, and four epilogue warps drain TMEM with
// tcgen05.ld and apply the fused epilogue (ReLU + save Z, or ⊙ relu′(Z)).
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "tc.cuh"

namespace cagnet {
namespace kern {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int kThreads = 128;

struct Params {
  int64_t m, n, k;
  const float* A;
  int64_t a_sm, a_sk;
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
  float* partial;  // split-K workspace [splits][m][n]
  int64_t k_chunk;
};

// Staging modes: 0 = K contiguous (float4 along K, K-major smem),
//                1 = MN contiguous (float4 along MN, MN-major smem),
//                2 = generic strides (scalar loads, K-major smem).
template <int MODE>
struct Stager {
  // Loads item i (4 floats) of an R-row operand tile into v; elements outside
  // [0, rows) x [k0, kend) are zero.
  template <int R>
  __device__ static void load(float4& v, int i, int tid, const float* __restrict__ base,
                              int64_t s_mn, int64_t s_k, int64_t r0, int64_t rows, int64_t k0,
                              int64_t kend) {
    const int c = i * kThreads + tid;
    if constexpr (MODE == 1) {
      const int k = ((c >> 5) & 3) * 8 + (c & 7);
      const int quad = (c >> 7) * 4 + ((c >> 3) & 3);
      const int64_t gk = k0 + k;
      const int64_t gm = r0 + 4 * quad;
      if (gk < kend && gm + 3 < rows) {
        v = __ldg(reinterpret_cast<const float4*>(base + gk * s_k + gm));
      } else {
        float t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          t[j] = (gk < kend && gm + j < rows) ? __ldg(base + gk * s_k + (gm + j)) : 0.f;
        v = make_float4(t[0], t[1], t[2], t[3]);
      }
    } else {
      const int row = (c >> 6) * 8 + (c & 7);
      const int kq = (c >> 3) & 7;
      const int64_t gr = r0 + row;
      const int64_t gk = k0 + 4 * kq;
      if (MODE == 0 && gr < rows && gk + 3 < kend) {
        v = __ldg(reinterpret_cast<const float4*>(base + gr * s_mn + gk));
      } else {
        float t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          t[j] = (gr < rows && gk + j < kend) ? __ldg(base + gr * s_mn + (gk + j) * s_k) : 0.f;
        v = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
  }

  // Splits item i into hi/lo tf32 and stores it into the K-major
  // SWIZZLE_NONE stage layout: element (row, k) of a 32-wide k-block lives at
  // (row/8)*1024 + (k/4)*128 + (row%8)*16 + (k%4)*4 bytes (core matrices of
  // 8 rows x 16 B; K-direction stride 128 B, 8-row-group stride 1 KB).
  template <int R>
  __device__ static void store(char* hi, char* lo, int i, int tid, const float4& v) {
    const int c = i * kThreads + tid;
    if constexpr (MODE == 1) {
      // v holds rows 4q..4q+3 of one k; scatter them as scalars.  The store
      // order is rotated per lane so each warp-wide store hits 32 banks.
      const int k_lo = c & 7, q_lo = (c >> 3) & 3, k_hi = (c >> 5) & 3, q_hi = c >> 7;
      const int k = k_hi * 8 + k_lo;
      const int q = q_hi * 4 + q_lo;
      const int rot = ((k_lo >> 2) + 2 * (q_lo >> 1)) & 3;
      const uint32_t kpart = static_cast<uint32_t>((k >> 2) * 128 + (k & 3) * 4);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = (j + rot) & 3;
        const float x = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
        const int row = 4 * q + e;
        const uint32_t off = static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 16) + kpart;
        const float h = tc::to_tf32(x);
        *reinterpret_cast<float*>(hi + off) = h;
        *reinterpret_cast<float*>(lo + off) = tc::to_tf32(x - h);
      }
    } else {
      const int r_lo = c & 7, kq = (c >> 3) & 7, r_hi = c >> 6;
      const uint32_t off = static_cast<uint32_t>(r_hi * 1024 + kq * 128 + r_lo * 16);
      float4 h, l;
      h.x = tc::to_tf32(v.x);
      h.y = tc::to_tf32(v.y);
      h.z = tc::to_tf32(v.z);
      h.w = tc::to_tf32(v.w);
      l.x = tc::to_tf32(v.x - h.x);
      l.y = tc::to_tf32(v.y - h.y);
      l.z = tc::to_tf32(v.z - h.z);
      l.w = tc::to_tf32(v.w - h.w);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) = l;
    }
  }

  // Descriptor of k-step kk (8 tf32 = two 16 B core-matrix columns).
  __device__ static uint64_t desc(uint32_t base, int kk) {
    return tc::smem_desc(base + kk * 256, /*lbo=*/128, /*sbo=*/1024);
  }
};

__device__ __forceinline__ float apply_epilogue(const Params& p, int64_t r, int64_t c, float v) {
  if (p.accumulate) v += p.C[r * p.ldc + c];
  if (p.epilogue == EPI_RELU) {
    if (p.aux_out) p.aux_out[r * p.ldao + c] = v > 0.f ? v : 0.f;
  } else if (p.epilogue == EPI_RELU_PRIME) {
    v = p.aux[r * p.ldaux + c] > 0.f ? v : v * 0.f;
  }
  return v;
}

template <int BN, int AMODE, int BMODE>
__global__ void __launch_bounds__(kThreads, 1) gemm_tf32x3_kernel(const Params p) {
  constexpr int A_ITEMS = BM * BK / 4 / kThreads;  // 8
  constexpr int B_ITEMS = BN * BK / 4 / kThreads;  // BN / 16
  constexpr uint32_t A_BYTES = BM * BK * 4;
  constexpr uint32_t B_BYTES = BN * BK * 4;
  constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  // Both operands K-major in smem.  (MN-major tf32 operands need the
  // SWIZZLE_128B_BASE32B layout — cute sm100 builders; the plain MN-major
  // layouts return zeros — so MN-contiguous operands are transposed while
  // staging instead.)
  constexpr uint32_t IDESC = tc::idesc_tf32(BM, BN, 0, 0);

  extern __shared__ __align__(1024) char smem_raw[];
  // Swizzled (mode 3) tiles need 1024 B alignment; the allocation carries 1 KB slack.
  char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 2 * STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 2 * STAGE_BYTES + 16);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.y) * BN;
  const int64_t kbeg = static_cast<int64_t>(blockIdx.z) * p.k_chunk;
  const int64_t kend = kbeg + p.k_chunk < p.k ? kbeg + p.k_chunk : p.k;
  const int nkb = kend > kbeg ? static_cast<int>((kend - kbeg + BK - 1) / BK) : 0;

  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  float4 ra[A_ITEMS], rb[B_ITEMS];
  auto load_stage = [&](int kb) {
    const int64_t k0 = kbeg + static_cast<int64_t>(kb) * BK;
#pragma unroll
    for (int i = 0; i < A_ITEMS; ++i)
      Stager<AMODE>::template load<BM>(ra[i], i, tid, p.A, p.a_sm, p.a_sk, m0, p.m, k0, kend);
#pragma unroll
    for (int i = 0; i < B_ITEMS; ++i)
      Stager<BMODE>::template load<BN>(rb[i], i, tid, p.B, p.b_sn, p.b_sk, n0, p.n, k0, kend);
  };

  if (nkb > 0) load_stage(0);
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb & 1;
    char* st = smem + s * STAGE_BYTES;
    if (kb >= 2) tc::mbar_wait(&mbar[s], static_cast<uint32_t>(((kb >> 1) - 1) & 1));
#pragma unroll
    for (int i = 0; i < A_ITEMS; ++i)
      Stager<AMODE>::template store<BM>(st, st + A_BYTES, i, tid, ra[i]);
#pragma unroll
    for (int i = 0; i < B_ITEMS; ++i)
      Stager<BMODE>::template store<BN>(st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES, i, tid, rb[i]);
    tc::fence_proxy_async_smem();
    __syncthreads();
    if (kb + 1 < nkb) load_stage(kb + 1);
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t a_hi = tc::smem_u32(st), a_lo = a_hi + A_BYTES;
      const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t ah = Stager<AMODE>::desc(a_hi, kk);
        const uint64_t al = Stager<AMODE>::desc(a_lo, kk);
        const uint64_t bh = Stager<BMODE>::desc(b_hi, kk);
        const uint64_t bl = Stager<BMODE>::desc(b_lo, kk);
        tc::mma_tf32(tmem, ah, bh, IDESC, (kb | kk) != 0);
        tc::mma_tf32(tmem, ah, bl, IDESC, 1);
        tc::mma_tf32(tmem, al, bh, IDESC, 1);
      }
      tc::mma_commit(&mbar[s]);
    }
  }
  if (nkb > 0) {
    const int last = nkb - 1;
    tc::mbar_wait(&mbar[last & 1], static_cast<uint32_t>((last >> 1) & 1));
  }
  tc::tc_fence_after();

  // Epilogue: warp w owns TMEM lanes / tile rows [32w, 32w + 32).
  const int64_t r = m0 + warp * 32 + (tid & 31);
  const bool split = gridDim.z > 1;
#pragma unroll 1
  for (int cb = 0; cb < BN / 16; ++cb) {
    float v[16];
    if (nkb > 0) {
      tc::tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb * 16, v);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
    }
    if (r < p.m) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t c = n0 + cb * 16 + j;
        if (c < p.n) {
          if (split)
            p.partial[(static_cast<int64_t>(blockIdx.z) * p.m + r) * p.n + c] = v[j];
          else
            p.C[r * p.ldc + c] = apply_epilogue(p, r, c, v[j]);
        }
      }
    }
  }

  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// Deterministic split-K fold: C = epilogue((acc ? C : 0) + sum_z partial[z]).
__global__ void splitk_reduce_kernel(const Params p, int splits) {
  const int64_t total = p.m * p.n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / p.n, c = e % p.n;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += p.partial[static_cast<int64_t>(z) * total + e];
    p.C[r * p.ldc + c] = apply_epilogue(p, r, c, s);
  }
}

template <int BN, int AMODE, int BMODE>
void launch_bn(const Params& p, dim3 grid, cudaStream_t s) {
  constexpr int smem = 2 * (2 * BM * BK * 4 + 2 * BN * BK * 4) + 64 + 1024;
  auto kfn = gemm_tf32x3_kernel<BN, AMODE, BMODE>;
  static std::atomic<uint64_t> configured{0};  // one bit per device
  const int dev = current_device();
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    CG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.fetch_or(bit);
  }
  kfn<<<grid, kThreads, smem, s>>>(p);
  CG_LAUNCH_CHECK();
}

template <int AMODE, int BMODE>
void launch_modes(int bn, const Params& p, dim3 grid, cudaStream_t s) {
  switch (bn) {
    case 16: return launch_bn<16, AMODE, BMODE>(p, grid, s);
    case 32: return launch_bn<32, AMODE, BMODE>(p, grid, s);
    case 48: return launch_bn<48, AMODE, BMODE>(p, grid, s);
    case 64: return launch_bn<64, AMODE, BMODE>(p, grid, s);
    default: return launch_bn<128, AMODE, BMODE>(p, grid, s);
  }
}

template <int AMODE>
void launch_bmode(int bmode, int bn, const Params& p, dim3 grid, cudaStream_t s) {
  switch (bmode) {
    case 0: return launch_modes<AMODE, 0>(bn, p, grid, s);
    case 1: return launch_modes<AMODE, 1>(bn, p, grid, s);
    default: return launch_modes<AMODE, 2>(bn, p, grid, s);
  }
}

bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }

// CAGNET_GEMM_TMA=0 forces the register-staged kernel (A/B comparisons).
bool gemm_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CAGNET_GEMM_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CAGNET_GEMM_TM=0 disables the A-in-TMEM kernel (A/B comparisons).
bool gemm_tm_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CAGNET_GEMM_TM");
    return !(e && e[0] == '0');
  }();
  return on;
}

// 0: K contiguous & vectorisable, 1: MN contiguous & vectorisable, 2: generic.
int pick_mode(const float* base, int64_t s_mn, int64_t s_k) {
  if (!aligned16(base)) return 2;
  if (s_k == 1 && s_mn % 4 == 0) return 0;
  if (s_mn == 1 && s_k % 4 == 0) return 1;
  return 2;
}

}  // namespace

void gemm_tf32x3(const GemmDesc& d, cudaStream_t stream) {
  if (d.m <= 0 || d.n <= 0) return;
  if (gemm_small_try(d, stream)) return;
  if (gemm_tm_enabled() && gemm_tm_try(d, stream)) return;
  if (gemm_tma_enabled() && gemm_tma_try(d, stream)) return;
  Params p{};
  p.m = d.m;
  p.n = d.n;
  p.k = d.k < 0 ? 0 : d.k;
  p.A = d.A;
  p.a_sm = d.a_sm;
  p.a_sk = d.a_sk;
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

  const int bn = d.n <= 16 ? 16 : d.n <= 32 ? 32 : d.n <= 48 ? 48 : d.n <= 64 ? 64 : 128;
  const int64_t m_tiles = ceil_div64(d.m, BM);
  const int64_t n_tiles = ceil_div64(d.n, bn);
  const int64_t tiles = m_tiles * n_tiles;
  const int sms = num_sms(current_device());

  // Split K when the output tiles cannot fill the machine (Hᵀ·S has K = n).
  int64_t splits = 1;
  const int64_t kblocks = ceil_div64(p.k, BK);
  if (tiles < 2 * sms && kblocks >= 8) {
    splits = ceil_div64(2 * sms, tiles);
    const int64_t max_splits = kblocks / 4;  // at least 4 k-blocks per split
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
  }
  p.k_chunk = splits > 1 ? round_up(ceil_div64(p.k, splits), BK) : (p.k > 0 ? p.k : BK);
  if (splits > 1) splits = ceil_div64(p.k, p.k_chunk);

  float* work = nullptr;
  if (splits > 1) {
    work = static_cast<float*>(stream_scratch(stream, static_cast<size_t>(splits) * d.m * d.n * sizeof(float)));
    p.partial = work;
  }
  const int amode = pick_mode(d.A, d.a_sm, d.a_sk);
  const int bmode = pick_mode(d.B, d.b_sn, d.b_sk);
  const dim3 grid(static_cast<unsigned>(m_tiles), static_cast<unsigned>(n_tiles),
                  static_cast<unsigned>(splits));
  switch (amode) {
    case 0: launch_bmode<0>(bmode, bn, p, grid, stream); break;
    case 1: launch_bmode<1>(bmode, bn, p, grid, stream); break;
    default: launch_bmode<2>(bmode, bn, p, grid, stream); break;
  }
  if (splits > 1) {
    const int64_t total = d.m * d.n;
    const int blocks = static_cast<int>(ceil_div64(total, 256) < 4 * sms ? ceil_div64(total, 256)
                                                                          : 4 * sms);
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(p, static_cast<int>(splits));
    CG_LAUNCH_CHECK();
  }
}

}  // namespace kern
}  // namespace cagnet
