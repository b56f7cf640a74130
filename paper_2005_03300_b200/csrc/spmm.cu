// K1 — CSR SpMM for the GCN propagation Aᵀ·H (forward) and A·G (backward).
//
// Reference: spmm_add, csr.cpp:164-179 — acc(i,:) += v_k * H(c_k,:) for the
// nonzeros of row i in ascending order.  The wide-row kernel keeps that order
// per output element (one fp32 FMA per nonzero, sequential per lane).  The
// narrow-row kernel (spmm_nzpar_kernel, every f <= 32 SpMM) splits a row's
// nonzeros over QPR sub-teams — sub-team q takes the entries at positions
// q, q + QPR, ... from the QPR-aligned start, each in ascending order — and
// folds the QPR partial sums in a fixed xor-shuffle tree: deterministic, but
// a different fp32 summation order than the reference's, within the 1e-4 bar.
//
// Wide-row mapping: a row group of LPR lanes owns one output row; each lane holds VPL
// 128-bit column vectors of the row in registers.  Column indices and values
// are loaded once, coalesced, by the LPR lanes of the group and broadcast to
// the group with warp shuffles; every gathered H row is read as LPR*16 B
// contiguous segments.  Rows of an Erdős–Rényi graph have near-uniform length
// (binomial degree), so row-group mapping balances without merge-path.
//
// Rows are given as [seg_begin[i], seg_end[i]) ranges, so a column block of
// a CSR matrix (a contiguous sub-range of every sorted row) is processed
// without copying: the L2-aware blocking in spmm_blocked() runs one pass per
// column block whose H panel fits in L2 and accumulates the passes in
// ascending column order — the reference's own order (csr.hpp:68-70).
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cagnet {
namespace kern {
namespace {

constexpr int kThreads = 256;

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
};
template <>
struct VecT<1> {
  using T = float;
};

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ldg_policy(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void fma_vec(float4& acc, float v, const float4& h) {
  acc.x = fmaf(v, h.x, acc.x);
  acc.y = fmaf(v, h.y, acc.y);
  acc.z = fmaf(v, h.z, acc.z);
  acc.w = fmaf(v, h.w, acc.w);
}
__device__ __forceinline__ void fma_vec(float& acc, float v, const float& h) {
  acc = fmaf(v, h, acc);
}
__device__ __forceinline__ void zero_vec(float4& a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void zero_vec(float& a) { a = 0.f; }

// Loads vector `vec` of a row (f valid floats) with a scalar tail.
__device__ __forceinline__ float4 load_vec(const float* __restrict__ row, int vec, int f) {
  const int c = vec * 4;
  if (c + 4 <= f) return __ldg(reinterpret_cast<const float4*>(row + c));
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c + 0 < f) r.x = __ldg(row + c + 0);
  if (c + 1 < f) r.y = __ldg(row + c + 1);
  if (c + 2 < f) r.z = __ldg(row + c + 2);
  return r;
}

__device__ __forceinline__ void store_vec(float* row, int vec, int f, const float4& v) {
  const int c = vec * 4;
  if (c + 4 <= f) {
    *reinterpret_cast<float4*>(row + c) = v;
    return;
  }
  if (c + 0 < f) row[c + 0] = v.x;
  if (c + 1 < f) row[c + 1] = v.y;
  if (c + 2 < f) row[c + 2] = v.z;
}

struct SpmmArgs {
  int64_t n_rows;
  const int64_t* seg_begin;
  const int64_t* seg_end;
  const int32_t* col_idx;
  const float* vals;
  const float* H;
  int64_t ldh;
  int f;
  float* T;
  int64_t ldt;
  double mean_row_nnz;  // host-side hint for the row-team shape
  SpmmEpi epi;          // fused row epilogue (EPI kernels only)
  // Optional interleaved copy of (col_idx, vals) as int2 {col, float bits}:
  // one 8 B load per nonzero instead of two 4 B loads (narrow-row kernel).
  const int2* colval = nullptr;
  SpmmPacked packed;  // packed.e != nullptr: the packed stream (narrow-row kernel, LV = 2 / 4)
};

// VEC = 4: 16-byte vectors (requires 16 B aligned rows, ld a multiple of 4); VEC = 1: scalars.
// With VEC = 4 a row's last vector is always gathered whole, even when f is not a
// multiple of 4: the floats past f lie inside the row's padded leading dimension, only
// feed accumulator lanes that are never stored (stores and the accumulate read are
// masked to f), so a ragged width costs no scalar loads.
template <int VEC, int LPR, int VPL, bool ACC, bool TAIL>
__global__ void __launch_bounds__(kThreads, VPL == 1 ? 4 : 1) spmm_rows_kernel(const SpmmArgs a) {
  using V = typename VecT<VEC>::T;
  constexpr int RPW = 32 / LPR;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane % LPR;
  const int grp = lane / LPR;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t row = warp * RPW + grp;
  const int f = a.f;
  const int nvec = (f + VEC - 1) / VEC;
  const int32_t* __restrict__ col_idx = a.col_idx;
  const float* __restrict__ vals = a.vals;
  const float* __restrict__ H = a.H;

  int64_t beg = 0, len = 0;
  if (row < a.n_rows) {
    beg = a.seg_begin[row];
    len = a.seg_end[row] - beg;
  }
  // Uniform trip count across the warp so every lane joins the shuffles.
  int64_t maxlen = len;
#pragma unroll
  for (int o = 16; o >= LPR; o >>= 1) {
    const int64_t other = __shfl_xor_sync(0xffffffffu, maxlen, o);
    maxlen = other > maxlen ? other : maxlen;
  }

  float* trow = a.T + row * a.ldt;
  V acc[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    zero_vec(acc[i]);
    const int vec = sub + i * LPR;
    if (ACC && row < a.n_rows && vec < nvec) {
      if constexpr (VEC == 4)
        acc[i] = load_vec(trow, vec, f);
      else
        acc[i] = trow[vec];
    }
  }

  const int src0 = grp * LPR;
  if constexpr (VPL > 1) {
    // Wide rows: every lane already has VPL independent vector gathers per
    // nonzero in flight; walk the group's nonzeros one at a time.
    for (int64_t base = 0; base < maxlen; base += LPR) {
      int c = 0;
      float v = 0.f;
      if (base + sub < len) {
        c = __ldg(col_idx + beg + base + sub);
        v = __ldg(vals + beg + base + sub);
      }
      const int64_t remain = len - base;
#pragma unroll 4
      for (int t = 0; t < LPR; ++t) {
        const int cc = __shfl_sync(0xffffffffu, c, src0 + t);
        const float vv = __shfl_sync(0xffffffffu, v, src0 + t);
        if (t < remain) {
          const float* hrow = H + static_cast<int64_t>(cc) * a.ldh;
          V hv[VPL];
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            const int vec = sub + i * LPR;
            zero_vec(hv[i]);
            if (vec < nvec) {
              if constexpr (VEC == 4)
                hv[i] = __ldg(reinterpret_cast<const float4*>(hrow) + vec);
              else
                hv[i] = __ldg(hrow + vec);
            }
          }
#pragma unroll
          for (int i = 0; i < VPL; ++i) fma_vec(acc[i], vv, hv[i]);
        }
      }
    }
  } else {
  // Narrow rows (one vector per lane): a chunk covers U*LPR nonzeros; the
  // gathers are issued in batches of TB nonzeros, predicated rather than
  // branched so they are all in flight, and folded in ascending order.
  constexpr int U = LPR >= 8 ? 1 : 8 / LPR;
  constexpr int CH = U * LPR;
  constexpr int TB = VPL >= 8 ? 1 : 8 / VPL;
  for (int64_t base = 0; base < maxlen; base += CH) {
    int c[U];
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = base + u * LPR + sub;
      c[u] = q < len ? __ldg(col_idx + beg + q) : 0;
      v[u] = q < len ? __ldg(vals + beg + q) : 0.f;
    }
#pragma unroll
    for (int t0 = 0; t0 < CH; t0 += TB) {
      V hv[TB][VPL];
      float w[TB];
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) {
        const int t = t0 + tb;
        if (t < CH) {
          const int cc = __shfl_sync(0xffffffffu, c[t / LPR], src0 + t % LPR);
          w[tb] = __shfl_sync(0xffffffffu, v[t / LPR], src0 + t % LPR);
          const bool live = base + t < len;
          const float* hrow = H + static_cast<int64_t>(cc) * a.ldh;
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            const int vec = sub + i * LPR;
            V zero;
            zero_vec(zero);
            // Select form (not a branch) so every gather is issued up front;
            // dead slots read nothing and contribute w = 0 times 0.
            if constexpr (VEC == 4)
              hv[tb][i] = (live && vec < nvec)
                              ? __ldg(reinterpret_cast<const float4*>(hrow) + vec)
                              : zero;
            else
              hv[tb][i] = (live && vec < nvec) ? __ldg(hrow + vec) : zero;
          }
        }
      }
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) {
        if (t0 + tb < CH) {
#pragma unroll
          for (int i = 0; i < VPL; ++i) fma_vec(acc[i], w[tb], hv[tb][i]);
        }
      }
    }
  }
  }

  if (row < a.n_rows) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int vec = sub + i * LPR;
      if (vec < nvec) {
        if constexpr (VEC == 4)
          store_vec(trow, vec, f, acc[i]);
        else
          trow[vec] = acc[i];
      }
    }
  }
}

template <int VEC, int LPR, int VPL>
void launch_one(const SpmmArgs& a, bool acc, cudaStream_t s) {
  constexpr int rows_per_block = (kThreads / 32) * (32 / LPR);
  const unsigned g = static_cast<unsigned>(ceil_div64(a.n_rows, rows_per_block));
  if (acc)
    spmm_rows_kernel<VEC, LPR, VPL, true, false><<<g, kThreads, 0, s>>>(a);
  else
    spmm_rows_kernel<VEC, LPR, VPL, false, false><<<g, kThreads, 0, s>>>(a);
  CG_LAUNCH_CHECK();
}

template <int VEC, int LPR>
void launch_vpl(int vpl, const SpmmArgs& a, bool acc, cudaStream_t s) {
  switch (vpl) {
    case 1: return launch_one<VEC, LPR, 1>(a, acc, s);
    case 2: return launch_one<VEC, LPR, 2>(a, acc, s);
    case 3: return launch_one<VEC, LPR, 3>(a, acc, s);
    case 4: return launch_one<VEC, LPR, 4>(a, acc, s);
    case 5: return launch_one<VEC, LPR, 5>(a, acc, s);
    case 6: return launch_one<VEC, LPR, 6>(a, acc, s);
    case 7: return launch_one<VEC, LPR, 7>(a, acc, s);
    default: return launch_one<VEC, LPR, 8>(a, acc, s);
  }
}

// Picks lanes-per-row (4..32) and vectors-per-lane (<= 8) maximising the share
// of active vector slots; ties go to wider groups (longer coalesced segments).
void pick_shape(int nvec, int* lpr, int* vpl) {
  int best_l = 32, best_v = (nvec + 31) / 32;
  double best_u = -1.0;
  for (int l = 4; l <= 32; l *= 2) {
    const int v = (nvec + l - 1) / l;
    if (v > 8) continue;
    const double u = static_cast<double>(nvec) / (l * v);
    if (u >= best_u) {
      best_u = u;
      best_l = l;
      best_v = v;
    }
  }
  *lpr = best_l;
  *vpl = best_v < 1 ? 1 : best_v;
}

// Fused epilogue (SpmmEpi) of a row team whose lanes all hold the reduced
// row: lane vec has columns [4 vec, 4 vec + 4).  With W, team lane tl
// computes output columns tl, tl + TEAM, ... as sum_k t_k W[k, c] in fp32
// (t_k fetched by warp shuffles); every lane of the warp runs the shuffle
// loop, rows past the end only skip the stores.
template <int LV, int TEAM>
__device__ __forceinline__ void spmm_row_epilogue(const SpmmArgs& a, int64_t row, int lane, int vec,
                                                  int q, bool vec_ok, const float4& acc) {
  const SpmmEpi& e = a.epi;
  const bool live = row < a.n_rows;
  const int f = a.f;
  if (e.raw_out && live && q == 0 && vec_ok) store_vec(e.raw_out + row * e.raw_ld, vec, f, acc);
  if (e.W == nullptr) {
    if (!(live && q == 0 && vec_ok)) return;
    float4 z = acc;
    if (e.mask) {
      const float4 m = load_vec(e.mask + row * e.mask_ld, vec, f);
      z.x = m.x > 0.f ? z.x : z.x * 0.f;
      z.y = m.y > 0.f ? z.y : z.y * 0.f;
      z.z = m.z > 0.f ? z.z : z.z * 0.f;
      z.w = m.w > 0.f ? z.w : z.w * 0.f;
    }
    store_vec(a.T + row * a.ldt, vec, f, z);
    const float4 rz = make_float4(fmaxf(z.x, 0.f), fmaxf(z.y, 0.f), fmaxf(z.z, 0.f), fmaxf(z.w, 0.f));
    if (e.relu_out) store_vec(e.relu_out + row * e.relu_ld, vec, f, rz);
    for (int p = 0; p < e.push_n; ++p)
      store_vec(e.push_bufs[p] + e.push_off + row * e.push_ld, vec, f, e.push_relu ? rz : z);
    return;
  }
  constexpr int SLOTS = (kSpmmEpiMaxFo + TEAM - 1) / TEAM;
  const int tl = lane % TEAM;
  const int base = lane - tl;
  const int nvec = (f + 3) / 4;
  float z[SLOTS];
#pragma unroll
  for (int i = 0; i < SLOTS; ++i) z[i] = 0.f;
  for (int v4 = 0; v4 < nvec; ++v4) {
    const int src = base + (v4 % LV);
    float t[4];
    t[0] = __shfl_sync(0xffffffffu, acc.x, src);
    t[1] = __shfl_sync(0xffffffffu, acc.y, src);
    t[2] = __shfl_sync(0xffffffffu, acc.z, src);
    t[3] = __shfl_sync(0xffffffffu, acc.w, src);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 4 * v4 + j;
      if (k < f) {
        const float* wk = e.W + k * e.w_sk;
#pragma unroll
        for (int i = 0; i < SLOTS; ++i) {
          const int c = tl + i * TEAM;
          if (c < e.fo) z[i] = fmaf(t[j], __ldg(wk + c * e.w_sn), z[i]);
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int i = 0; i < SLOTS; ++i) {
    const int c = tl + i * TEAM;
    if (c < e.fo) {
      float v = z[i];
      if (e.mask) v = e.mask[row * e.mask_ld + c] > 0.f ? v : v * 0.f;
      a.T[row * a.ldt + c] = v;
      if (e.relu_out) e.relu_out[row * e.relu_ld + c] = fmaxf(v, 0.f);
    }
  }
}

// Narrow rows (f <= 32): a team of QPR x LV lanes owns one output row; LV
// lanes cover the row's float4 vectors and the QPR sub-teams stride over the
// row's nonzeros (sub-team q takes q, q+QPR, ...), so every lane streams
// independent gathers with no shuffles in the loop (U in flight); the QPR
// partial sums are folded with xor shuffles at the end (deterministic order).
// CV = 1: the nonzeros come from the interleaved (col, value) stream a.colval
// (one 8 B load per step instead of a column and a value load).  CV = 2: the
// packed stream a.packed — 4 B per nonzero, 8 sub-teams' entries in 32 B: one L1
// wavefront per step, where 8 B loads take about two (half-warp passes); the
// kernel is bound by L1 LSU wavefronts (one per gathered 64 B row), so this is
// ~10 % of its time (profiles/r02_micro_packed_stream.txt).
template <int LV, int QPR, int U, bool ACC, int CV, int NT = kThreads, int HINT = 0,
          bool FULLV = false, bool EPI = false>
// Full occupancy (32 registers): the gathers need every warp in flight.  The
// fused-epilogue variants of short rows (teams of < 16 lanes) spill in their
// epilogue at 32, and are still faster than at 64 registers and half the
// warps (Amazon-shaped SpMM 5.14 -> 5.34 ms with 64).
__global__ void __launch_bounds__(NT, 2048 / NT) spmm_nzpar_kernel(const SpmmArgs a) {
  constexpr int TEAM = LV * QPR;
  constexpr int RPW = 32 / TEAM;
  const int lane = threadIdx.x & 31;
  const int vec = lane % LV;
  const int q = (lane % TEAM) / LV;
  const int64_t row =
      ((static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x) >> 5) * RPW + lane / TEAM;
  uint64_t pol = 0;
  if (HINT) pol = l2_evict_last_policy();
  const int f = a.f;
  const int nvec = (f + 3) / 4;
  // Lanes past the row's last vector idle on the gathers (only when nvec < LV).
  const bool vec_ok = FULLV || vec < nvec;
  // Row c of H starts c * ldh * 4 bytes in: one 32x32->64 multiply-add.
  const char* __restrict__ hbase = reinterpret_cast<const char*>(a.H) + vec * 16;
  const uint32_t ldh_bytes = static_cast<uint32_t>(a.ldh * 4);

  int64_t nz_b = 0, nz_e = 0;
  if (row < a.n_rows) {
    nz_b = a.seg_begin[row];
    nz_e = a.seg_end[row];
  }
  const int32_t* __restrict__ cp = a.col_idx + nz_b + q;
  const float* __restrict__ vp = a.vals + nz_b + q;
  const int32_t* ce = a.col_idx + nz_e;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  auto gather = [&](int c) -> float4 {
    if (!vec_ok) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* src = reinterpret_cast<const float4*>(
        hbase + static_cast<uint64_t>(static_cast<uint32_t>(c)) * ldh_bytes);
    if (HINT) return ldg_policy(src, pol);
    return __ldg(src);
  };
  // The CSR arrays are streamed once: evict-first so they do not push the
  // gathered H rows out of L2.
  auto ld_c = [&](const int32_t* p) { return HINT ? __ldcs(p) : __ldg(p); };
  auto ld_v = [&](const float* p) { return HINT ? __ldcs(p) : __ldg(p); };
  if constexpr (CV == 2) {
    // Same walk over the packed stream; w = rsqrt(d_col), the row scale is
    // applied once after the fold.
    const uint32_t* __restrict__ pk = a.packed.e;
    const int bits = a.packed.bits;
    const uint32_t cmask = (1u << bits) - 1u;
    auto weight = [&](uint32_t x) { return rsqrtf(static_cast<float>(x >> bits)); };
    const uint32_t* pe = pk + nz_e;
    const uint32_t* p = pk + nz_b + q;
    if constexpr (QPR > 1) {
      const int64_t head = nz_b & ~static_cast<int64_t>(QPR - 1);
      if (head != nz_b) {
        const uint32_t* hp = pk + head + q;
        if (hp >= pk + nz_b && hp < pe) {
          const uint32_t x = __ldg(hp);
          fma_vec(acc, weight(x), gather(static_cast<int>(x & cmask)));
        }
        p = hp + QPR;
      }
    }
    for (; p + (U - 1) * QPR < pe; p += U * QPR) {
      float4 h[U];
      float w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t x = __ldg(p + u * QPR);
        w[u] = weight(x);
        h[u] = gather(static_cast<int>(x & cmask));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) fma_vec(acc, w[u], h[u]);
    }
#pragma unroll 1
    for (; p < pe; p += QPR) {
      const uint32_t x = __ldg(p);
      fma_vec(acc, weight(x), gather(static_cast<int>(x & cmask)));
    }
  } else if constexpr (CV) {
    // The QPR sub-teams read QPR consecutive {col, val} entries per step; the
    // row's segment is walked from the QPR-aligned entry at or below nz_b, so
    // every step's entries sit in one 64 B-aligned chunk (one L1 wavefront,
    // never two) — the head group is peeled with a range predicate.
    const int2* pe = a.colval + nz_e;
    const int2* __restrict__ p = a.colval + nz_b + q;
    if constexpr (QPR > 1) {
      const int64_t head = nz_b & ~static_cast<int64_t>(QPR - 1);
      if (head != nz_b) {
        const int2* hp = a.colval + head + q;
        if (hp >= a.colval + nz_b && hp < pe) {
          const int2 x = __ldg(hp);
          fma_vec(acc, __int_as_float(x.y), gather(x.x));
        }
        p = hp + QPR;
      }
    }
    for (; p + (U - 1) * QPR < pe; p += U * QPR) {
      float4 h[U];
      float w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int2 x = __ldg(p + u * QPR);
        w[u] = __int_as_float(x.y);
        h[u] = gather(x.x);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) fma_vec(acc, w[u], h[u]);
    }
    for (; p < pe; p += QPR) {
      const int2 x = __ldg(p);
      fma_vec(acc, __int_as_float(x.y), gather(x.x));
    }
  } else {
    for (; cp + (U - 1) * QPR < ce; cp += U * QPR, vp += U * QPR) {
      float4 h[U];
      float w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = ld_c(cp + u * QPR);
        w[u] = ld_v(vp + u * QPR);
        h[u] = gather(c);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) fma_vec(acc, w[u], h[u]);
    }
    for (; cp < ce; cp += QPR, vp += QPR) fma_vec(acc, ld_v(vp), gather(ld_c(cp)));
  }
#pragma unroll
  for (int o = LV; o < TEAM; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if constexpr (CV == 2) {
    if (row < a.n_rows) {
      const float s = __ldg(a.packed.row_scale + row);
      acc.x *= s;
      acc.y *= s;
      acc.z *= s;
      acc.w *= s;
    }
  }
  if constexpr (EPI) {
    if (ACC && row < a.n_rows && vec_ok) {
      // Final pass of a split propagation: fold in the earlier passes' partial.
      const float4 old = load_vec(a.T + row * a.ldt, vec, f);
      acc.x = old.x + acc.x;
      acc.y = old.y + acc.y;
      acc.z = old.z + acc.z;
      acc.w = old.w + acc.w;
    }
    // Pushed rows become visible to the peers at kernel completion; the flag
    // kernel that follows on this stream fences before raising their flags.
    spmm_row_epilogue<LV, TEAM>(a, row, lane, vec, q, vec_ok, acc);
    return;
  }
  if (row < a.n_rows && q == 0 && vec_ok) {
    float* trow = a.T + row * a.ldt;
    if (ACC) {
      const float4 old = load_vec(trow, vec, f);
      acc.x = old.x + acc.x;
      acc.y = old.y + acc.y;
      acc.z = old.z + acc.z;
      acc.w = old.w + acc.w;
    }
    store_vec(trow, vec, f, acc);
  }
}

template <int LV, int QPR, int U, int NT, int HINT, int CV>
void launch_nzpar_cv(const SpmmArgs& a, bool acc, bool epi, unsigned g, bool full, cudaStream_t s) {
  if (epi && acc) {
    if (full)
      spmm_nzpar_kernel<LV, QPR, U, true, CV, NT, 0, true, true><<<g, NT, 0, s>>>(a);
    else
      spmm_nzpar_kernel<LV, QPR, U, true, CV, NT, 0, false, true><<<g, NT, 0, s>>>(a);
  } else if (epi) {
    if (full)
      spmm_nzpar_kernel<LV, QPR, U, false, CV, NT, 0, true, true><<<g, NT, 0, s>>>(a);
    else
      spmm_nzpar_kernel<LV, QPR, U, false, CV, NT, 0, false, true><<<g, NT, 0, s>>>(a);
  } else if (acc) {
    if (full)
      spmm_nzpar_kernel<LV, QPR, U, true, CV, NT, HINT, true><<<g, NT, 0, s>>>(a);
    else
      spmm_nzpar_kernel<LV, QPR, U, true, CV, NT, HINT><<<g, NT, 0, s>>>(a);
  } else {
    if (full)
      spmm_nzpar_kernel<LV, QPR, U, false, CV, NT, HINT, true><<<g, NT, 0, s>>>(a);
    else
      spmm_nzpar_kernel<LV, QPR, U, false, CV, NT, HINT><<<g, NT, 0, s>>>(a);
  }
}

template <int LV, int QPR, int U, int NT, int HINT>
void launch_nzpar_v(const SpmmArgs& a, bool acc, bool epi, cudaStream_t s) {
  constexpr int rows_per_block = (NT / 32) * (32 / (LV * QPR));
  const unsigned g = static_cast<unsigned>(ceil_div64(a.n_rows, rows_per_block));
  // Full vectors: every lane of the LV-wide row team owns a live float4.
  const bool full = (a.f + 3) / 4 == LV;
  if constexpr (LV == 2 || LV == 4) {
    if (a.packed.e) {
      launch_nzpar_cv<LV, QPR, U, NT, HINT, 2>(a, acc, epi, g, full, s);
      CG_LAUNCH_CHECK();
      return;
    }
  }
  if (a.colval)
    launch_nzpar_cv<LV, QPR, U, NT, HINT, 1>(a, acc, epi, g, full, s);
  else
    launch_nzpar_cv<LV, QPR, U, NT, HINT, 0>(a, acc, epi, g, full, s);
  CG_LAUNCH_CHECK();
}

// Tuning knob for experiments (CAGNET_SPMM_TUNE=<variant>); 0 = the default
// (128-thread CTAs, U = 4 gathers in flight per lane, no cache hints — the
// fastest on the Reddit-shaped graph: 0.548 ms vs 0.565 ms with L2 evict hints
// (variant 2), 0.561 ms with 256-thread CTAs and no gain from U = 8 at f = 16).
int spmm_tune() {
  static const int v = [] {
    const char* e = getenv("CAGNET_SPMM_TUNE");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int LV, int QPR>
void launch_nzpar(const SpmmArgs& a, bool acc, bool epi, cudaStream_t s) {
  if (epi) return launch_nzpar_v<LV, QPR, 4, 128, 0>(a, acc, true, s);
  switch (spmm_tune()) {
    case 2: return launch_nzpar_v<LV, QPR, 4, 128, 1>(a, acc, false, s);
    default: return launch_nzpar_v<LV, QPR, 4, 128, 0>(a, acc, false, s);
  }
}

template <int LV>
void launch_nzpar_q(int qpr, const SpmmArgs& a, bool acc, bool epi, cudaStream_t s) {
  switch (qpr) {
    case 1: return launch_nzpar<LV, 1>(a, acc, epi, s);
    case 2: if constexpr (LV <= 16) return launch_nzpar<LV, 2>(a, acc, epi, s); break;
    case 4: if constexpr (LV <= 8) return launch_nzpar<LV, 4>(a, acc, epi, s); break;
    default: if constexpr (LV <= 4) return launch_nzpar<LV, 8>(a, acc, epi, s); break;
  }
  launch_nzpar<LV, 1>(a, acc, epi, s);
}

template <int VEC>
void dispatch(const SpmmArgs& a, bool acc, bool epi, cudaStream_t s) {
  const int nvec = (a.f + VEC - 1) / VEC;
  if (VEC == 4 && nvec <= 8) {
    // Sub-teams per row from the mean row length (8 nonzeros per sub-team
    // at least), capped by the warp width.
    const int lv = nvec <= 1 ? 1 : nvec <= 2 ? 2 : nvec <= 4 ? 4 : 8;
    int qpr = 32 / lv;
    const double mean = a.mean_row_nnz;
    while (qpr > 1 && mean < 8.0 * qpr) qpr >>= 1;
    if (qpr > 8) qpr = 8;
    switch (lv) {
      case 1: return launch_nzpar_q<1>(qpr, a, acc, epi, s);
      case 2: return launch_nzpar_q<2>(qpr, a, acc, epi, s);
      case 4: return launch_nzpar_q<4>(qpr, a, acc, epi, s);
      default: return launch_nzpar_q<8>(qpr, a, acc, epi, s);
    }
  }
  require(!epi, "spmm: fused epilogue needs f <= 32 and 16 B-aligned rows");
  int lpr, vpl;
  pick_shape(nvec, &lpr, &vpl);
  switch (lpr) {
    case 4: return launch_vpl<VEC, 4>(vpl, a, acc, s);
    case 8: return launch_vpl<VEC, 8>(vpl, a, acc, s);
    case 16: return launch_vpl<VEC, 16>(vpl, a, acc, s);
    default: return launch_vpl<VEC, 32>(vpl, a, acc, s);
  }
}

// split[b * rows + r] = first nonzero of row r with column >= b * step.
__global__ void column_splits_kernel(int64_t rows, int nb, int64_t step,
                                     const int64_t* __restrict__ row_ptr,
                                     const int32_t* __restrict__ col_idx,
                                     int64_t* __restrict__ split) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t b0 = row_ptr[r], e0 = row_ptr[r + 1];
  int64_t lo = b0;
  split[r] = b0;
  for (int b = 1; b < nb; ++b) {
    const int64_t key = static_cast<int64_t>(b) * step;
    int64_t hi = e0;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col_idx[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    split[static_cast<int64_t>(b) * rows + r] = lo;
  }
  split[static_cast<int64_t>(nb) * rows + r] = e0;
}

}  // namespace

void spmm_segments(int64_t n_rows, const int64_t* seg_begin, const int64_t* seg_end,
                   const int32_t* col_idx, const float* vals, const float* H, int64_t ldh, int f,
                   float* T, int64_t ldt, bool accumulate, cudaStream_t stream, int64_t nnz,
                   const SpmmEpi* epi, const int2* colval, const SpmmPacked* packed) {
  if (n_rows <= 0 || f <= 0) return;
  const double mean = nnz >= 0 ? static_cast<double>(nnz) / static_cast<double>(n_rows) : 64.0;
  const bool aligned = (ldh % 4 == 0) && (ldt % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(H) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(T) % 16 == 0);
  if (epi) {
    require(aligned && f <= kSpmmEpiMaxF && epi->fo <= kSpmmEpiMaxFo,
            "spmm: fused epilogue needs a final f <= 32 SpMM on 16 B-aligned rows");
    require(!accumulate || epi->W == nullptr,
            "spmm: an accumulating fused epilogue cannot change the row width");
    SpmmArgs a{n_rows, seg_begin, seg_end, col_idx, vals, H, ldh, f, T, ldt, mean, *epi, colval,
               packed ? *packed : SpmmPacked{}};
    dispatch<4>(a, accumulate, true, stream);
    return;
  }
  // Column chunks of at most 32 lanes * 8 vectors keep accumulators in registers.
  const int chunk = aligned ? 32 * 8 * 4 : 32 * 8;
  for (int c0 = 0; c0 < f; c0 += chunk) {
    SpmmArgs a{n_rows, seg_begin, seg_end, col_idx, vals, H + c0, ldh, f - c0 < chunk ? f - c0 : chunk,
               T + c0, ldt, mean, SpmmEpi{}, colval, packed ? *packed : SpmmPacked{}};
    if (aligned)
      dispatch<4>(a, accumulate, false, stream);
    else
      dispatch<1>(a, accumulate, false, stream);
  }
}

void spmm_csr(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
              const float* H, int64_t ldh, int f, float* T, int64_t ldt, bool accumulate,
              cudaStream_t stream, int64_t nnz, const SpmmEpi* epi, const int2* colval,
              const SpmmPacked* packed) {
  spmm_segments(n_rows, row_ptr, row_ptr + 1, col_idx, vals, H, ldh, f, T, ldt, accumulate, stream,
                nnz, epi, colval, packed);
}

namespace {
__global__ void interleave_kernel(int64_t nnz, const int32_t* __restrict__ ci, const float* __restrict__ v,
                                  int2* __restrict__ out) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = make_int2(ci[k], __float_as_int(v[k]));
}

// Warp per row: the row scale, then the row's entries (lanes over nonzeros).
__global__ void pack_normalized_kernel(int64_t n_rows, const int64_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col_idx,
                                       const float* __restrict__ vals, const int32_t* __restrict__ deg,
                                       int64_t row_off, int64_t col_off, int bits,
                                       uint32_t* __restrict__ out, float* __restrict__ row_scale,
                                       unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint32_t dmax = bits >= 32 ? 0u : (0xffffffffu >> bits);
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += warps) {
    const double dr = static_cast<double>(deg[row_off + r]);
    if (lane == 0) row_scale[r] = static_cast<float>(1.0 / sqrt(dr));
    unsigned long long nbad = 0;
    for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) {
      const int32_t c = col_idx[k];
      const int32_t dc = deg[col_off + c];
      // dataset normalization (graph.cu normalize_device, csr.cpp:94-116), bitwise
      const float want = static_cast<float>(1.0 / sqrt(dr * static_cast<double>(dc)));
      const bool ok = __float_as_uint(want) == __float_as_uint(vals[k]) && dc > 0 &&
                      static_cast<uint32_t>(dc) <= dmax && (static_cast<uint32_t>(c) >> bits) == 0;
      nbad += ok ? 0 : 1;
      out[k] = (static_cast<uint32_t>(dc) << bits) | static_cast<uint32_t>(c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
    if (lane == 0 && nbad) atomicAdd(bad, nbad);
  }
}
__global__ void row_degrees_kernel(int64_t n, const int64_t* __restrict__ rp, int32_t* __restrict__ deg) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) deg[i] = static_cast<int32_t>(rp[i + 1] - rp[i]);
}
}  // namespace

void row_degrees(int64_t n, const int64_t* row_ptr, int32_t* deg, cudaStream_t s) {
  if (n <= 0) return;
  row_degrees_kernel<<<static_cast<unsigned>(ceil_div64(n, 256)), 256, 0, s>>>(n, row_ptr, deg);
  CG_LAUNCH_CHECK();
}

void pack_normalized(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                     const float* vals, const int32_t* deg, int64_t row_off, int64_t col_off,
                     int bits, uint32_t* out, float* row_scale, unsigned long long* bad,
                     cudaStream_t s) {
  if (n_rows <= 0) return;
  const int64_t want = ceil_div64(n_rows, 8);
  const unsigned g = static_cast<unsigned>(want < 16LL * 1024 ? want : 16LL * 1024);
  pack_normalized_kernel<<<g, 256, 0, s>>>(n_rows, row_ptr, col_idx, vals, deg, row_off, col_off, bits,
                                           out, row_scale, bad);
  CG_LAUNCH_CHECK();
}

void interleave_colval(int64_t nnz, const int32_t* col_idx, const float* vals, int2* out, cudaStream_t s) {
  if (nnz <= 0) return;
  const int64_t want = ceil_div64(nnz, 256);
  const unsigned g = static_cast<unsigned>(want < 16LL * 1024 ? want : 16LL * 1024);
  interleave_kernel<<<g, 256, 0, s>>>(nnz, col_idx, vals, out);
  CG_LAUNCH_CHECK();
}

void column_splits(int64_t rows, int64_t n_cols, int nb, const int64_t* row_ptr,
                   const int32_t* col_idx, int64_t* split, cudaStream_t stream) {
  if (rows <= 0) return;
  const int64_t step = ceil_div64(n_cols > 0 ? n_cols : 1, nb);
  column_splits_kernel<<<static_cast<unsigned>(ceil_div64(rows, 256)), 256, 0, stream>>>(
      rows, nb, step, row_ptr, col_idx, split);
  CG_LAUNCH_CHECK();
}

}  // namespace kern
}  // namespace cagnet
