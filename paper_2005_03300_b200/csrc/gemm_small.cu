// K2d — CUDA-core kernels for the GCN's narrow x narrow contractions (gemm_add,
// dense.cpp:37-70), the shapes the tensor-core kernels serve worst:
//   U = H·W, S·Wᵀ with K, N <= 32   (every hidden layer of a 16-wide GCN)
//   Y = Hᵀ·S      with M, N <= 32   (the weight gradient of those layers)
// Each is one pass over tall n x 16 operands — ~64 B per row in, ~64 B out, or
// 128 B per row reduced into a 16 x 16 tile — so HBM, not FLOPs, bounds them
// (AI ~ 2 flop/B).  The tcgen05 kernels pay a whole k-block pipeline per 2 KB
// of operand here (Amazon: 1.8 GB Hᵀ·S at 1.2 TB/s, Protein at 0.25 TB/s);
// these stream at HBM rate instead.  Plain fp32 FMA, k ascending per output
// element (the reference's order), so they are at least as accurate as the
// split-TF32 path.  Hᵀ·S reduces rows in fixed contiguous per-warp chunks, then
// warps in order, then blocks in order: deterministic.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cagnet {
namespace kern {
namespace {

constexpr int kRowThreads = 128;
constexpr int kTnThreads = 256;
constexpr int kTnWarps = kTnThreads / 32;

__device__ __forceinline__ float epi_value(const GemmDesc& d, int64_t r, int64_t c, float v) {
  if (d.accumulate) v += d.C[r * d.ldc + c];
  if (d.epilogue == EPI_RELU) {
    if (d.aux_out) d.aux_out[r * d.ldao + c] = v > 0.f ? v : 0.f;
  } else if (d.epilogue == EPI_RELU_PRIME) {
    v = d.aux[r * d.ldaux + c] > 0.f ? v : v * 0.f;
  }
  return v;
}

// Row teams of LV lanes: every lane of a team loads the whole A row (the
// team's lanes hit the same 16 B vectors, so a warp instruction moves 32/LV
// rows), lane q computes output columns [4q + 4 LV g, +4) for the NG column
// groups g from B kept in shared memory and stores each as one float4: a warp
// writes 32/LV whole row segments per instruction.  R rows per team per
// iteration keep several independent row loads in flight.
template <int LV, int KMAX, int NG, int R, bool VEC>
__global__ void __launch_bounds__(kRowThreads) gemm_rows_small_kernel(const GemmDesc d) {
  constexpr int NW = 4 * LV * NG;
  __shared__ __align__(16) float Bs[KMAX][NW];
  const int k = static_cast<int>(d.k), n = static_cast<int>(d.n);
  for (int e = threadIdx.x; e < KMAX * NW; e += blockDim.x) {
    const int kk = e / NW, j = e % NW;
    Bs[kk][j] = (kk < k && j < n) ? d.B[kk * d.b_sk + j * d.b_sn] : 0.f;
  }
  __syncthreads();
  const int q = threadIdx.x % LV;
  // Whole-vector stores (and epilogue operands) when every row segment is 16 B aligned.
  const bool cvec_ok = ((d.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(d.C) & 15) == 0) &&
                       (d.epilogue != EPI_RELU || !d.aux_out ||
                        (((d.ldao & 3) == 0) && ((reinterpret_cast<uintptr_t>(d.aux_out) & 15) == 0))) &&
                       (d.epilogue != EPI_RELU_PRIME ||
                        (((d.ldaux & 3) == 0) && ((reinterpret_cast<uintptr_t>(d.aux) & 15) == 0)));
  const int64_t teams = static_cast<int64_t>(gridDim.x) * (blockDim.x / LV);
  const int64_t team = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / LV;
  for (int64_t rbase = team * R; rbase < d.m; rbase += teams * R) {
    float a[R][KMAX];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t r = rbase + u;
      const float* ar = d.A + (r < d.m ? r : 0) * d.a_sm;
      if constexpr (VEC) {
        // 16 B-aligned rows with ld >= round4(k): whole vectors, junk past k zeroed.
#pragma unroll
        for (int v4 = 0; v4 < KMAX / 4; ++v4) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (4 * v4 < k) v = __ldg(reinterpret_cast<const float4*>(ar) + v4);
          a[u][4 * v4 + 0] = 4 * v4 + 0 < k ? v.x : 0.f;
          a[u][4 * v4 + 1] = 4 * v4 + 1 < k ? v.y : 0.f;
          a[u][4 * v4 + 2] = 4 * v4 + 2 < k ? v.z : 0.f;
          a[u][4 * v4 + 3] = 4 * v4 + 3 < k ? v.w : 0.f;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk) a[u][kk] = kk < k ? __ldg(ar + kk * d.a_sk) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t r = rbase + u;
      if (r >= d.m) break;
      float* cr = d.C + r * d.ldc;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const int c0 = 4 * q + 4 * LV * g;
        if (c0 >= n) break;
        float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk) {
          const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][c0]);
          c.x = fmaf(a[u][kk], b.x, c.x);
          c.y = fmaf(a[u][kk], b.y, c.y);
          c.z = fmaf(a[u][kk], b.z, c.z);
          c.w = fmaf(a[u][kk], b.w, c.w);
        }
        if (cvec_ok && c0 + 4 <= n) {
          if (d.accumulate) {
            const float4 o = *reinterpret_cast<const float4*>(cr + c0);
            c.x += o.x;
            c.y += o.y;
            c.z += o.z;
            c.w += o.w;
          }
          if (d.epilogue == EPI_RELU && d.aux_out) {
            *reinterpret_cast<float4*>(d.aux_out + r * d.ldao + c0) =
                make_float4(fmaxf(c.x, 0.f), fmaxf(c.y, 0.f), fmaxf(c.z, 0.f), fmaxf(c.w, 0.f));
          } else if (d.epilogue == EPI_RELU_PRIME) {
            const float4 z = __ldg(reinterpret_cast<const float4*>(d.aux + r * d.ldaux + c0));
            c.x = z.x > 0.f ? c.x : c.x * 0.f;
            c.y = z.y > 0.f ? c.y : c.y * 0.f;
            c.z = z.z > 0.f ? c.z : c.z * 0.f;
            c.w = z.w > 0.f ? c.w : c.w * 0.f;
          }
          *reinterpret_cast<float4*>(cr + c0) = c;
        } else {
          const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (c0 + t < n) cr[c0 + t] = epi_value(d, r, c0 + t, cv[t]);
        }
      }
    }
  }
}

// k <= 16, n <= 16, 16 B-aligned rows: a quad of lanes per row, every lane
// loading ONE float4 of its row (a warp instruction moves 8 whole rows, 512
// contiguous bytes) instead of the team-wide whole-row broadcast loads above,
// which cost one L1 wavefront per row per vector (LSU-bound at 98 %).  Lane q
// multiplies its k-slice [4q, 4q + 4) by B's matching rows (slices in shared
// memory at bank offsets 8q, conflict-free) into 16 partial outputs, then a
// two-round butterfly reduce-scatter (xor 2: keep 8 columns, xor 1: keep 4)
// leaves lane q with columns [4q, 4q + 4) summed over the row, stored as one
// float4.  Sum order: slices in fixed butterfly order (deterministic).
constexpr int kQuadSlice = 72;  // floats per k-slice of B (64 + 8 bank shift)
template <int R>
__global__ void __launch_bounds__(kRowThreads) gemm_rows_quad_kernel(const GemmDesc d) {
  __shared__ __align__(16) float Bs[4 * kQuadSlice];
  const int k = static_cast<int>(d.k), n = static_cast<int>(d.n);
  for (int e = threadIdx.x; e < 4 * kQuadSlice; e += blockDim.x) {
    const int q = e / kQuadSlice, w = e % kQuadSlice, i = w / 16, j = w % 16;
    const int kk = 4 * q + i;
    Bs[e] = (w < 64 && kk < k && j < n) ? d.B[kk * d.b_sk + j * d.b_sn] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, q = lane & 3;
  const float* bq = Bs + q * kQuadSlice;
  const bool live_k = 4 * q < k;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kRowThreads / 32);
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kRowThreads + threadIdx.x) >> 5;
  for (int64_t base = warp * 8 * R; base < d.m; base += warps * 8 * R) {
    float4 a[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t r = base + u * 8 + (lane >> 2);
      a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < d.m && live_k) a[u] = __ldg(reinterpret_cast<const float4*>(d.A + r * d.a_sm) + q);
      // junk past k inside the last vector contributes nothing
      if (4 * q + 1 >= k) a[u].y = 0.f;
      if (4 * q + 2 >= k) a[u].z = 0.f;
      if (4 * q + 3 >= k) a[u].w = 0.f;
      if (4 * q >= k) a[u].x = 0.f;
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      float p[16];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 b0 = *reinterpret_cast<const float4*>(bq + 0 * 16 + 4 * j4);
        const float4 b1 = *reinterpret_cast<const float4*>(bq + 1 * 16 + 4 * j4);
        const float4 b2 = *reinterpret_cast<const float4*>(bq + 2 * 16 + 4 * j4);
        const float4 b3 = *reinterpret_cast<const float4*>(bq + 3 * 16 + 4 * j4);
        p[4 * j4 + 0] = fmaf(a[u].w, b3.x, fmaf(a[u].z, b2.x, fmaf(a[u].y, b1.x, a[u].x * b0.x)));
        p[4 * j4 + 1] = fmaf(a[u].w, b3.y, fmaf(a[u].z, b2.y, fmaf(a[u].y, b1.y, a[u].x * b0.y)));
        p[4 * j4 + 2] = fmaf(a[u].w, b3.z, fmaf(a[u].z, b2.z, fmaf(a[u].y, b1.z, a[u].x * b0.z)));
        p[4 * j4 + 3] = fmaf(a[u].w, b3.w, fmaf(a[u].z, b2.w, fmaf(a[u].y, b1.w, a[u].x * b0.w)));
      }
      // xor 2: lane keeps columns [8 (q >> 1), +8)
      const bool hi = (q >> 1) != 0;
      float h[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float send = hi ? p[t] : p[8 + t];
        const float keep = hi ? p[8 + t] : p[t];
        h[t] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      // xor 1: lane keeps columns [4q, 4q + 4)
      const bool odd = (q & 1) != 0;
      float c[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float send = odd ? h[t] : h[4 + t];
        const float keep = odd ? h[4 + t] : h[t];
        c[t] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      const int64_t r = base + u * 8 + (lane >> 2);
      const int c0 = 4 * q;
      if (r >= d.m || c0 >= n) continue;
      float4 v = make_float4(c[0], c[1], c[2], c[3]);
      float* cr = d.C + r * d.ldc + c0;
      if (d.accumulate) {
        const float4 o = *reinterpret_cast<const float4*>(cr);
        v.x += o.x;
        v.y += o.y;
        v.z += o.z;
        v.w += o.w;
      }
      if (d.epilogue == EPI_RELU && d.aux_out) {
        *reinterpret_cast<float4*>(d.aux_out + r * d.ldao + c0) =
            make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
      } else if (d.epilogue == EPI_RELU_PRIME) {
        const float4 z = __ldg(reinterpret_cast<const float4*>(d.aux + r * d.ldaux + c0));
        v.x = z.x > 0.f ? v.x : v.x * 0.f;
        v.y = z.y > 0.f ? v.y : v.y * 0.f;
        v.z = z.z > 0.f ? v.z : v.z * 0.f;
        v.w = z.w > 0.f ? v.w : v.w * 0.f;
      }
      if (c0 + 4 <= n) {
        *reinterpret_cast<float4*>(cr) = v;
      } else {
        const float cv[4] = {v.x, v.y, v.z, v.w};
        for (int t = 0; t < n - c0; ++t) cr[t] = cv[t];
      }
    }
  }
}

template <int LV, int NG, int R>
void launch_rows(const GemmDesc& d, bool vec, unsigned blocks, cudaStream_t s) {
  if (d.k <= 16) {
    if (vec) gemm_rows_small_kernel<LV, 16, NG, R, true><<<blocks, kRowThreads, 0, s>>>(d);
    else gemm_rows_small_kernel<LV, 16, NG, R, false><<<blocks, kRowThreads, 0, s>>>(d);
  } else {
    if (vec) gemm_rows_small_kernel<LV, 32, NG, R, true><<<blocks, kRowThreads, 0, s>>>(d);
    else gemm_rows_small_kernel<LV, 32, NG, R, false><<<blocks, kRowThreads, 0, s>>>(d);
  }
}

// Y[m x n] = sum_r A[r, 0:m]ᵀ B[r, 0:n] (A row r at A + r a_sk with a_sm = 1,
// B row r at B + r b_sk with b_sn = 1).  Lane = (group g, column j): NT lanes
// per group cover the columns, the 32 / NT groups split the m rows of Y into
// MI-row slices held in registers.  Each warp reduces one contiguous chunk of
// graph rows; the CTA folds its warps in order into partial[blockIdx].
template <int NT, int MI>
__global__ void __launch_bounds__(kTnThreads) gemm_tn_small_kernel(const GemmDesc d, int64_t rows_per_warp,
                                                                   float* __restrict__ partial) {
  __shared__ float red[kTnWarps][32 * MI];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = lane % NT, g = lane / NT, i0 = g * MI;
  const int m = static_cast<int>(d.m), n = static_cast<int>(d.n);
  const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * kTnWarps + warp) * rows_per_warp;
  const int64_t r1 = r0 + rows_per_warp < d.k ? r0 + rows_per_warp : d.k;
  float acc[MI];
#pragma unroll
  for (int ii = 0; ii < MI; ++ii) acc[ii] = 0.f;
  const bool jok = j < n;
  int64_t r = r0;
  constexpr int U = 4;
  for (; r + U <= r1; r += U) {
    float s[U], h[U][MI];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float* hr = d.A + (r + u) * d.a_sk;
      s[u] = jok ? __ldg(d.B + (r + u) * d.b_sk + j) : 0.f;
#pragma unroll
      for (int ii = 0; ii < MI; ++ii) h[u][ii] = i0 + ii < m ? __ldg(hr + i0 + ii) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ii = 0; ii < MI; ++ii) acc[ii] = fmaf(h[u][ii], s[u], acc[ii]);
  }
  for (; r < r1; ++r) {
    const float* hr = d.A + r * d.a_sk;
    const float s = jok ? __ldg(d.B + r * d.b_sk + j) : 0.f;
#pragma unroll
    for (int ii = 0; ii < MI; ++ii) acc[ii] = fmaf(i0 + ii < m ? __ldg(hr + i0 + ii) : 0.f, s, acc[ii]);
  }
#pragma unroll
  for (int ii = 0; ii < MI; ++ii) red[warp][ii * 32 + lane] = acc[ii];
  __syncthreads();
  // Output element (i, j) lives at red[w][(i - i0(g)) * 32 + g * NT + j].
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e / n, jj = e % n;
    const int gg = i / MI, ii = i % MI;
    float v = 0.f;
    for (int w = 0; w < kTnWarps; ++w) v += red[w][ii * 32 + gg * NT + jj];
    partial[static_cast<int64_t>(blockIdx.x) * m * n + e] = v;
  }
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}

// Staged variant for 16 B-aligned rows: the CTA streams tiles of kTile graph
// rows of H (MP float4s per row) and S (NP float4s) into shared memory with
// cp.async, double-buffered, so ~2 tiles per CTA are in flight; warp w folds
// rows [32w, 32w + 32) of every tile, lanes as in gemm_tn_small_kernel.
constexpr int kTile = 256;
template <int NT, int MI, int MP, int NP>
__global__ void __launch_bounds__(kTnThreads) gemm_tn_staged_kernel(const GemmDesc d, int64_t rows_per_block,
                                                                    float* __restrict__ partial, int mp, int np) {
  extern __shared__ __align__(16) float4 stage[];  // [2][kTile][MP + NP]
  __shared__ float red[kTnWarps][32 * MI];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = lane % NT, g = lane / NT, i0 = g * MI;
  const int m = static_cast<int>(d.m), n = static_cast<int>(d.n);
  const int64_t rb = static_cast<int64_t>(blockIdx.x) * rows_per_block;
  const int64_t re = rb + rows_per_block < d.k ? rb + rows_per_block : d.k;
  const int64_t tiles = re > rb ? (re - rb + kTile - 1) / kTile : 0;
  constexpr int W4 = MP + NP;
  auto load = [&](int64_t t) {
    float4* buf = stage + (t & 1) * kTile * W4;
    const int64_t r0 = rb + t * kTile;
    // Only the mp (np) vectors that exist in a row are copied; the rest of the
    // slot feeds accumulators of rows / columns past m (n) that are never stored.
    const int w = mp + np;
    for (int e = threadIdx.x; e < kTile * w; e += kTnThreads) {
      const int rr = e / w, v = e % w;
      const int64_t r = r0 + rr;
      if (r < re) {
        if (v < mp)
          cp16(buf + rr * W4 + v, d.A + r * d.a_sk + 4 * v);
        else
          cp16(buf + rr * W4 + MP + (v - mp), d.B + r * d.b_sk + 4 * (v - mp));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  float acc[MI];
#pragma unroll
  for (int ii = 0; ii < MI; ++ii) acc[ii] = 0.f;
  if (tiles > 0) load(0);
  for (int64_t t = 0; t < tiles; ++t) {
    if (t + 1 < tiles) {
      load(t + 1);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();
    const float4* buf = stage + (t & 1) * kTile * W4;
    const int64_t r0 = rb + t * kTile;
    const int rows = static_cast<int>(re - r0 < kTile ? re - r0 : kTile);
    const int rlo = warp * 32, rhi = rlo + 32 < rows ? rlo + 32 : rows;
    for (int rr = rlo; rr < rhi; ++rr) {
      const float* hrow = reinterpret_cast<const float*>(buf + rr * W4);
      const float sv = reinterpret_cast<const float*>(buf + rr * W4 + MP)[j];
#pragma unroll
      for (int ii = 0; ii < MI; ii += 4) {
        if (i0 + ii < 4 * MP) {
          const float4 h = *reinterpret_cast<const float4*>(hrow + i0 + ii);
          acc[ii + 0] = fmaf(h.x, sv, acc[ii + 0]);
          acc[ii + 1] = fmaf(h.y, sv, acc[ii + 1]);
          acc[ii + 2] = fmaf(h.z, sv, acc[ii + 2]);
          acc[ii + 3] = fmaf(h.w, sv, acc[ii + 3]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int ii = 0; ii < MI; ++ii) red[warp][ii * 32 + lane] = acc[ii];
  __syncthreads();
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e / n, jj = e % n;
    const int gg = i / MI, ii = i % MI;
    float v = 0.f;
    for (int w = 0; w < kTnWarps; ++w) v += red[w][ii * 32 + gg * NT + jj];
    partial[static_cast<int64_t>(blockIdx.x) * m * n + e] = v;
  }
}

__global__ void gemm_tn_fold_kernel(const GemmDesc d, const float* __restrict__ partial, int blocks) {
  const int m = static_cast<int>(d.m), n = static_cast<int>(d.n);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int b = 0; b < blocks; ++b) v += partial[static_cast<int64_t>(b) * m * n + e];
    const int i = e / n, jj = e % n;
    d.C[static_cast<int64_t>(i) * d.ldc + jj] = epi_value(d, i, jj, v);
  }
}

template <int NT>
void launch_tn_mi(int mi, const GemmDesc& d, int blocks, int64_t rpw, float* part, cudaStream_t s) {
  switch (mi) {
    case 4: gemm_tn_small_kernel<NT, 4><<<blocks, kTnThreads, 0, s>>>(d, rpw, part); break;
    case 8: gemm_tn_small_kernel<NT, 8><<<blocks, kTnThreads, 0, s>>>(d, rpw, part); break;
    case 16: gemm_tn_small_kernel<NT, 16><<<blocks, kTnThreads, 0, s>>>(d, rpw, part); break;
    default: gemm_tn_small_kernel<NT, 32><<<blocks, kTnThreads, 0, s>>>(d, rpw, part); break;
  }
}

bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }

// Rows from which the quad kernel beats the tcgen05 path (CAGNET_GEMM_QUAD_MIN).
int64_t quad_min_rows() {
  static const int64_t v = [] {
    const char* e = std::getenv("CAGNET_GEMM_QUAD_MIN");  // Reddit (233 K rows): S·Wᵀ 30 -> 22 us
    return e ? std::atoll(e) : 100000LL;
  }();
  return v;
}

// CAGNET_GEMM_QUAD=0 keeps the row-team kernel for k, n <= 16 (comparison).
bool quad_enabled() {
  const char* e = std::getenv("CAGNET_GEMM_QUAD");
  return !(e && e[0] == '0');
}

// CAGNET_GEMM_SMALL=0 routes these shapes back to the tensor-core kernels.
bool small_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CAGNET_GEMM_SMALL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

// Below ~1 M rows (Reddit: 233 K) the tensor-core kernels' fixed costs are
// already small and they win (measured: Reddit Hᵀ·S 16x16 45 us vs 67 us).
// CAGNET_GEMM_SMALL_MIN overrides (tests use it to reach these kernels).
int64_t min_rows() {
  static const int64_t v = [] {
    const char* e = std::getenv("CAGNET_GEMM_SMALL_MIN");
    return e ? std::atoll(e) : 1000000LL;
  }();
  return v;
}

bool gemm_small_try(const GemmDesc& d, cudaStream_t s) {
  const int64_t kMinRows = min_rows();
  if (!small_enabled() || d.k <= 0) return false;
  const int sms = num_sms(current_device());
  const bool vec = d.a_sk == 1 && d.a_sm % 4 == 0 && aligned16(d.A) && d.a_sm >= ((d.k + 3) / 4) * 4;
  const bool cvec = d.ldc % 4 == 0 && aligned16(d.C) &&
                    (d.epilogue != EPI_RELU || !d.aux_out || (d.ldao % 4 == 0 && aligned16(d.aux_out))) &&
                    (d.epilogue != EPI_RELU_PRIME || (d.ldaux % 4 == 0 && aligned16(d.aux)));
  const bool quad = vec && cvec && d.k <= 16 && d.n <= 16 && quad_enabled();
  if (d.k <= 32 && d.n <= 256 && (d.m >= kMinRows || (quad && d.m >= quad_min_rows()))) {
    if (quad) {
      static const int R = [] {
        const char* e = std::getenv("CAGNET_GEMM_QUAD_R");  // rows in flight per lane (measured: 4 best)
        return e ? std::atoi(e) : 4;
      }();
      const int64_t want = ceil_div64(ceil_div64(d.m, 8 * R), kRowThreads / 32);
      const unsigned blocks = static_cast<unsigned>(want < 16LL * sms ? want : 16LL * sms);
      if (R >= 4)
        gemm_rows_quad_kernel<4><<<blocks, kRowThreads, 0, s>>>(d);
      else if (R == 1)
        gemm_rows_quad_kernel<1><<<blocks, kRowThreads, 0, s>>>(d);
      else
        gemm_rows_quad_kernel<2><<<blocks, kRowThreads, 0, s>>>(d);
      CG_LAUNCH_CHECK();
      return true;
    }
    const int lv = d.n <= 16 ? 4 : 8;
    const int ng = d.n <= 32 ? 1 : d.n <= 64 ? 2 : d.n <= 128 ? 4 : 8;
    const int r = ng == 1 ? 2 : 1;
    const int64_t want = ceil_div64(ceil_div64(d.m, r) * lv, kRowThreads);
    const unsigned blocks = static_cast<unsigned>(want < 32LL * sms ? want : 32LL * sms);
    if (lv == 4) launch_rows<4, 1, 2>(d, vec, blocks, s);
    else if (ng == 1) launch_rows<8, 1, 2>(d, vec, blocks, s);
    else if (ng == 2) launch_rows<8, 2, 1>(d, vec, blocks, s);
    else if (ng == 4) launch_rows<8, 4, 1>(d, vec, blocks, s);
    else launch_rows<8, 8, 1>(d, vec, blocks, s);
    CG_LAUNCH_CHECK();
    return true;
  }
  if (d.m <= 32 && d.n <= 32 && d.k >= kMinRows && d.a_sm == 1 && d.b_sn == 1) {
    const int nt = d.n <= 4 ? 4 : d.n <= 8 ? 8 : d.n <= 16 ? 16 : 32;
    const int groups = 32 / nt;
    const int64_t per = ceil_div64(d.m, groups);
    const int mi = per <= 4 ? 4 : per <= 8 ? 8 : per <= 16 ? 16 : 32;
    if (static_cast<int64_t>(mi) * groups < d.m) return false;
    int blocks = 2 * sms;
    const int64_t min_rows = 256;  // rows per warp at least
    const int64_t cap = ceil_div64(d.k, min_rows * kTnWarps);
    if (blocks > cap) blocks = static_cast<int>(cap < 1 ? 1 : cap);
    const int64_t rpw = ceil_div64(d.k, static_cast<int64_t>(blocks) * kTnWarps);
    float* part = nullptr;
    // Staged path: 16 B-aligned rows whose padded widths stay inside ld.
    const int mp = static_cast<int>((d.m + 3) / 4), np = static_cast<int>((d.n + 3) / 4);
    const bool staged = aligned16(d.A) && aligned16(d.B) && d.a_sk % 4 == 0 && d.b_sk % 4 == 0 &&
                        d.a_sk >= 4 * mp && d.b_sk >= 4 * np && mi % 4 == 0 &&
                        ((mp <= 4 && np <= 4) || (mp <= 8 && np <= 8));
    if (staged) {
      const bool narrow = mp <= 4 && np <= 4;
      const int w4 = narrow ? 8 : 16;
      const size_t smem = 2ull * kTile * w4 * sizeof(float4);
      int sblocks = (narrow ? 3 : 1) * sms;
      const int64_t scap = ceil_div64(d.k, 4LL * kTile);
      if (sblocks > scap) sblocks = static_cast<int>(scap < 1 ? 1 : scap);
      const int64_t rpb = ceil_div64(d.k, sblocks);
      part = static_cast<float*>(stream_scratch(s, static_cast<size_t>(sblocks) * d.m * d.n * sizeof(float)));
      auto go = [&](auto kern) {
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<sblocks, kTnThreads, smem, s>>>(d, rpb, part, mp, np);
      };
      if (narrow) {
        if (nt == 4 && mi == 4) go(gemm_tn_staged_kernel<4, 4, 4, 4>);
        else if (nt == 4) go(gemm_tn_staged_kernel<4, 8, 4, 4>);       // m <= 16 -> mi <= 4 with 8 groups
        else if (nt == 8 && mi == 4) go(gemm_tn_staged_kernel<8, 4, 4, 4>);
        else if (nt == 8) go(gemm_tn_staged_kernel<8, 8, 4, 4>);
        else if (mi == 4) go(gemm_tn_staged_kernel<16, 4, 4, 4>);
        else if (mi == 8) go(gemm_tn_staged_kernel<16, 8, 4, 4>);
        else go(gemm_tn_staged_kernel<16, 16, 4, 4>);
      } else {
        if (nt <= 8 && mi <= 8) go(gemm_tn_staged_kernel<8, 8, 8, 8>);
        else if (nt <= 16 && mi <= 16) go(gemm_tn_staged_kernel<16, 16, 8, 8>);
        else go(gemm_tn_staged_kernel<32, 32, 8, 8>);
      }
      CG_LAUNCH_CHECK();
      gemm_tn_fold_kernel<<<static_cast<unsigned>(ceil_div64(d.m * d.n, 256)), 256, 0, s>>>(d, part, sblocks);
      CG_LAUNCH_CHECK();
      return true;
    }
    part = static_cast<float*>(stream_scratch(s, static_cast<size_t>(blocks) * d.m * d.n * sizeof(float)));
    switch (nt) {
      case 4: launch_tn_mi<4>(mi, d, blocks, rpw, part, s); break;
      case 8: launch_tn_mi<8>(mi, d, blocks, rpw, part, s); break;
      case 16: launch_tn_mi<16>(mi, d, blocks, rpw, part, s); break;
      default: launch_tn_mi<32>(mi, d, blocks, rpw, part, s); break;
    }
    CG_LAUNCH_CHECK();
    gemm_tn_fold_kernel<<<static_cast<unsigned>(ceil_div64(d.m * d.n, 256)), 256, 0, s>>>(d, part, blocks);
    CG_LAUNCH_CHECK();
    return true;
  }
  return false;
}

}  // namespace kern
}  // namespace cagnet
