/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See cagnet_oracle.h. */
#include "cagnet_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:29-82 -------------------------------------------------------- */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    r->s[i] = z ^ (z >> 31);
  }
}

uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

double orc_rng_double(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

uint64_t orc_rng_bounded(orc_rng* r, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = orc_rng_next(r);
    if (x >= threshold) return x % bound;
  }
}

void orc_rng_permutation(orc_rng* r, int64_t n, int64_t* p) {
  for (int64_t i = 0; i < n; ++i) p[i] = i;
  for (int64_t i = n; i > 1; --i) {
    const int64_t j = (int64_t)orc_rng_bounded(r, (uint64_t)i);
    const int64_t t = p[i - 1];
    p[i - 1] = p[j];
    p[j] = t;
  }
}

/* ---- dist_common.cpp:24-36 ------------------------------------------------ */
void orc_block_range(int64_t n, int parts, int idx, int64_t* begin, int64_t* end) {
  const int64_t step = n == 0 ? 0 : (n + parts - 1) / parts;
  int64_t b = (int64_t)idx * step;
  if (b > n) b = n;
  int64_t e = b + step;
  if (e > n) e = n;
  *begin = b;
  *end = e;
}

/* ---- csr.cpp:195-218 ------------------------------------------------------ */
int64_t orc_er_generate(int64_t n, double degree, uint64_t seed, int64_t* row_ptr,
                        int64_t* col_idx) {
  const double p = degree / (double)n;
  orc_rng r;
  orc_rng_seed(&r, seed);
  int64_t nnz = 0;
  row_ptr[0] = 0;
  for (int64_t u = 0; u < n; ++u) {
    for (int64_t v = 0; v < n; ++v) {
      if (u == v) continue;
      if (orc_rng_double(&r) < p) {
        if (col_idx) col_idx[nnz] = v;
        ++nnz;
      }
    }
    row_ptr[u + 1] = nnz;
  }
  return nnz;
}

/* ---- GF(2) jump-ahead of the xoshiro256** state update (rng.hpp:45-57) ---- */
/* A 256 x 256 bit matrix stored as the images of the 256 basis states. */
typedef struct { uint64_t col[256][4]; } gf2mat;

static void state_step(uint64_t* s) { /* the update of orc_rng_next without the output */
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
}

static void gf2_apply(const gf2mat* m, const uint64_t* v, uint64_t* out) {
  uint64_t r[4] = {0, 0, 0, 0};
  for (int j = 0; j < 256; ++j)
    if ((v[j >> 6] >> (j & 63)) & 1) {
      r[0] ^= m->col[j][0];
      r[1] ^= m->col[j][1];
      r[2] ^= m->col[j][2];
      r[3] ^= m->col[j][3];
    }
  memcpy(out, r, sizeof(r));
}

static gf2mat* jump_table(void) { /* T^(2^i), i = 0..63, built once */
  static gf2mat* tab = NULL;
  if (tab) return tab;
  gf2mat* t = (gf2mat*)malloc(64 * sizeof(gf2mat));
  for (int j = 0; j < 256; ++j) {
    uint64_t v[4] = {0, 0, 0, 0};
    v[j >> 6] = 1ULL << (j & 63);
    state_step(v);
    memcpy(t[0].col[j], v, sizeof(v));
  }
  for (int i = 1; i < 64; ++i)
    for (int j = 0; j < 256; ++j) gf2_apply(&t[i - 1], t[i - 1].col[j], t[i].col[j]);
  tab = t;
  return tab;
}

void orc_rng_jump(orc_rng* r, uint64_t draws) {
  const gf2mat* t = jump_table();
  for (int i = 0; i < 64; ++i)
    if ((draws >> i) & 1) gf2_apply(&t[i], r->s, r->s);
}

typedef struct {
  int64_t n, chunk_rows, nchunks;
  double p;
  uint64_t seed;
  int64_t* row_cnt;   /* n counts */
  int64_t** chunk_cols;
  int64_t* chunk_nnz;
  volatile int64_t next;
} er_job;

static void* er_worker(void* arg) {
  er_job* job = (er_job*)arg;
  for (;;) {
    const int64_t c = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
    if (c >= job->nchunks) break;
    const int64_t u0 = c * job->chunk_rows;
    int64_t u1 = u0 + job->chunk_rows;
    if (u1 > job->n) u1 = job->n;
    orc_rng r;
    orc_rng_seed(&r, job->seed);
    orc_rng_jump(&r, (uint64_t)u0 * (uint64_t)(job->n - 1));
    int64_t cap = 1024, cnt = 0;
    int64_t* cols = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
    for (int64_t u = u0; u < u1; ++u) {
      int64_t deg = 0;
      for (int64_t v = 0; v < job->n; ++v) {
        if (u == v) continue;
        if (orc_rng_double(&r) < job->p) {
          if (cnt == cap) {
            cap *= 2;
            cols = (int64_t*)realloc(cols, (size_t)cap * sizeof(int64_t));
          }
          cols[cnt++] = v;
          ++deg;
        }
      }
      job->row_cnt[u] = deg;
    }
    job->chunk_cols[c] = cols;
    job->chunk_nnz[c] = cnt;
  }
  return NULL;
}

int64_t orc_er_generate_mt(int64_t n, double degree, uint64_t seed, int threads,
                           int64_t* row_ptr, int64_t** col_idx) {
  if (n <= 0 || threads <= 0) return -1;
  er_job job;
  job.n = n;
  job.p = degree / (double)n;
  job.seed = seed;
  job.chunk_rows = n / (64 * threads) + 1;
  job.nchunks = (n + job.chunk_rows - 1) / job.chunk_rows;
  job.row_cnt = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  job.chunk_cols = (int64_t**)calloc((size_t)job.nchunks, sizeof(int64_t*));
  job.chunk_nnz = (int64_t*)calloc((size_t)job.nchunks, sizeof(int64_t));
  job.next = 0;
  jump_table();
  pthread_t* tid = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, er_worker, &job);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  row_ptr[0] = 0;
  for (int64_t u = 0; u < n; ++u) row_ptr[u + 1] = row_ptr[u] + job.row_cnt[u];
  const int64_t nnz = row_ptr[n];
  int64_t* ci = (int64_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
  int64_t off = 0;
  for (int64_t c = 0; c < job.nchunks; ++c) {
    memcpy(ci + off, job.chunk_cols[c], (size_t)job.chunk_nnz[c] * sizeof(int64_t));
    off += job.chunk_nnz[c];
    free(job.chunk_cols[c]);
  }
  free(job.chunk_cols);
  free(job.chunk_nnz);
  free(job.row_cnt);
  *col_idx = ci;
  return nnz;
}

void orc_free(void* p) { free(p); }

/* ---- csr.cpp:59-92 -------------------------------------------------------- */
typedef struct { int64_t r, c; } pair64;

static int pair_cmp(const void* a, const void* b) {
  const pair64* x = (const pair64*)a;
  const pair64* y = (const pair64*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return 0;
}

/* from_pairs: sort + unique; returns nnz. */
static int64_t from_pairs(pair64* pairs, int64_t m, int64_t n_rows, int64_t* row_ptr,
                          int64_t* col_idx) {
  qsort(pairs, (size_t)m, sizeof(pair64), pair_cmp);
  int64_t k = 0;
  for (int64_t i = 0; i < m; ++i)
    if (k == 0 || pair_cmp(&pairs[k - 1], &pairs[i]) != 0) pairs[k++] = pairs[i];
  for (int64_t i = 0; i <= n_rows; ++i) row_ptr[i] = 0;
  for (int64_t i = 0; i < k; ++i) {
    row_ptr[pairs[i].r + 1]++;
    if (col_idx) col_idx[i] = pairs[i].c;
  }
  for (int64_t i = 0; i < n_rows; ++i) row_ptr[i + 1] += row_ptr[i];
  return k;
}

int64_t orc_from_edge_list(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                           int undirected, int64_t* row_ptr, int64_t* col_idx) {
  pair64* pairs = (pair64*)malloc(sizeof(pair64) * (size_t)(2 * m + 1));
  int64_t k = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (u[i] < 0 || u[i] >= n || v[i] < 0 || v[i] >= n) {
      free(pairs);
      return -1;
    }
    pairs[k].r = u[i];
    pairs[k++].c = v[i];
    if (undirected && u[i] != v[i]) {
      pairs[k].r = v[i];
      pairs[k++].c = u[i];
    }
  }
  const int64_t nnz = from_pairs(pairs, k, n, row_ptr, col_idx);
  free(pairs);
  return nnz;
}

/* ---- csr.cpp:94-116 ------------------------------------------------------- */
int64_t orc_normalize(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                      int64_t* out_row_ptr, int64_t* out_col, double* out_vals) {
  const int64_t m = row_ptr[n] + n;
  pair64* pairs = (pair64*)malloc(sizeof(pair64) * (size_t)(m + 1));
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    pairs[k].r = i;
    pairs[k++].c = i;
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
      pairs[k].r = i;
      pairs[k++].c = col_idx[q];
    }
  }
  int64_t* cols = out_col ? out_col : (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  const int64_t nnz = from_pairs(pairs, k, n, out_row_ptr, cols);
  free(pairs);
  if (out_vals) {
    double* degree = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) degree[i] = (double)(out_row_ptr[i + 1] - out_row_ptr[i]);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t q = out_row_ptr[i]; q < out_row_ptr[i + 1]; ++q)
        out_vals[q] = 1.0 / sqrt(degree[i] * degree[cols[q]]);
    free(degree);
  }
  if (!out_col) free(cols);
  return nnz;
}

/* ---- csr.cpp:118-138 ------------------------------------------------------ */
void orc_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                   const int64_t* col_idx, const double* vals, int64_t* t_row_ptr,
                   int64_t* t_col, double* t_vals) {
  const int64_t nnz = row_ptr[n_rows];
  for (int64_t j = 0; j <= n_cols; ++j) t_row_ptr[j] = 0;
  for (int64_t k = 0; k < nnz; ++k) t_row_ptr[col_idx[k] + 1]++;
  for (int64_t j = 0; j < n_cols; ++j) t_row_ptr[j + 1] += t_row_ptr[j];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_cols + 1));
  memcpy(cursor, t_row_ptr, sizeof(int64_t) * (size_t)n_cols);
  for (int64_t i = 0; i < n_rows; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const int64_t pos = cursor[col_idx[k]]++;
      t_col[pos] = i;
      if (t_vals) t_vals[pos] = vals[k];
    }
  free(cursor);
}

/* ---- csr.cpp:140-162 ------------------------------------------------------ */
int64_t orc_extract_block(const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                          int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                          int64_t* out_row_ptr, int64_t* out_col, double* out_vals) {
  int64_t nnz = 0;
  out_row_ptr[0] = 0;
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const int64_t c = col_idx[k];
      if (c < c0 || c >= c1) continue;
      if (out_col) out_col[nnz] = c - c0;
      if (out_vals) out_vals[nnz] = vals[k];
      ++nnz;
    }
    out_row_ptr[i - r0 + 1] = nnz;
  }
  return nnz;
}

/* ---- csr.cpp:164-179 ------------------------------------------------------ */
void orc_spmm_add(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* vals, const double* h, int64_t f, double* acc) {
  for (int64_t i = 0; i < n_rows; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const double v = vals[k];
      const double* hr = h + col_idx[k] * f;
      double* ar = acc + i * f;
      for (int64_t j = 0; j < f; ++j) ar[j] += v * hr[j];
    }
}

/* ---- dense.cpp:37-61 ------------------------------------------------------ */
void orc_gemm_add(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br,
                  int64_t bc, double* acc, int ta, int tb) {
  const int64_t m = ta ? ac : ar;
  const int64_t k = ta ? ar : ac;
  const int64_t n = tb ? br : bc;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t p = 0; p < k; ++p) {
        const double av = ta ? a[p * ac + i] : a[i * ac + p];
        const double bv = tb ? b[j * bc + p] : b[p * bc + j];
        s += av * bv;
      }
      acc[i * n + j] += s;
    }
}

/* ---- dense.cpp:80-107 ----------------------------------------------------- */
void orc_relu(const double* z, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = z[i] > 0.0 ? z[i] : 0.0;
}

void orc_log_softmax_rows(const double* z, int64_t rows, int64_t cols, double* out) {
  for (int64_t i = 0; i < rows; ++i) {
    const double* zr = z + i * cols;
    double mx = zr[0];
    for (int64_t j = 1; j < cols; ++j)
      if (zr[j] > mx) mx = zr[j];
    double s = 0.0;
    for (int64_t j = 0; j < cols; ++j) s += exp(zr[j] - mx);
    const double lse = log(s);
    for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = zr[j] - mx - lse;
  }
}

/* ---- dense.cpp:109-136 ---------------------------------------------------- */
double orc_nll_tile(const double* logp, int64_t rows, int64_t cols, const int64_t* labels,
                    const uint8_t* mask, int64_t train_total, int64_t col_begin,
                    double* grad) {
  const double inv = 1.0 / (double)train_total;
  double loss = 0.0;
  memset(grad, 0, sizeof(double) * (size_t)(rows * cols));
  const int64_t col_end = col_begin + cols;
  for (int64_t i = 0; i < rows; ++i) {
    if (!mask[i]) continue;
    for (int64_t j = 0; j < cols; ++j) grad[i * cols + j] = exp(logp[i * cols + j]) * inv;
    const int64_t y = labels[i];
    if (y >= 0 && y >= col_begin && y < col_end) {
      const int64_t jl = y - col_begin;
      grad[i * cols + jl] -= inv;
      loss += -logp[i * cols + jl];
    }
  }
  return loss;
}

/* ---- dataset.cpp:92-108 --------------------------------------------------- */
void orc_random_features(int64_t n, int64_t f, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n * f; ++i) out[i] = orc_rng_double(&r);
}

void orc_random_labels(int64_t n, int64_t classes, uint64_t seed, int64_t* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = (int64_t)orc_rng_bounded(&r, (uint64_t)classes);
}

/* ---- gnn.cpp:24-44 -------------------------------------------------------- */
void orc_init_glorot(const int64_t* dims, int ndims, uint64_t seed, double* weights) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  int64_t off = 0;
  for (int l = 0; l + 1 < ndims; ++l) {
    const int64_t fin = dims[l], fout = dims[l + 1];
    const double bound = sqrt(6.0 / (double)(fin + fout));
    for (int64_t i = 0; i < fin * fout; ++i) {
      /* Rng::uniform(lo, hi) = lo + (hi - lo) * next_double()  (rng.hpp:61) */
      weights[off + i] = -bound + (bound - -bound) * orc_rng_double(&r);
    }
    off += fin * fout;
  }
}

/* ---- gnn.cpp:68-132 ------------------------------------------------------- */
int orc_train_serial(int64_t n, const int64_t* adj_rp, const int64_t* adj_ci,
                     const double* adj_v, const int64_t* adjt_rp, const int64_t* adjt_ci,
                     const double* adjt_v, const double* features, const int64_t* labels,
                     const uint8_t* mask, const int64_t* dims, int ndims, double lr,
                     int epochs, double* weights, double* losses, double* h_final,
                     double* y_out, double* g_out) {
  const int L = ndims;
  int64_t woff[64], maxf = 0;
  if (L < 2 || L > 60) return -1;
  woff[0] = 0;
  for (int l = 0; l + 1 < L; ++l) woff[l + 1] = woff[l] + dims[l] * dims[l + 1];
  for (int l = 0; l < L; ++l)
    if (dims[l] > maxf) maxf = dims[l];
  int64_t count = 0;
  for (int64_t i = 0; i < n; ++i) count += mask[i] ? 1 : 0;
  if (count == 0) return -2;

  double** h = (double**)calloc((size_t)L, sizeof(double*));
  double** z = (double**)calloc((size_t)L, sizeof(double*));
  h[0] = (double*)features;
  for (int l = 1; l < L; ++l) {
    h[l] = (double*)malloc(sizeof(double) * (size_t)(n * dims[l]));
    z[l - 1] = (double*)malloc(sizeof(double) * (size_t)(n * dims[l]));
  }
  double* t = (double*)malloc(sizeof(double) * (size_t)(n * maxf));
  double* g = (double*)malloc(sizeof(double) * (size_t)(n * maxf));
  double* gn = (double*)malloc(sizeof(double) * (size_t)(n * maxf));
  double* s = (double*)malloc(sizeof(double) * (size_t)(n * maxf));
  double* y = (double*)malloc(sizeof(double) * (size_t)woff[L - 1]);

  for (int e = 0; e < epochs; ++e) {
    /* forward_serial (gnn.cpp:68-82) */
    for (int l = 1; l < L; ++l) {
      const int64_t fin = dims[l - 1], fout = dims[l];
      memset(t, 0, sizeof(double) * (size_t)(n * fin));
      orc_spmm_add(n, adjt_rp, adjt_ci, adjt_v, h[l - 1], fin, t);
      memset(z[l - 1], 0, sizeof(double) * (size_t)(n * fout));
      orc_gemm_add(t, n, fin, weights + woff[l - 1], fin, fout, z[l - 1], 0, 0);
      if (l + 1 == L)
        orc_log_softmax_rows(z[l - 1], n, fout, h[l]);
      else
        orc_relu(z[l - 1], n * fout, h[l]);
    }
    /* backward_serial (gnn.cpp:84-104), nll_loss_and_grad (dense.cpp:138-156) */
    const int64_t C = dims[L - 1];
    const double partial = orc_nll_tile(h[L - 1], n, C, labels, mask, count, 0, g);
    const double loss = partial / (double)count;
    for (int l = L - 1; l >= 1; --l) {
      const int64_t fin = dims[l - 1], fout = dims[l];
      if (e + 1 == epochs && g_out) {
        int64_t goff = 0;
        for (int q = 1; q < l; ++q) goff += n * dims[q];
        memcpy(g_out + goff, g, sizeof(double) * (size_t)(n * fout));
      }
      memset(s, 0, sizeof(double) * (size_t)(n * fout));
      orc_spmm_add(n, adj_rp, adj_ci, adj_v, g, fout, s);
      memset(y + woff[l - 1], 0, sizeof(double) * (size_t)(fin * fout));
      orc_gemm_add(h[l - 1], n, fin, s, n, fout, y + woff[l - 1], 1, 0);
      if (l >= 2) {
        memset(gn, 0, sizeof(double) * (size_t)(n * fin));
        orc_gemm_add(s, n, fout, weights + woff[l - 1], fin, fout, gn, 0, 1);
        const double* zp = z[l - 2];
        for (int64_t i = 0; i < n * fin; ++i) gn[i] = gn[i] * (zp[i] > 0.0 ? 1.0 : 0.0);
        double* tmp = g;
        g = gn;
        gn = tmp;
      }
    }
    /* sgd_step (gnn.cpp:106-120) */
    for (int64_t i = 0; i < woff[L - 1]; ++i) weights[i] -= lr * y[i];
    if (losses) losses[e] = loss;
    if (e + 1 == epochs) {
      if (h_final) memcpy(h_final, h[L - 1], sizeof(double) * (size_t)(n * dims[L - 1]));
      if (y_out) memcpy(y_out, y, sizeof(double) * (size_t)woff[L - 1]);
    }
  }
  for (int l = 1; l < L; ++l) {
    free(h[l]);
    free(z[l - 1]);
  }
  free(h);
  free(z);
  free(t);
  free(g);
  free(gn);
  free(s);
  free(y);
  return 0;
}
