// Trainer base: tiles, weights, streams, shared GEMM/SpMM plumbing, and the
// device GraphDataset constructors.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "kernels.cuh"
#include "rng.hpp"

#include "nvtx.hpp"
#include "trainer.hpp"

namespace cagnet {

// ---- datasets ----------------------------------------------------------------
namespace {

void finish_dataset(DeviceDataset& d, const std::vector<int32_t>& labels,
                    const std::vector<uint8_t>& mask, cudaStream_t s) {
  d.labels.resize(static_cast<size_t>(d.n));
  d.mask.resize(static_cast<size_t>(d.n));
  if (d.n) {
    CG_CUDA(cudaMemcpyAsync(d.labels.get(), labels.data(), d.n * sizeof(int32_t),
                            cudaMemcpyHostToDevice, s));
    CG_CUDA(cudaMemcpyAsync(d.mask.get(), mask.data(), d.n, cudaMemcpyHostToDevice, s));
  }
  int64_t cnt = 0;
  for (int64_t i = 0; i < d.n; ++i) {
    if (!mask[static_cast<size_t>(i)]) continue;
    ++cnt;
    if (labels[static_cast<size_t>(i)] < 0 || labels[static_cast<size_t>(i)] >= d.num_classes)
      throw std::invalid_argument("GraphDataset: label " + std::to_string(labels[static_cast<size_t>(i)]) +
                                  " of training vertex " + std::to_string(i) + " outside [0, " +
                                  std::to_string(d.num_classes) + ")");
  }
  d.train_count = cnt;
  CG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

std::unique_ptr<DeviceDataset> dataset_generate(int64_t n, double degree, int64_t f,
                                                int64_t classes, uint64_t sg, uint64_t sf,
                                                uint64_t sl, int generator) {
  require(classes > 0, "random_labels: need at least one class");
  auto d = std::make_unique<DeviceDataset>();
  d->device = current_device();
  d->n = n;
  d->f = f;
  d->num_classes = classes;
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    {
      DeviceCsr raw = generator == 0 ? er_generate_device(n, degree, sg, s)
                                     : er_skip_generate_device(n, degree, sg, s);
      d->adj = normalize_device(raw, nullptr, s);
    }
    d->adj_t = transpose_device(d->adj, s);
    d->ldf = padded_ld(f);
    d->features.resize(static_cast<size_t>(n * d->ldf));
    CG_CUDA(cudaMemsetAsync(d->features.get(), 0, n * d->ldf * sizeof(float), s));
    random_features_device(n, f, sf, d->features.get(), d->ldf, s);
    std::vector<int32_t> labels = random_labels_host(n, classes, sl);
    std::vector<uint8_t> mask(static_cast<size_t>(n), 1);
    finish_dataset(*d, labels, mask, s);
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  CG_CUDA(cudaStreamDestroy(s));
  return d;
}

namespace {
// out[i, :] = in[perm[i], :] for features (ld), labels and mask.
__global__ void permute_rows_kernel(int64_t n, int64_t ldf, const int64_t* __restrict__ perm,
                                    const float* __restrict__ fin, float* __restrict__ fout,
                                    const int32_t* __restrict__ lin, int32_t* __restrict__ lout,
                                    const uint8_t* __restrict__ min, uint8_t* __restrict__ mout) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const int64_t r = perm[i];
  for (int64_t j = threadIdx.x; j < ldf; j += blockDim.x) fout[i * ldf + j] = fin[r * ldf + j];
  if (threadIdx.x == 0) {
    lout[i] = lin[r];
    mout[i] = min[r];
  }
}
}  // namespace

std::unique_ptr<DeviceDataset> dataset_permute(const DeviceDataset& d, uint64_t seed,
                                               std::vector<int64_t>* perm_out) {
  CG_CUDA(cudaSetDevice(d.device));
  const int64_t n = d.n;
  std::vector<int64_t> perm(static_cast<size_t>(n)), inv(static_cast<size_t>(n));
  {
    Xoshiro rng(seed);  // rng.hpp:73-82, Fisher-Yates
    for (int64_t i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = i;
    for (int64_t i = n; i > 1; --i) {
      const int64_t j = static_cast<int64_t>(rng.bounded(static_cast<uint64_t>(i)));
      std::swap(perm[static_cast<size_t>(i - 1)], perm[static_cast<size_t>(j)]);
    }
  }
  for (int64_t i = 0; i < n; ++i) inv[static_cast<size_t>(perm[static_cast<size_t>(i)])] = i;
  auto out = std::make_unique<DeviceDataset>();
  out->device = d.device;
  out->n = n;
  out->f = d.f;
  out->num_classes = d.num_classes;
  out->train_count = d.train_count;
  out->ldf = d.ldf;
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    DevBuf<int64_t> dp(static_cast<size_t>(std::max<int64_t>(n, 1))), di(static_cast<size_t>(std::max<int64_t>(n, 1)));
    if (n) {
      CG_CUDA(cudaMemcpyAsync(dp.get(), perm.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      CG_CUDA(cudaMemcpyAsync(di.get(), inv.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    }
    out->adj = permute_csr_device(d.adj, dp.get(), di.get(), s);
    out->adj_t = permute_csr_device(d.adj_t, dp.get(), di.get(), s);
    out->features.resize(static_cast<size_t>(std::max<int64_t>(n * d.ldf, 1)));
    out->labels.resize(static_cast<size_t>(std::max<int64_t>(n, 1)));
    out->mask.resize(static_cast<size_t>(std::max<int64_t>(n, 1)));
    if (n) {
      permute_rows_kernel<<<static_cast<unsigned>(n), 128, 0, s>>>(
          n, d.ldf, dp.get(), d.features.get(), out->features.get(), d.labels.get(), out->labels.get(),
          d.mask.get(), out->mask.get());
      CG_LAUNCH_CHECK();
    }
    CG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  CG_CUDA(cudaStreamDestroy(s));
  if (perm_out) *perm_out = std::move(perm);
  return out;
}

std::unique_ptr<DeviceDataset> dataset_make(int64_t n, const int64_t* raw_rp,
                                            const int64_t* raw_ci, const double* features,
                                            int64_t f, const int64_t* labels,
                                            const uint8_t* mask, int64_t classes) {
  // validate_csr-style checks on the raw structure (csr.cpp:25-48).
  require(raw_rp[0] == 0, "make_dataset: row_ptr must start at 0");
  for (int64_t i = 0; i < n; ++i) {
    require(raw_rp[i] <= raw_rp[i + 1], "make_dataset: row_ptr decreases at row " + std::to_string(i));
    for (int64_t k = raw_rp[i]; k < raw_rp[i + 1]; ++k) {
      require(raw_ci[k] >= 0 && raw_ci[k] < n, "make_dataset: column index out of range in row " + std::to_string(i));
      require(k == raw_rp[i] || raw_ci[k - 1] < raw_ci[k],
              "make_dataset: columns not strictly increasing in row " + std::to_string(i));
    }
  }
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  DeviceCsr raw;
  try {
    raw = upload_csr(n, n, raw_rp, raw_ci, nullptr, s);
    CG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  CG_CUDA(cudaStreamDestroy(s));
  return dataset_make_device(std::move(raw), features, f, labels, mask, classes);
}

std::unique_ptr<DeviceDataset> dataset_make_device(DeviceCsr raw, const double* features, int64_t f,
                                                   const int64_t* labels, const uint8_t* mask,
                                                   int64_t classes) {
  auto d = std::make_unique<DeviceDataset>();
  d->device = current_device();
  const int64_t n = raw.n_rows;
  d->n = n;
  d->f = f;
  d->num_classes = classes;
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    d->adj = normalize_device(raw, nullptr, s);
    { DeviceCsr drop = std::move(raw); }
    d->adj_t = transpose_device(d->adj, s);
    d->ldf = padded_ld(f);
    d->features.resize(static_cast<size_t>(n * d->ldf));
    std::vector<float> hf(static_cast<size_t>(n * d->ldf), 0.f);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < f; ++j) hf[static_cast<size_t>(i * d->ldf + j)] = static_cast<float>(features[i * f + j]);
    CG_CUDA(cudaMemcpyAsync(d->features.get(), hf.data(), hf.size() * sizeof(float),
                            cudaMemcpyHostToDevice, s));
    std::vector<int32_t> lab(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) lab[static_cast<size_t>(i)] = static_cast<int32_t>(labels[i]);
    std::vector<uint8_t> m(static_cast<size_t>(n), 1);
    if (mask) std::memcpy(m.data(), mask, static_cast<size_t>(n));
    finish_dataset(*d, lab, m, s);
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  CG_CUDA(cudaStreamDestroy(s));
  return d;
}

// ---- OwnedMat ------------------------------------------------------------------
void OwnedMat::alloc(int64_t rows, int64_t cols, int64_t ld, int64_t capacity_rows) {
  if (ld < 0) ld = padded_ld(cols);
  const int64_t cap = capacity_rows > rows ? capacity_rows : rows;
  const size_t count = static_cast<size_t>((cap > 0 ? cap : 1) * (ld > 0 ? ld : 1));
  buf.resize(count);
  // The zeroing runs on the legacy stream, which does not order against the
  // trainers' non-blocking streams: wait for it, or a lazily allocated tile
  // (the kept T of a widening layer) could be zeroed after its first writes.
  CG_CUDA(cudaMemset(buf.get(), 0, count * sizeof(float)));
  CG_CUDA(cudaStreamSynchronize(nullptr));
  m.p = buf.get();
  m.rows = rows;
  m.cols = cols;
  m.ld = ld;
}

// ---- Trainer ---------------------------------------------------------------------
Trainer::Trainer(const DeviceDataset& data, std::vector<int64_t> dims, const double* weights,
                 double lr, Strategy strat, int rank, const ncclUniqueId* id)
    : data_(data),
      dims_(std::move(dims)),
      lr_(lr),
      strat_(strat),
      grid_(ProcessGrid::make(strat)),
      rank_(rank),
      train_total_(data.train_count),
      device_(data.device) {
  require(dims_.size() >= 2, "model: need at least two layers");
  for (int64_t d : dims_) require(d > 0, "init_glorot: zero-width layer");
  require(dims_.front() == data.f, "model: input width " + std::to_string(dims_.front()) +
                                       " but dataset has " + std::to_string(data.f) + " features");
  require(dims_.back() == data.num_classes,
          "model: output width " + std::to_string(dims_.back()) + " but dataset has " +
              std::to_string(data.num_classes) + " classes");
  require(train_total_ > 0, "distributed training: empty training set");
  require(rank >= 0 && rank < grid_.ranks(), "trainer: rank outside the grid");
  CG_CUDA(cudaSetDevice(device_));
  CG_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
  comm_ = std::make_unique<Comm>(grid_, rank, id);
  // The comm stream runs at the highest priority: its NCCL / peer-push
  // kernels then get SM slots as soon as CTAs of a running SpMM retire
  // instead of queueing behind the SpMM's whole grid (measured: SUMMA stage
  // broadcasts otherwise start only after the previous stage's SpMM ends).
  // CAGNET_LOCAL_STREAMS=1 gives each rank of an in-process world a single
  // stream (device order = host issue order; a debugging aid).
  const char* ls = std::getenv("CAGNET_LOCAL_STREAMS");
  if (comm_->is_local() && ls && std::atoi(ls) == 1) {
    ms_ = cs_;
  } else {
    int lo = 0, hi = 0;
    CG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CG_CUDA(cudaStreamCreateWithPriority(&ms_, cudaStreamNonBlocking, hi));
  }
  CG_CUDA(cudaEventCreateWithFlags(&ev_cs_, cudaEventDisableTiming));
  CG_CUDA(cudaEventCreateWithFlags(&ev_ms_, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CG_CUDA(cudaEventCreateWithFlags(&ev_ready_[i], cudaEventDisableTiming));
    CG_CUDA(cudaEventCreateWithFlags(&ev_free_[i], cudaEventDisableTiming));
  }
  CG_CUDA(cudaEventCreate(&ev_t0_));
  CG_CUDA(cudaEventCreate(&ev_t1_));

  const int L = num_layers();
  W_.resize(static_cast<size_t>(L - 1));
  Y_.resize(static_cast<size_t>(L - 1));
  int64_t off = 0;
  const int side = grid_.kind() == GridKind::Grid2D || grid_.kind() == GridKind::Grid3D ? grid_.rows() : 1;
  for (int l = 0; l + 1 < L; ++l) {
    const int64_t r = dims_[static_cast<size_t>(l)], c = dims_[static_cast<size_t>(l + 1)];
    W_[static_cast<size_t>(l)].alloc(r, c, c);
    // Y gets the padded slot rows of the 2D/3D row all-gather.
    Y_[static_cast<size_t>(l)].alloc(r, c, c, side * ceil_div64(r, side));
    std::vector<float> wf(static_cast<size_t>(r * c));
    for (int64_t e = 0; e < r * c; ++e) wf[static_cast<size_t>(e)] = static_cast<float>(weights[off + e]);
    CG_CUDA(cudaMemcpy(W_[static_cast<size_t>(l)].m.p, wf.data(), wf.size() * sizeof(float),
                       cudaMemcpyHostToDevice));
    off += r * c;
  }
  loss_partial_.resize(1);
  CG_CUDA(cudaMemset(loss_partial_.get(), 0, sizeof(double)));
  losses_dev_.resize(4096);
  loss_slot_.resize(1);
  CG_CUDA(cudaMemset(loss_slot_.get(), 0, sizeof(int)));
  CG_CUDA(cudaStreamSynchronize(nullptr));  // legacy-stream zeroing before the trainer's streams run
}

Trainer::~Trainer() {
  cudaSetDevice(device_);
  if (xs_) {
    cudaStreamSynchronize(xs_);
    cudaStreamDestroy(xs_);
    for (cudaEvent_t e : {ev_staged_[0], ev_staged_[1], ev_consumed_[0], ev_consumed_[1]})
      if (e) cudaEventDestroy(e);
  }
  if (cs_) cudaStreamSynchronize(cs_);
  if (ms_ && ms_ != cs_) cudaStreamSynchronize(ms_);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  comm_.reset();
  for (cudaEvent_t e : {ev_cs_, ev_ms_, ev_t0_, ev_t1_, ev_ready_[0], ev_ready_[1], ev_free_[0], ev_free_[1]})
    if (e) cudaEventDestroy(e);
  if (ms_ && ms_ != cs_) cudaStreamDestroy(ms_);
  if (cs_) cudaStreamDestroy(cs_);
}

const int2* Trainer::colval(const int32_t* ci, const float* v, int64_t nnz) {
  static const bool on = [] {
    const char* e = std::getenv("CAGNET_SPMM_CV");
    return !(e && e[0] == '0');
  }();
  if (!on || nnz <= 0 || ci == nullptr || v == nullptr) return nullptr;
  const auto key = std::make_pair(static_cast<const void*>(ci), static_cast<const void*>(v));
  auto it = colval_.find(key);
  if (it != colval_.end()) return it->second.get();
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CG_CUDA(cudaStreamIsCapturing(cs_, &st));
  if (st != cudaStreamCaptureStatusNone) return nullptr;  // no allocation inside a capture
  DevBuf<int2> buf(static_cast<size_t>(nnz));
  kern::interleave_colval(nnz, ci, v, buf.get(), cs_);
  return colval_.emplace(key, std::move(buf)).first->second.get();
}

std::vector<const DeviceCsr*> Trainer::stream_csrs() const {
  std::vector<const DeviceCsr*> v;
  for (const DeviceCsr& c : a_parts_) v.push_back(&c);
  for (const DeviceCsr& c : at_parts_) v.push_back(&c);
  return v;
}

void Trainer::prepare_streams() {
  for (const DeviceCsr* c : stream_csrs())
    build_packed(c->n_rows, c->n_cols, c->nnz, c->row_ptr.get(), c->col_idx.get(), c->vals.get(), c->row_off,
                 c->col_off);
}

const kern::SpmmPacked* Trainer::packed(const int32_t* ci, const float* v) const {
  auto it = packed_.find(std::make_pair(static_cast<const void*>(ci), static_cast<const void*>(v)));
  return it != packed_.end() && it->second.view.e ? &it->second.view : nullptr;
}

void Trainer::build_packed(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int32_t* ci,
                           const float* v, int64_t row_off, int64_t col_off) {
  static const bool on = [] {
    const char* e = std::getenv("CAGNET_SPMM_PACK");
    return !(e && e[0] == '0');
  }();
  if (!on || nnz <= 0 || rows <= 0) return;
  const auto key = std::make_pair(static_cast<const void*>(ci), static_cast<const void*>(v));
  if (packed_.count(key)) return;
  const int64_t n = data_.adj.n_rows;
  PackedCsr pc;
  // Column bits for the block's local columns; the degree takes the rest.
  int bits = 1;
  while (bits < 31 && (int64_t{1} << bits) < cols) ++bits;
  const bool fits = row_off >= 0 && col_off >= 0 && row_off + rows <= n && col_off + cols <= n && bits <= 28;
  if (fits) {
    if (!deg_.get()) {
      deg_.resize(static_cast<size_t>(n));
      kern::row_degrees(n, data_.adj.row_ptr.get(), deg_.get(), cs_);
    }
    pc.e.resize(static_cast<size_t>(nnz));
    pc.row_scale.resize(static_cast<size_t>(rows));
    DevBuf<unsigned long long> bad(1);
    CG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned long long), cs_));
    kern::pack_normalized(rows, rp, ci, v, deg_.get(), row_off, col_off, bits, pc.e.get(), pc.row_scale.get(),
                          bad.get(), cs_);
    unsigned long long nbad = 0;
    CG_CUDA(cudaMemcpyAsync(&nbad, bad.get(), sizeof(nbad), cudaMemcpyDeviceToHost, cs_));
    CG_CUDA(cudaStreamSynchronize(cs_));
    if (nbad == 0) pc.view = kern::SpmmPacked{pc.e.get(), pc.row_scale.get(), bits};
  }
  if (!pc.view.e) pc = PackedCsr{};  // not a normalized block: keep the int2 stream
  packed_.emplace(key, std::move(pc));
}

void Trainer::init_tiles() {
  colval_.clear();
  packed_.clear();
  colblocks_.clear();  // keyed by row_ptr addresses, which a new distribute() may reuse
  const int L = num_layers();
  const BlockRange rows = tile_rows(rank_);
  h_.clear();
  z_.clear();
  g_.clear();
  h_.resize(static_cast<size_t>(L));
  z_.resize(static_cast<size_t>(L - 1));
  g_.resize(static_cast<size_t>(L - 1));
  for (int l = 0; l < L; ++l) {
    const BlockRange cols = tile_cols(rank_, dims_[static_cast<size_t>(l)]);
    h_[static_cast<size_t>(l)].alloc(rows.size(), cols.size());
    if (l > 0) {
      z_[static_cast<size_t>(l - 1)].alloc(rows.size(), cols.size());
      g_[static_cast<size_t>(l - 1)].alloc(rows.size(), cols.size());
    }
  }
  const BlockRange fc = tile_cols(rank_, data_.f);
  kern::copy2d(h_[0].m.p, h_[0].m.ld, data_.features.get() + rows.begin * data_.ldf + fc.begin,
               data_.ldf, rows.size(), fc.size(), cs_);
  labels_.resize(static_cast<size_t>(rows.size()));
  mask_.resize(static_cast<size_t>(rows.size()));
  if (rows.size()) {
    CG_CUDA(cudaMemcpyAsync(labels_.get(), data_.labels.get() + rows.begin,
                            rows.size() * sizeof(int32_t), cudaMemcpyDeviceToDevice, cs_));
    CG_CUDA(cudaMemcpyAsync(mask_.get(), data_.mask.get() + rows.begin, rows.size(),
                            cudaMemcpyDeviceToDevice, cs_));
  }
}

void Trainer::ms_after_cs() {
  CG_CUDA(cudaEventRecord(ev_cs_, cs_));
  CG_CUDA(cudaStreamWaitEvent(ms_, ev_cs_, 0));
}
void Trainer::cs_after_ms() {
  CG_CUDA(cudaEventRecord(ev_ms_, ms_));
  CG_CUDA(cudaStreamWaitEvent(cs_, ev_ms_, 0));
}

bool Trainer::spmm_single_pass(const DeviceCsr& a, const Mat& h) const {
  return spmm_passes(a, h) <= 1;
}

// L2-aware column blocking (SURVEY §7 hard parts).  One pass per column block
// keeps the gathered H slice L2-resident, but every pass re-reads the row
// segments and read-modify-writes the n_rows x f output, so it only pays when
// rows carry many nonzeros per pass.  Measured on B200 (scripts/tune_spmm_big.py):
// Amazon-shaped (17 nnz/row, 912 MB panel) is fastest unblocked (5.6 ms vs
// 17 ms in 12 passes); Protein-shaped (150 nnz/row, 560 MB) at ~47 MB panels
// (15.6 ms vs 24.6 ms unblocked) — the effective L2 capacity for random 64 B
// gathers is about half the nominal 126 MB.
int Trainer::spmm_passes(const DeviceCsr& a, const Mat& h) const {
  if (a.nnz == 0 || a.n_rows == 0) return 1;
  const double panel = static_cast<double>(a.n_cols) * h.cols * 4.0;
  const double per_row = static_cast<double>(a.nnz) / static_cast<double>(a.n_rows);
  int nb = static_cast<int>(std::min<double>(64.0, std::ceil(panel / l2_panel_bytes())));
  // Keep >= 12 nonzeros per row per pass; below ~64 per row blocking loses.
  if (per_row < 64.0) return 1;
  nb = std::min<int>(nb, static_cast<int>(per_row / 12.0));
  return nb < 1 ? 1 : nb;
}

void Trainer::spmm(const DeviceCsr& a, const Mat& h, Mat out, bool acc, const kern::SpmmEpi* epi) {
  if (a.n_cols != h.rows)
    throw std::invalid_argument("spmm: sparse is " + std::to_string(a.n_rows) + "x" +
                                std::to_string(a.n_cols) + " but dense has " +
                                std::to_string(h.rows) + " rows");
  // L2-aware column blocking: when the gathered panel H (n_cols x f) does not
  // fit the L2 budget, run one pass per column block so every pass gathers
  // from an L2-resident slice (SURVEY §7 hard parts).
  const int nb = spmm_passes(a, h);
  if (epi) {
    if (nb > 1) throw std::logic_error("spmm: fused epilogue needs one pass");
    spmm_raw(a.n_rows, a.nnz, a.row_ptr.get(), a.col_idx.get(), a.vals.get(), h, out, acc, epi, true, &a);
    return;
  }
  if (nb <= 1 || a.nnz == 0 || out.rows != a.n_rows || out.cols != h.cols) {
    spmm_raw(a.n_rows, a.nnz, a.row_ptr.get(), a.col_idx.get(), a.vals.get(), h, out, acc, nullptr, true, &a);
    return;
  }
  // Column blocks materialised once per (matrix, pass count) as contiguous
  // CSR copies: each pass then streams its own nonzeros (row segments of the
  // full CSR would be ~50 B scattered DRAM reads per row and pass).
  auto key = std::make_pair(static_cast<const void*>(a.row_ptr.get()), nb);
  auto it = colblocks_.find(key);
  if (it == colblocks_.end()) {
    std::vector<DeviceCsr> blocks;
    for (int b = 0; b < nb; ++b) {
      const BlockRange cr = block_range(a.n_cols, nb, b);
      blocks.push_back(extract_block_device(a, 0, a.n_rows, cr.begin, cr.end, cs_));
    }
    it = colblocks_.emplace(key, std::move(blocks)).first;
  }
  std::vector<const int2*> cvs;
  std::vector<const kern::SpmmPacked*> pks;
  for (int b = 0; b < nb; ++b) {
    const DeviceCsr& blk = it->second[static_cast<size_t>(b)];
    pks.push_back(packed(blk.col_idx.get(), blk.vals.get()));
    cvs.push_back(pks.back() ? nullptr : colval(blk.col_idx.get(), blk.vals.get(), blk.nnz));
  }
  const int slot = prof_begin();
  for (int b = 0; b < nb; ++b) {
    const DeviceCsr& blk = it->second[static_cast<size_t>(b)];
    const BlockRange cr = block_range(a.n_cols, nb, b);
    kern::spmm_csr(blk.n_rows, blk.row_ptr.get(), blk.col_idx.get(), blk.vals.get(), h.p + cr.begin * h.ld,
                   h.ld, static_cast<int>(h.cols), out.p, out.ld, acc || b > 0, cs_, blk.nnz, nullptr,
                   cvs[static_cast<size_t>(b)], pks[static_cast<size_t>(b)]);
  }
  if (slot >= 0) {
    const double f = static_cast<double>(h.cols), r = static_cast<double>(a.n_rows);
    const double bytes = 8.0 * (r + 1) + 8.0 * a.nnz + 4.0 * f * h.rows + 4.0 * f * r * (acc ? 2 : 1);
    prof_end(slot, "spmm", h.cols, bytes, 2.0 * a.nnz * f);
  }
}

double Trainer::l2_panel_bytes() {
  // Read per call (a getenv per SpMM dispatch): tests force the multi-pass path.
  const char* e = std::getenv("CAGNET_L2_PANEL_MB");
  const double v = (e ? std::atof(e) : 48.0) * 1048576.0;
  return v > 0 ? v : 1e30;
}

void Trainer::spmm_raw(int64_t rows, int64_t nnz, const int64_t* rp, const int32_t* ci,
                       const float* v, const Mat& h, Mat out, bool acc, const kern::SpmmEpi* epi,
                       bool stable, const DeviceCsr* src) {
  const int64_t width = epi && epi->W ? epi->fo : h.cols;
  if (out.rows != rows || out.cols != width)
    throw std::invalid_argument("spmm: accumulator shape mismatch");
  // nnz here is the length of the (0-based) arrays, so the interleaved copy covers every row.
  (void)src;
  const kern::SpmmPacked* pk = stable ? packed(ci, v) : nullptr;
  const int2* cv = stable && !pk ? colval(ci, v, nnz) : nullptr;
  const int slot = prof_begin();
  kern::spmm_csr(rows, rp, ci, v, h.p, h.ld, static_cast<int>(h.cols), out.p, out.ld, acc, cs_, nnz,
                 epi, cv, pk);
  if (slot >= 0) {
    // B = 8(r+1) + 8 nnz + 4 f c + 4 f r (1 + acc); F = 2 nnz f;
    // plus the fused epilogue's extra row traffic (raw copy, relu′ mask, relu).
    const double f = static_cast<double>(h.cols), r = static_cast<double>(rows);
    double bytes = 8.0 * (r + 1) + 8.0 * nnz + 4.0 * f * h.rows + 4.0 * f * r * (acc ? 2 : 1);
    if (epi) {
      const double fo = static_cast<double>(width);
      bytes += 4.0 * r * (fo - f) + (epi->raw_out ? 4.0 * r * f : 0.0) +
               (epi->mask ? 4.0 * r * fo : 0.0) + (epi->relu_out ? 4.0 * r * fo : 0.0);
    }
    prof_end(slot, "spmm", h.cols, bytes, 2.0 * nnz * f + (epi && epi->W ? 2.0 * r * f * width : 0.0));
  }
}

void Trainer::spmm_seg(int64_t rows, int64_t nnz, const int64_t* seg_b, const int64_t* seg_e,
                       const int32_t* ci, const float* v, const Mat& h, Mat out, bool acc,
                       const kern::SpmmEpi* epi, const char* kind) {
  if (out.rows != rows || out.cols != h.cols) throw std::invalid_argument("spmm: accumulator shape mismatch");
  const int slot = prof_begin();
  kern::spmm_segments(rows, seg_b, seg_e, ci, v, h.p, h.ld, static_cast<int>(h.cols), out.p, out.ld, acc, cs_,
                      nnz, epi);
  if (slot >= 0) {
    const double f = static_cast<double>(h.cols), r = static_cast<double>(rows);
    double bytes = 16.0 * r + 8.0 * nnz + 4.0 * f * h.rows + 4.0 * f * r * (acc ? 2 : 1);
    if (epi) bytes += (epi->mask ? 4.0 * r * f : 0.0) + (epi->relu_out ? 4.0 * r * f : 0.0);
    prof_end(slot, kind, h.cols, bytes, 2.0 * nnz * f);
  }
}

int Trainer::prof_begin() {
  if (!timing_) return -1;
  if (recs_used_ == recs_.size()) {
    ProfRec r;
    CG_CUDA(cudaEventCreate(&r.a));
    CG_CUDA(cudaEventCreate(&r.b));
    recs_.push_back(r);
  }
  const int slot = static_cast<int>(recs_used_++);
  CG_CUDA(cudaEventRecord(recs_[static_cast<size_t>(slot)].a, cs_));
  return slot;
}

void Trainer::prof_end(int slot, const char* kind, int64_t f, double bytes, double flops) {
  ProfRec& r = recs_[static_cast<size_t>(slot)];
  CG_CUDA(cudaEventRecord(r.b, cs_));
  r.name = std::string(kind) + "_f" + std::to_string(f);
  r.bytes = bytes;
  r.flops = flops;
}

void Trainer::collect_profile() {
  if (recs_used_ == 0) return;
  CG_CUDA(cudaSetDevice(device_));
  CG_CUDA(cudaStreamSynchronize(cs_));
  for (size_t i = 0; i < recs_used_; ++i) {
    float ms = 0.f;
    CG_CUDA(cudaEventElapsedTime(&ms, recs_[i].a, recs_[i].b));
    ProfEntry* e = nullptr;
    for (auto& p : profile_)
      if (p.name == recs_[i].name) e = &p;
    if (!e) {
      profile_.push_back(ProfEntry{recs_[i].name});
      e = &profile_.back();
    }
    e->launches += 1;
    e->ms += ms;
    e->bytes += recs_[i].bytes;
    e->flops += recs_[i].flops;
  }
  recs_used_ = 0;
}

double Trainer::step_host(const float* x_tile, const int32_t* labels_tile) {
  CG_CUDA(cudaSetDevice(device_));
  const Mat& h0 = h_.at(0).m;
  if (h0.rows && h0.cols) {
    // One contiguous DMA (pitched 2D copies run row by row), then re-pitch on the GPU.
    stage_.resize(static_cast<size_t>(h0.rows * h0.cols));
    CG_CUDA(cudaMemcpyAsync(stage_.get(), x_tile, h0.rows * h0.cols * sizeof(float),
                            cudaMemcpyHostToDevice, cs_));
    kern::copy2d(h0.p, h0.ld, stage_.get(), h0.cols, h0.rows, h0.cols, cs_);
  }
  if (h0.rows)
    CG_CUDA(cudaMemcpyAsync(labels_.get(), labels_tile, h0.rows * sizeof(int32_t),
                            cudaMemcpyHostToDevice, cs_));
  epoch();
  std::vector<double> l = run_epochs(0);
  return losses_host_.empty() ? 0.0 : losses_host_.back();
}

void Trainer::prefetch_host(const float* x_tile, const int32_t* labels_tile) {
  CG_CUDA(cudaSetDevice(device_));
  if (pf_count_ >= 2) throw std::logic_error("prefetch_host: two steps are already staged");
  if (!xs_) {
    CG_CUDA(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CG_CUDA(cudaEventCreateWithFlags(&ev_staged_[i], cudaEventDisableTiming));
      CG_CUDA(cudaEventCreateWithFlags(&ev_consumed_[i], cudaEventDisableTiming));
      CG_CUDA(cudaEventRecord(ev_consumed_[i], cs_));
    }
  }
  const int b = (pf_head_ + pf_count_) % 2;
  const Mat& h0 = h_.at(0).m;
  pstage_[b].resize(static_cast<size_t>(h0.rows * h0.cols > 0 ? h0.rows * h0.cols : 1));
  plabels_[b].resize(static_cast<size_t>(h0.rows > 0 ? h0.rows : 1));
  // The slot is free once the step that last consumed it re-pitched it.
  CG_CUDA(cudaStreamWaitEvent(xs_, ev_consumed_[b], 0));
  if (h0.rows && h0.cols)
    CG_CUDA(cudaMemcpyAsync(pstage_[b].get(), x_tile, h0.rows * h0.cols * sizeof(float), cudaMemcpyHostToDevice, xs_));
  if (h0.rows)
    CG_CUDA(cudaMemcpyAsync(plabels_[b].get(), labels_tile, h0.rows * sizeof(int32_t), cudaMemcpyHostToDevice, xs_));
  CG_CUDA(cudaEventRecord(ev_staged_[b], xs_));
  ++pf_count_;
}

double Trainer::step_prefetched() {
  CG_CUDA(cudaSetDevice(device_));
  if (pf_count_ == 0) throw std::logic_error("step_prefetched: no staged inputs (call prefetch_host first)");
  const int b = pf_head_;
  const Mat& h0 = h_.at(0).m;
  CG_CUDA(cudaStreamWaitEvent(cs_, ev_staged_[b], 0));
  if (h0.rows && h0.cols) kern::copy2d(h0.p, h0.ld, pstage_[b].get(), h0.cols, h0.rows, h0.cols, cs_);
  if (h0.rows) kern::copy_bytes(labels_.get(), plabels_[b].get(), h0.rows * sizeof(int32_t), cs_);
  CG_CUDA(cudaEventRecord(ev_consumed_[b], cs_));
  pf_head_ = (pf_head_ + 1) % 2;
  --pf_count_;
  epoch();
  run_epochs(0);
  return losses_host_.empty() ? 0.0 : losses_host_.back();
}

void Trainer::gemm_aw(const Mat& a, int l, int64_t r0, int64_t c0, Mat c, bool acc, int epi,
                      Mat aux_out) {
  const Mat& w = W_[static_cast<size_t>(l)].m;
  kern::GemmDesc d;
  d.m = a.rows;
  d.n = c.cols;
  d.k = a.cols;
  d.A = a.p;
  d.a_sm = a.ld;
  d.a_sk = 1;
  d.B = w.p + r0 * w.ld + c0;
  d.b_sk = w.ld;
  d.b_sn = 1;
  d.C = c.p;
  d.ldc = c.ld;
  d.accumulate = acc;
  d.epilogue = epi;
  d.aux_out = aux_out.p;
  d.ldao = aux_out.ld;
  run_gemm(d, "gemm_tw");
}

void Trainer::run_gemm(const kern::GemmDesc& d, const char* kind, cudaStream_t st) {
  // Profiled (timing) epochs keep every GEMM on the compute stream, where the
  // per-launch events are recorded.
  if (timing_ || st == nullptr) st = cs_;
  const int slot = prof_begin();
  kern::gemm_tf32x3(d, st);
  if (slot >= 0) {
    // 4 (m k + k n + m n) algorithmic bytes, 2 m n k flops.
    const double m = static_cast<double>(d.m), n = static_cast<double>(d.n), k = static_cast<double>(d.k);
    // Named by the feature width of the streamed operand: f_in for T·W / S·Wᵀ,
    // the width of H for Hᵀ·S (whose K is the graph dimension).
    const bool hts = std::string(kind) == "gemm_hts";
    prof_end(slot, kind, hts ? d.m : d.k, 4.0 * (m * k + k * n + m * n * (d.accumulate ? 2 : 1)) +
                                  (d.epilogue == kern::EPI_RELU ? 4.0 * m * n : 0.0) +
                                  (d.epilogue == kern::EPI_RELU_PRIME ? 4.0 * m * n : 0.0),
             2.0 * m * n * k);
  }
}

void Trainer::gemm_hts(const Mat& h, const Mat& s, Mat c, bool acc, cudaStream_t st) {
  kern::GemmDesc d;
  d.m = h.cols;
  d.n = s.cols;
  d.k = h.rows;
  d.A = h.p;
  d.a_sm = 1;
  d.a_sk = h.ld;
  d.B = s.p;
  d.b_sk = s.ld;
  d.b_sn = 1;
  d.C = c.p;
  d.ldc = c.ld;
  d.accumulate = acc;
  run_gemm(d, "gemm_hts", st);
}

void Trainer::gemm_swt(const Mat& s, int l, int64_t r0, int64_t c0, Mat c, bool acc, int epi,
                       const Mat* aux) {
  const Mat& w = W_[static_cast<size_t>(l)].m;
  kern::GemmDesc d;
  d.m = s.rows;
  d.n = c.cols;
  d.k = s.cols;
  d.A = s.p;
  d.a_sm = s.ld;
  d.a_sk = 1;
  d.B = w.p + r0 * w.ld + c0;
  d.b_sk = 1;
  d.b_sn = w.ld;
  d.C = c.p;
  d.ldc = c.ld;
  d.accumulate = acc;
  d.epilogue = epi;
  if (aux) {
    d.aux = aux->p;
    d.ldaux = aux->ld;
  }
  run_gemm(d, "gemm_swt");
}

void Trainer::bcast_mat(const Group& g, int root, Mat m, Category cat) {
  comm_->bcast(g, root, m.p, static_cast<size_t>(m.rows * m.ld), ncclFloat32, cat, words(m), ms_);
}

void Trainer::sgd_all() {
  for (size_t l = 0; l < W_.size(); ++l)
    kern::sgd(W_[l].m.p, Y_[l].m.p, W_[l].m.rows * W_[l].m.cols, static_cast<float>(lr_), cs_);
}

void Trainer::loss_all_reduce(double* partial_dev) {
  // Off the critical path: the loss is reduced and appended on the comm
  // stream while the backward pass runs (joined at the end of the epoch).
  ms_after_cs();
  comm_->all_reduce(grid_.world(), partial_dev, 1, ncclFloat64, Category::Reduce, 1, ms_);
  kern::push_loss(losses_dev_.get(), loss_slot_.get(), partial_dev, ms_);
  ++epochs_done_;
}

void Trainer::run_forward_layer(int l) {
  CG_CUDA(cudaSetDevice(device_));
  forward_layer(l);
  finish_external_layer();
  cs_after_ms();
}

void Trainer::epoch_body() {
  begin_epoch();
  static const char* const kLayerNames[] = {"forward_layer 1", "forward_layer 2", "forward_layer 3",
                                            "forward_layer 4", "forward_layer 5", "forward_layer"};
  for (int l = 1; l < num_layers(); ++l) {
    NvtxRange r(kLayerNames[l <= 5 ? l - 1 : 5]);
    forward_layer(l);
  }
  {
    NvtxRange r("backward_and_step");
    backward_and_step();
  }
  cs_after_ms();  // join the comm stream (graph capture needs every fork joined)
}

void Trainer::reset_graph() {
  if (graph_exec_) {
    CG_CUDA(cudaSetDevice(device_));
    CG_CUDA(cudaStreamSynchronize(cs_));
    CG_CUDA(cudaGraphExecDestroy(graph_exec_));
    graph_exec_ = nullptr;
  }
  graph_warm_ = false;
}

void Trainer::epoch() {
  CG_CUDA(cudaSetDevice(device_));
  if (epochs_done_ - epochs_read_ >= static_cast<int>(losses_dev_.count)) flush_losses();
  // Per-kernel timing events stay eager (collect_profile reads every launch).
  if (!use_graph_ || timing_ || !graph_warm_) {
    NvtxRange r("epoch (eager)");
    // Eager.  The first graph-mode epoch is eager too: lazy allocations
    // (split tables, workspaces) and kernel attributes happen outside capture.
    CG_CUDA(cudaEventRecord(ev_t0_, cs_));
    epoch_body();
    CG_CUDA(cudaEventRecord(ev_t1_, cs_));
    if (use_graph_ && !timing_) graph_warm_ = true;
    return;
  }
  NvtxRange r(graph_exec_ ? "epoch (graph replay)" : "epoch (capture + replay)");
  if (!graph_exec_) {
    const size_t notes0 = prered_.size();
    comm_->snapshot(ledger_before_);
    const uint64_t k0 = launch_counter().load();
    CG_CUDA(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeRelaxed));
    try {
      epoch_body();
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(cs_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    CG_CUDA(cudaStreamEndCapture(cs_, &g));
    // Per-node priorities: kernels captured from the high-priority comm stream
    // (NCCL, peer pushes) keep their priority inside the replayed graph.
    CG_CUDA(cudaGraphInstantiate(&graph_exec_, g, cudaGraphInstantiateFlagUseNodePriority));
    CG_CUDA(cudaGraphDestroy(g));
    // In-process world: every rank instantiates before any replays, so a
    // replayed wait never targets a peer still inside its capture.
    comm_->local_barrier();
    comm_->snapshot(ledger_after_);  // the capture metered this epoch once
    prered_graph_.assign(prered_.begin() + static_cast<std::ptrdiff_t>(notes0), prered_.end());
    graph_kernels_ = launch_counter().load() - k0;
  } else {
    comm_->add_delta(ledger_before_, ledger_after_);
    prered_.insert(prered_.end(), prered_graph_.begin(), prered_graph_.end());
    launch_counter().fetch_add(graph_kernels_);  // the replay runs the captured kernels
    ++epochs_done_;
  }
  CG_CUDA(cudaEventRecord(ev_t0_, cs_));
  CG_CUDA(cudaGraphLaunch(graph_exec_, cs_));
  CG_CUDA(cudaEventRecord(ev_t1_, cs_));
}

void Trainer::flush_losses() {
  sync();
  const int pending = epochs_done_ - epochs_read_;
  std::vector<double> tot(static_cast<size_t>(pending));
  if (pending) {
    CG_CUDA(cudaMemcpy(tot.data(), losses_dev_.get(), pending * sizeof(double), cudaMemcpyDeviceToHost));
    // On the compute stream: later pushes (comm stream, behind an event on
    // it) must see the reset.
    CG_CUDA(cudaMemsetAsync(loss_slot_.get(), 0, sizeof(int), cs_));
  }
  for (double t : tot) losses_host_.push_back(t / static_cast<double>(train_total_));
  epochs_read_ = epochs_done_;
}

std::vector<double> Trainer::run_epochs(int epochs) {
  if (epochs < 0) throw std::invalid_argument("run_epochs: epoch count must be positive");
  const size_t first = losses_host_.size() + static_cast<size_t>(epochs_done_ - epochs_read_);
  if (epochs > 0) {  // gauges reset per run (runtime.cpp:235-240)
    prered_.clear();
    mem_peak_ = 0;
  }
  for (int e = 0; e < epochs; ++e) epoch();
  flush_losses();
  if (epochs > 0) CG_CUDA(cudaEventElapsedTime(&last_epoch_ms_, ev_t0_, ev_t1_));
  return std::vector<double>(losses_host_.begin() + static_cast<std::ptrdiff_t>(first), losses_host_.end());
}

double Trainer::last_loss() {
  flush_losses();
  return losses_host_.empty() ? 0.0 : losses_host_.back();
}

int64_t Trainer::big_width() const {
  int64_t maxf = 0, rest = 0;
  for (size_t i = 0; i < dims_.size(); ++i) {
    maxf = std::max(maxf, dims_[i]);
    if (i > 0) rest = std::max(rest, dims_[i]);
  }
  return (reassociate_ && dims_.size() >= 2 && dims_[0] > dims_[1]) ? rest : maxf;
}

void Trainer::settle() {
  CG_CUDA(cudaStreamSynchronize(nullptr));
  sync();
}

void Trainer::sync() {
  CG_CUDA(cudaSetDevice(device_));
  const cudaStream_t streams[2] = {ms_, ms_ == cs_ ? nullptr : cs_};
  for (cudaStream_t s : streams) {
    if (!s) continue;  // one stream per rank (in-process world)
    // Poll instead of blocking: a failed peer surfaces as an NCCL async
    // error or a recorded wait timeout, not as a hang.
    int spins = 0;
    for (;;) {
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) break;
      if (e != cudaErrorNotReady) CG_CUDA(e);
      // Busy-poll the first ~thousand queries (short epochs), then back off.
      if (++spins % 1024 == 0) check_async();
      if (spins > 1024) std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
  }
  check_async();
}

namespace {
void download(const Mat& m, float* out) {
  if (m.rows == 0 || m.cols == 0) return;
  CG_CUDA(cudaMemcpy2D(out, m.cols * sizeof(float), m.p, m.ld * sizeof(float), m.cols * sizeof(float),
                       m.rows, cudaMemcpyDeviceToHost));
}
}  // namespace

void Trainer::h_tile(int layer, float* out) const { download(h_.at(static_cast<size_t>(layer)).m, out); }
void Trainer::g_tile(int idx, float* out) const { download(g_.at(static_cast<size_t>(idx)).m, out); }
void Trainer::weight(int l, float* out) const { download(W_.at(static_cast<size_t>(l)).m, out); }
void Trainer::ygrad(int l, float* out) const { download(Y_.at(static_cast<size_t>(l)).m, out); }

}  // namespace cagnet
