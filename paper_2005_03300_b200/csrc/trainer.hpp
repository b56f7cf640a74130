// Device-resident GraphDataset and the per-rank Trainer of the four CAGNET
// partitioning strategies (dist.hpp:59-131, dist_impl.hpp, dist_{1d,15d,2d,3d}.cpp).
//
// One Trainer object is one rank: it owns its GPU tiles, its NCCL
// communicators and two streams (compute `cs`, communication `ms`).  Stage
// loops double-buffer their broadcast panels so that the NCCL broadcast of
// stage q+1 runs on `ms` while the SpMM of stage q runs on `cs`.
#pragma once

#include <nccl.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "comm.hpp"
#include "graph.cuh"
#include "grid.hpp"
#include "kernels.cuh"

namespace cagnet {

// dataset.hpp:31-45 with device-resident arrays.
struct DeviceDataset {
  int device = 0;
  int64_t n = 0, f = 0, num_classes = 0, train_count = 0;
  DeviceCsr adj, adj_t;
  DevBuf<float> features;  // n x f, ld = ldf
  int64_t ldf = 0;
  DevBuf<int32_t> labels;
  DevBuf<uint8_t> mask;
};

// generate_dataset (dataset.cpp:110-118) on the current device.
std::unique_ptr<DeviceDataset> dataset_generate(int64_t n, double degree, int64_t f,
                                                int64_t classes, uint64_t sg, uint64_t sf,
                                                uint64_t sl, int generator);
// permute_random (dataset.cpp:120-144) on the GPU: perm from the reference's
// seeded Fisher-Yates (rng.hpp:73-82) on the host, then both CSR
// orientations, features, labels and mask permuted on the device; perm_out
// (n entries) receives perm.
std::unique_ptr<DeviceDataset> dataset_permute(const DeviceDataset& d, uint64_t seed,
                                               std::vector<int64_t>* perm_out);
// load_dataset (dataset.cpp:293-307): the reference's text formats parsed
// from mapped files on all host cores, from_edge_list's sort + unique on the
// GPU (io.cu), then make_dataset on the current device.
std::unique_ptr<DeviceDataset> dataset_load(const std::string& edges_path,
                                            const std::string& features_path,
                                            const std::string& labels_path, bool undirected, int device);
// from_edge_list (csr.cpp:79-92): sort + unique of the (u, v) pairs (and the
// mirrored pairs when undirected) on the GPU; unit-valued raw CSR.
DeviceCsr csr_from_edges_device(int64_t n, int64_t m, const int64_t* u, const int64_t* v, bool undirected,
                                cudaStream_t s);
// Binary dataset cache (io.cu): a finished dataset written / mapped back.
void dataset_save(const DeviceDataset& d, const std::string& path);
std::unique_ptr<DeviceDataset> dataset_load_binary(const std::string& path, int device);
// make_dataset (dataset.cpp:76-90) from a raw unit-valued CSR already on the
// current device (load_dataset's GPU-built from_edge_list).
std::unique_ptr<DeviceDataset> dataset_make_device(DeviceCsr raw, const double* features, int64_t f,
                                                   const int64_t* labels, const uint8_t* mask,
                                                   int64_t classes);
// make_dataset (dataset.cpp:76-90) from host arrays.
std::unique_ptr<DeviceDataset> dataset_make(int64_t n, const int64_t* raw_rp,
                                            const int64_t* raw_ci, const double* features,
                                            int64_t f, const int64_t* labels,
                                            const uint8_t* mask, int64_t classes);

struct Mat {
  float* p = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
};

struct OwnedMat {
  DevBuf<float> buf;
  Mat m;
  // Zero-initialised rows x cols with ld = padded_ld(cols) unless given;
  // extra_rows adds zeroed padding rows (for equal-count NCCL slices).
  void alloc(int64_t rows, int64_t cols, int64_t ld = -1, int64_t capacity_rows = -1);
};

class Trainer {
 public:
  Trainer(const DeviceDataset& data, std::vector<int64_t> dims, const double* weights,
          double lr, Strategy strat, int rank, const ncclUniqueId* id);
  virtual ~Trainer();

  const ProcessGrid& grid() const { return grid_; }
  const Strategy& strategy() const { return strat_; }
  int rank() const { return rank_; }
  int device() const { return device_; }
  int num_layers() const { return static_cast<int>(dims_.size()); }
  const std::vector<int64_t>& dims() const { return dims_; }

  virtual void distribute() = 0;
  virtual void forward_layer(int l) = 0;  // 1-based, consumes h[l-1]
  // Trainer::run_forward_layer (dist_common.cpp:110-115): one layer outside
  // an epoch, called on every rank.  Leaves the exchange machinery at an
  // epoch boundary (see finish_external_layer), so later eager or replayed
  // epochs are unaffected.
  void run_forward_layer(int l);
  // Loss (into the device loss slot), gradients and the SGD update.
  virtual void backward_and_step() = 0;
  virtual BlockRange tile_rows(int rank) const = 0;
  virtual BlockRange tile_cols(int rank, int64_t width) const = 0;
  virtual int tile_owner(int rank) const { return rank; }

  // dist_common.cpp:97-100.  Losses stay on the device until read.  With
  // graphs on, the second and later epochs replay a CUDA graph captured from
  // one epoch (kernels, NCCL collectives, cross-stream events): one launch per
  // epoch, immune to host scheduling jitter between ranks.
  void epoch();
  void set_graph(bool on) {
    if (on != use_graph_) reset_graph();
    use_graph_ = on;
  }
  bool graph() const { return use_graph_; }
  std::vector<double> run_epochs(int epochs);
  double last_loss();
  void flush_losses();
  const std::vector<double>& all_losses() {
    flush_losses();
    return losses_host_;
  }
  // Waits for both streams, polling for asynchronous communication failures
  // (NCCL async errors, timed-out device waits) meanwhile; throws NcclError.
  void sync();
  // Raises the recorded asynchronous communication failure, if any.
  virtual void check_async() { comm_->check_async(); }

  // Readback helpers (host fp32, dense ld = cols).
  void h_tile(int layer, float* out) const;
  void g_tile(int idx, float* out) const;
  void weight(int l, float* out) const;
  void ygrad(int l, float* out) const;
  int num_parts() const { return static_cast<int>(a_parts_.size()); }
  const DeviceCsr& part(int which, int idx) const {
    return which == 0 ? a_parts_.at(static_cast<size_t>(idx)) : at_parts_.at(static_cast<size_t>(idx));
  }
  const Comm& comm() const { return *comm_; }
  Comm& comm_mut() { return *comm_; }
  // SimRuntime gauges of the last run_epochs call (runtime.cpp:287-295,
  // 450-459; only the 3D strategy notes them, dist_3d.cpp:84-87, 147-150):
  // per-note words of the pre-reduction partials in call order, and the peak
  // resident words.  Reset by every run_epochs, like the reference's run().
  const std::vector<uint64_t>& prereductions() const { return prered_; }
  uint64_t memory_peak() const { return mem_peak_; }
  cudaStream_t stream() const { return cs_; }
  float last_epoch_ms() const { return last_epoch_ms_; }

  // --- per-launch CUDA-event profile (bench roofline) ---
  struct ProfEntry {
    std::string name;
    int64_t launches = 0;
    double ms = 0, bytes = 0, flops = 0;
  };
  void set_timing(bool on) {
    if (on != timing_) reset_graph();
    timing_ = on;
  }
  // Narrow-first propagation Aᵀ(H W) when f_out < f_in (every strategy).
  void set_reassociate(bool on) {
    if (on != reassociate_) reset_graph();
    reassociate_ = on;
  }
  bool reassociate() const { return reassociate_; }
  // Fused SpMM row epilogues (block-row strategies, 1D): 0 = none,
  // 1 = elementwise (ReLU, ⊙relu′; default), 2 = also the small dense
  // transforms (T·W, S·Wᵀ) — per-row W reads compete with the gathers for
  // the L1 data pipe, so level 2 is slower on B200 and kept for comparison.
  void set_fuse(int level) {
    if (level != fuse_) reset_graph();
    fuse_ = level;
  }
  int fuse() const { return fuse_; }
  // SUMMA (2D/3D): keep the row group's sparse tiles resident after
  // distribute() instead of re-broadcasting them every SpMM stage.  Set before
  // distribute(); off reproduces the reference's per-stage SBcast ledger.
  void set_resident_sparse(bool on) { resident_sparse_ = on; }
  // 1D: exchange the stage panels through NVLink peer memory instead of an
  // NCCL all-gather (set before distribute(); falls back to NCCL when the
  // GPUs lack peer access).
  void set_p2p(bool on) { p2p_enabled_ = on; }
  // 1D peer-memory stages: SpMM the rank's own vertex block from its local
  // panel while the pushes to the peers are in flight, then the remaining
  // columns (set before distribute(); off = one SpMM after the exchange).
  void set_overlap(bool on) { overlap_enabled_ = on; }
  // 1D peer-memory stages with large slots (>= 32 MB per peer): per-destination
  // pushes and per-block SpMMs as slots land (off by default: the per-block
  // SpMM passes cost more than the transfer they hide).
  void set_pipeline(bool on) {
    if (on != pipeline_enabled_) reset_graph();
    pipeline_enabled_ = on;
  }
  void reset_profile() {
    collect_profile();
    profile_.clear();
  }
  const std::vector<ProfEntry>& profile() {
    collect_profile();
    return profile_;
  }
  // One epoch from host buffers: H2D of this rank's feature tile (rows x
  // cols, dense) and label rows, the epoch, D2H of the loss.
  double step_host(const float* x_tile, const int32_t* labels_tile);
  // Pipelined form of step_host: prefetch_host queues the H2D copies of a
  // later step's inputs on a copy stream into one of two staging slots
  // (returns at once); step_prefetched consumes the oldest staged inputs,
  // runs the epoch and returns its loss.  Step k + 1's copy then overlaps
  // step k's epoch.  At most two steps may be staged ahead.
  void prefetch_host(const float* x_tile, const int32_t* labels_tile);
  double step_prefetched();

 protected:
  void epoch_body();  // one epoch's launches (eager or under capture)
  void reset_graph();
  // Per-epoch reset of strategy-private host state so every epoch issues the
  // identical launch sequence (required for graph replay).
  virtual void begin_epoch() {}
  // After a layer run outside an epoch: strategy-private exchange state back
  // to an epoch boundary (pending direct pushes waited for, buffer rotation
  // padded) so a replayed epoch graph sees the state it was captured with.
  virtual void finish_external_layer() {}
  // --- helpers shared by the strategies ---
  void init_tiles();  // h/z/g tile shapes from tile_rows/tile_cols, labels, H0
  // End of distribute(): setup work on the legacy stream (zeroing memsets)
  // and both trainer streams complete.  Not a device-wide synchronisation:
  // ranks sharing one GPU must never wait for each other's streams.
  void settle();
  // Width the strategies' large n-proportional scratch panels must hold: the
  // widest layer, except under narrow-first propagation with a narrowing first
  // layer, where nothing f0-wide is ever propagated or swept (the f0-wide H0
  // tile is only read by the first GEMM) — Amazon {300,16,16,24}: 24, not 300.
  int64_t big_width() const;
  void ms_after_cs();
  void cs_after_ms();
  // out (+)= a · h.  With epi (f <= 32, acc = false, one pass) the layer's
  // next dense step runs in the SpMM's row epilogue (kern::SpmmEpi).
  void spmm(const DeviceCsr& a, const Mat& h, Mat out, bool acc,
            const kern::SpmmEpi* epi = nullptr);
  // out (+)= A·h over row segments [seg_b[r], seg_e[r]) of (ci, v); h.p may be
  // offset so that column index c addresses row c of the view (no shape check
  // on h.rows).  `kind` labels the profile entry.
  void spmm_seg(int64_t rows, int64_t nnz, const int64_t* seg_b, const int64_t* seg_e, const int32_t* ci,
                const float* v, const Mat& h, Mat out, bool acc, const kern::SpmmEpi* epi, const char* kind);
  // stable = false: the CSR arrays are a scratch buffer whose contents change
  // between calls (no interleaved copy is cached for them).
  // src (optional): the block these arrays belong to, for the packed stream.
  void spmm_raw(int64_t rows, int64_t nnz, const int64_t* rp, const int32_t* ci, const float* v,
                const Mat& h, Mat out, bool acc, const kern::SpmmEpi* epi = nullptr, bool stable = true,
                const DeviceCsr* src = nullptr);
  // True when spmm(a, h, ...) is a single kernel pass (no L2 column blocking).
  bool spmm_single_pass(const DeviceCsr& a, const Mat& h) const;
  int spmm_passes(const DeviceCsr& a, const Mat& h) const;
  // C (+)= A · W[r0:r0+k, c0:c0+n]
  void gemm_aw(const Mat& a, int l, int64_t r0, int64_t c0, Mat c, bool acc, int epi,
               Mat aux_out);
  // C (+)= H^T · S
  // st = nullptr: the compute stream.
  void gemm_hts(const Mat& h, const Mat& s, Mat c, bool acc, cudaStream_t st = nullptr);
  // C (+)= S · W[r0:r0+n, c0:c0+k]^T, optional relu' epilogue with aux
  void gemm_swt(const Mat& s, int l, int64_t r0, int64_t c0, Mat c, bool acc, int epi,
                const Mat* aux);
  void run_gemm(const kern::GemmDesc& d, const char* kind, cudaStream_t st = nullptr);
  void bcast_mat(const Group& g, int root, Mat m, Category cat);
  void sgd_all();
  void note_prereduction(uint64_t words) { prered_.push_back(words); }
  void note_memory_words(uint64_t words) { mem_peak_ = words > mem_peak_ ? words : mem_peak_; }
  void loss_all_reduce(double* partial_dev);
  uint64_t words(const Mat& m) const { return static_cast<uint64_t>(m.rows * m.cols); }
  // Brackets one kernel launch on cs_ with events when timing is on.
  int prof_begin();
  void prof_end(int slot, const char* kind, int64_t f, double bytes, double flops);
  void collect_profile();

  struct ProfRec {
    cudaEvent_t a = nullptr, b = nullptr;
    std::string name;
    double bytes = 0, flops = 0;
  };
  bool timing_ = false;
  bool reassociate_ = false;
  int fuse_ = 1;
  bool resident_sparse_ = true;
  bool p2p_enabled_ = true;
  bool overlap_enabled_ = false;
  bool pipeline_enabled_ = false;
  std::vector<ProfRec> recs_;
  size_t recs_used_ = 0;
  std::vector<ProfEntry> profile_;

  const DeviceDataset& data_;
  std::vector<int64_t> dims_;
  double lr_;
  Strategy strat_;
  ProcessGrid grid_;
  int rank_;
  int64_t train_total_;
  int device_;
  std::unique_ptr<Comm> comm_;
  cudaStream_t cs_ = nullptr, ms_ = nullptr;
  cudaEvent_t ev_cs_ = nullptr, ev_ms_ = nullptr, ev_t0_ = nullptr, ev_t1_ = nullptr;
  cudaEvent_t ev_ready_[2] = {nullptr, nullptr}, ev_free_[2] = {nullptr, nullptr};

  std::vector<OwnedMat> W_, Y_;  // replicated, dims[l] x dims[l+1], ld = cols
  std::vector<OwnedMat> h_, z_, g_;
  DevBuf<int32_t> labels_;
  DevBuf<uint8_t> mask_;
  std::vector<DeviceCsr> a_parts_, at_parts_;
  DevBuf<double> loss_partial_;
  DevBuf<float> stage_;  // host-input staging for step_host
  // prefetch_host / step_prefetched: two staging slots filled on xs_.
  DevBuf<float> pstage_[2];
  DevBuf<int32_t> plabels_[2];
  cudaStream_t xs_ = nullptr;
  cudaEvent_t ev_staged_[2] = {nullptr, nullptr}, ev_consumed_[2] = {nullptr, nullptr};
  int pf_head_ = 0, pf_count_ = 0;  // oldest filled slot, filled slots
  // Column blocks of the local CSR parts for L2-blocked SpMM passes, keyed by
  // (row_ptr, blocks).
  std::map<std::pair<const void*, int>, std::vector<DeviceCsr>> colblocks_;
  // Interleaved (col, value) copies of the CSR arrays the SpMMs stream, keyed
  // by the arrays they copy; built on first use outside graph capture
  // (CAGNET_SPMM_CV=0 disables them).
  std::map<std::pair<const void*, const void*>, DevBuf<int2>> colval_;
  const int2* colval(const int32_t* ci, const float* v, int64_t nnz);
  // Packed streams (kern::SpmmPacked) of blocks of the normalized adjacency,
  // keyed like colval_; a block whose values fail the check maps to an empty
  // entry (CAGNET_SPMM_PACK=0 disables them).  deg_: degrees of A + I.
  struct PackedCsr {
    DevBuf<uint32_t> e;
    DevBuf<float> row_scale;
    kern::SpmmPacked view;
  };
  std::map<std::pair<const void*, const void*>, PackedCsr> packed_;
  DevBuf<int32_t> deg_;
  // The packed stream built for these arrays, if any.  Built only in
  // distribute() (build_packed / prepare_streams): the check needs a host
  // read, and a host sync mid-epoch can deadlock ranks whose streams wait on
  // each other.
  const kern::SpmmPacked* packed(const int32_t* ci, const float* v) const;
  void build_packed(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int32_t* ci,
                    const float* v, int64_t row_off, int64_t col_off);
  // Builds the packed streams of stream_csrs() (end of distribute()).
  void prepare_streams();
  virtual std::vector<const DeviceCsr*> stream_csrs() const;
  static double l2_panel_bytes();
  DevBuf<double> losses_dev_;
  DevBuf<int> loss_slot_;  // device-side write index into losses_dev_
  bool use_graph_ = false;
  bool graph_warm_ = false;
  cudaGraphExec_t graph_exec_ = nullptr;
  uint64_t graph_kernels_ = 0;  // kernels per replay (added to the launch counter)
  CommCounter ledger_before_[kNumCategories], ledger_after_[kNumCategories];
  std::vector<uint64_t> prered_, prered_graph_;  // notes; the captured epoch's notes
  uint64_t mem_peak_ = 0;
  int epochs_done_ = 0;
  int epochs_read_ = 0;
  std::vector<double> losses_host_;
  float last_epoch_ms_ = 0.f;
};

std::unique_ptr<Trainer> make_trainer(const DeviceDataset& data, std::vector<int64_t> dims,
                                      const double* weights, double lr, Strategy strat,
                                      int rank, const ncclUniqueId* id);

}  // namespace cagnet
