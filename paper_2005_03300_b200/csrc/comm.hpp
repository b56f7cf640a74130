// Rank-boundary collectives on NCCL over NVLink / NVSwitch, one communicator
// per grid group (ncclCommSplit of the world communicator by group id).  This
// replaces the reference's SimRuntime rendezvous (runtime.cpp:186-228) and
// RankContext collectives (runtime.hpp:55-96).  Every call meters the same
// per-category counters as the reference ledger (runtime.cpp:142-184), so the
// traffic of a GPU run can be reconciled with the simulator's ledger word for
// word.  Singleton groups short-circuit and meter nothing, exactly like the
// reference.
#pragma once

#include <nccl.h>

#include <cstdint>
#include <map>
#include <memory>
#include <vector>

#include "comm_local.hpp"
#include "common.cuh"
#include "grid.hpp"

namespace cagnet {

enum class Category : int { DBcast = 0, SBcast = 1, Reduce = 2, AllGather = 3 };
constexpr int kNumCategories = 4;

struct CommCounter {
  uint64_t messages = 0;
  uint64_t words_sent = 0;
  uint64_t words_received = 0;
  uint64_t payload_words = 0;
  uint64_t calls = 0;
};

#define CG_NCCL(expr)                                                                     \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess)                                                                \
      throw ::cagnet::NcclError(std::string(#expr) + ": " + ncclGetErrorString(_r) + " (" + \
                                __FILE__ + ":" + std::to_string(__LINE__) + ")");        \
  } while (0)

// Two backends behind one interface: NCCL (one rank per GPU, the product
// path) and an in-process LocalWorld (all ranks as threads on one GPU;
// comm_local.hpp), chosen by the id: a LocalId selects the local backend.
// Every collective of one group must be issued from one stream per rank
// (the trainers use their comm stream), like calls on one NCCL communicator.
class Comm {
 public:
  // id may be null only when the grid has a single rank.
  Comm(const ProcessGrid& grid, int rank, const ncclUniqueId* id);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;

  int rank() const { return rank_; }

  // One-to-all broadcast of `count` elements in place at `buf` (root sends
  // from it, others receive into it).  `words` is the ledger payload.
  void bcast(const Group& g, int root_rank, void* buf, size_t count, ncclDataType_t t,
             Category cat, uint64_t words, cudaStream_t s);
  // Three-array sparse panel broadcast; ledger payload = nnz (CsrMatrix::words).
  void bcast_csr(const Group& g, int root_rank, int64_t* row_ptr, int64_t n_rows, int32_t* col,
                 float* vals, int64_t nnz, Category cat, cudaStream_t s);
  // In-place elementwise sum, every member gets the result.
  void all_reduce(const Group& g, void* buf, size_t count, ncclDataType_t t, Category cat,
                  uint64_t words, cudaStream_t s);
  // Sum then scatter equal padded slices of `slice_count` elements; slot_words
  // are the logical (unpadded) words per member for the ledger.
  void reduce_scatter(const Group& g, const void* send, void* recv, size_t slice_count,
                      ncclDataType_t t, Category cat, const std::vector<uint64_t>& slot_words,
                      cudaStream_t s);
  // Concatenate equal padded slices in ascending member order.
  void all_gather(const Group& g, const void* send, void* recv, size_t slice_count,
                  ncclDataType_t t, Category cat, const std::vector<uint64_t>& slot_words,
                  cudaStream_t s);

  // Every member broadcasts its slot of `buf` (slot q = [q * slice_count,
  // (q + 1) * slice_count) elements) to the group: ONE in-place ncclAllGather,
  // metered exactly like the reference's g.size() broadcasts with roots in
  // member order and payloads words[q] (same ledger, NVLS/ring-optimal data path).
  void bcast_all(const Group& g, void* buf, size_t slice_count, ncclDataType_t t, Category cat,
                 const std::vector<uint64_t>& words, cudaStream_t s);

  // Meters g.size() broadcasts (roots in member order, payloads words[q])
  // for data moved outside NCCL (the NVLink peer-memory panel exchange).
  void meter_bcast_all(const Group& g, Category cat, const std::vector<uint64_t>& words);

  // Fuse the collectives issued in between into one NCCL launch.
  void group_start() {
    if (ranks_ > 1 && !local_) CG_NCCL(ncclGroupStart());
  }
  void group_end() {
    if (ranks_ > 1 && !local_) CG_NCCL(ncclGroupEnd());
  }

  // In-process world (null on the NCCL backend).
  LocalWorld* local_world() const { return local_ ? &local_->world() : nullptr; }
  bool is_local() const { return local_ != nullptr; }
  // All ranks of the world (local backend; no-op on NCCL).
  // A fresh host channel id for a peer-memory exchange of the local world
  // (every rank creates its exchanges in the same order).
  int next_local_channel() { return -1000 - local_channels_++; }
  void local_barrier() {
    if (local_) local_->world().barrier(rank_);
  }
  // Raises NcclError when an asynchronous communication failure was
  // recorded: NCCL's async error (the communicators are aborted first) or a
  // timed-out device wait of the local world.
  void check_async();

  // Unmetered world all-gather for setup metadata (tile shapes).
  void setup_all_gather(const void* send, void* recv, size_t count, ncclDataType_t t,
                        cudaStream_t s);

  const CommCounter& counter(Category c) const { return counters_[static_cast<int>(c)]; }
  // Ledger arithmetic for CUDA-graph replays: the counters metered while one
  // epoch was captured are added again for every replay of that graph.
  void snapshot(CommCounter* out) const {
    for (int c = 0; c < kNumCategories; ++c) out[c] = counters_[c];
  }
  void restore(const CommCounter* in) {
    for (int c = 0; c < kNumCategories; ++c) counters_[c] = in[c];
  }
  void add_delta(const CommCounter* before, const CommCounter* after) {
    for (int c = 0; c < kNumCategories; ++c) {
      counters_[c].messages += after[c].messages - before[c].messages;
      counters_[c].words_sent += after[c].words_sent - before[c].words_sent;
      counters_[c].words_received += after[c].words_received - before[c].words_received;
      counters_[c].payload_words += after[c].payload_words - before[c].payload_words;
      counters_[c].calls += after[c].calls - before[c].calls;
    }
  }

 private:
  ncclComm_t comm_for(const Group& g) const;
  CommCounter& ctr(Category c) { return counters_[static_cast<int>(c)]; }

  int rank_ = 0;
  int ranks_ = 1;
  ncclComm_t world_ = nullptr;
  std::unique_ptr<LocalCollectives> local_;
  int local_channels_ = 0;
  std::map<int, ncclComm_t> comms_;  // group id -> communicator
  CommCounter counters_[kNumCategories];
};

}  // namespace cagnet
