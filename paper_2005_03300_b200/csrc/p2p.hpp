// NVLink peer-memory panel exchange for the 1D propagation stages.
//
// The 1D strategy's stage broadcasts (dist_1d.cpp:46-56: every rank roots the
// panel of its vertex block) are an all-gather of an n x f panel whose f is
// 16 after narrow-first reassociation: ~15 MB for Reddit, which NCCL moves in
// ~58 us on 4 B200s (busbw ~200 GB/s at this size, measured by
// scripts/nccl_micro.py).  Here every rank instead *pushes* its own panel
// rows straight into every peer's panel buffer over NVLink (CUDA IPC mapped
// peer memory, one copy kernel writing P slots), then raises a per-peer
// ready flag in the peer's memory; consumers spin on their local flags before
// the SpMM.  Flags carry a device-side stage sequence number, so the exchange
// works unchanged inside a replayed CUDA graph.
//
// (Three buffers rotate because a producer SpMM may push the next exchange's
// panel directly — strategy_rows.cu, "direct push".)
// Buffer reuse needs no "consumed" flags: buffers rotate and every
// rank waits for all peers' ready flags at every stage, on the stream that
// also runs its SpMMs, and publishes stage s only after that stream passed
// its wait for stage s-1.  A peer's ready(s-1) is raised only after the
// peer's SpMM of stage s-2 — the last reader of the buffer that stage s
// overwrites — has finished (stream order on the peer), so when a rank
// publishes stage s nobody still reads that buffer.
//
// All waits are bounded (~20 s of spinning): a broken peer makes the wait
// record itself in a host-mapped error word and return instead of hanging
// the GPU or trapping the context; check() turns the record into an
// NcclError (CAGNET_ENCCL) at the trainer's next synchronisation.
//
// With an in-process LocalWorld (all ranks on one GPU, comm_local.hpp) the
// same kernels and flags run unchanged; each publish additionally posts a
// host-side "issued" count and each wait first waits for the peers' posts,
// so a device wait only ever targets already-issued work.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "comm.hpp"
#include "common.cuh"

namespace cagnet {

class PeerPanels {
 public:
  PeerPanels() = default;
  ~PeerPanels();
  PeerPanels(const PeerPanels&) = delete;
  PeerPanels& operator=(const PeerPanels&) = delete;

  // Collective over the world communicator: allocates 2 x `bytes` of panel
  // buffer plus flags on this rank, exchanges IPC handles (or raw pointers
  // when all ranks share a process) and maps every peer's buffers.  Returns
  // false (nothing allocated) when some pair of GPUs lacks peer access; the
  // caller then keeps the NCCL path.  Every rank must call it.
  bool init(Comm& comm, int rank, int ranks, int device, size_t bytes, cudaStream_t s);
  bool ready() const { return ranks_ > 1 && base_[0] != nullptr; }

  // Panel buffers rotate over consecutive exchanges; three, so a producer
  // kernel can push stage s's panel while peers still read stage s-1's and
  // may be finishing stage s-2's (see strategy_rows.cu).
  static constexpr int kBuffers = 3;
  // Buffer b of this rank: P slots of slot_floats each.
  float* buffer(int b) const { return base_[b]; }
  // Device array of the P ranks' buffer b (for kernels that push directly).
  float* const* device_buffers(int b) const { return d_bufs_[b].get(); }
  // Raises this stage's ready flag on every peer without copying: the panel
  // was already pushed by a producer kernel earlier on the same stream.
  void signal(cudaStream_t s);

  // Publishes rows x cols (ld_src) of `src` into slot `rank` of buffer b on
  // every peer (and on this rank too unless skip_self) at leading dimension
  // ld_dst, then raises this stage's ready flag on every peer.  The stream
  // must already be ordered after this rank's wait_ready() of the previous
  // stage (see above).
  void publish(int b, const float* src, int64_t ld_src, int64_t rows, int64_t cols,
               int64_t slot_floats, int64_t ld_dst, bool skip_self, cudaStream_t s);
  // Waits until every peer published the current stage, then advances the
  // local stage counter.
  void wait_ready(cudaStream_t s);

  // Pipelined form of publish(): one destination per call, in the caller's
  // order, each raising that destination's ready flag when its copy is done;
  // `last` closes the stage (advances the publish count).  Every stage must
  // still end with wait_ready() on the SpMM stream.
  void publish_to(int b, int dest, const float* src, int64_t ld_src, int64_t rows, int64_t cols,
                  int64_t slot_floats, int64_t ld_dst, bool last, cudaStream_t s);
  // Waits until peer q published the current stage (no counter change).
  void wait_slot(int q, cudaStream_t s);
  // Throws NcclError when a device wait of this exchange timed out.
  void check() const;

 private:
  int rank_ = 0, ranks_ = 1, device_ = 0;
  bool same_process_ = false;
  float* base_[kBuffers] = {};          // own allocations
  uint64_t* flags_ = nullptr;            // own: ready[P] | pub_ctr | wait_ctr | arrivals
  std::vector<float*> peer_buf_[kBuffers];  // [b][q] (q == rank: own)
  std::vector<uint64_t*> peer_flags_;    // [q]
  DevBuf<float*> d_bufs_[kBuffers];      // device copies of peer_buf_
  DevBuf<uint64_t*> d_flags_;            // device copy of peer_flags_
  std::vector<void*> opened_;            // IPC mappings to close
  WaitError* err_host_ = nullptr;        // host-mapped wait-error word
  WaitError* err_dev_ = nullptr;
  // In-process world: host-side issued counts (publish / wait stages).
  LocalWorld* local_ = nullptr;
  int channel_ = 0;
  uint64_t host_pub_ = 0, host_wait_ = 0;
  std::vector<int> peers_;
  void post_issued();
  void wait_issued(const std::vector<int>& who, uint64_t stage);
};

}  // namespace cagnet
