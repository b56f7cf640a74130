// In-process communication world: P ranks as host threads of ONE process
// sharing one GPU (the reference's execution model, runtime.cpp:270-285:
// ranks are OS threads moving real data through rendezvous collectives).
//
// It exists so every P > 1 strategy — collectives, ledger metering, the
// NVLink peer-memory flag protocol, CUDA-graph replays — runs on a single
// B200, where NCCL refuses two ranks on one device.  The data path is the
// same device-flag design as the product's peer-memory exchange (p2p.cu):
//
//   1. raise   : a kernel bumps the member's device sequence counter and
//                raises its arrive flag (never waits);
//   2. host    : rendezvous — the members exchange buffer pointers (blocking,
//                like the reference's collectives);
//   3. wait    : a kernel spins until every member's arrive flag reached the
//                sequence; then data kernels read the peers' buffers directly;
//   4. done    : raise the done flag, a host post/wait, spin on every done
//                flag (nobody overwrites a buffer a peer still reads).
//
// Flags carry device-side sequence numbers, so a captured epoch replays
// unchanged.  Because every raise is SUBMITTED before the host step that
// releases the peers' waits, a spinning kernel only ever waits for kernels
// submitted before it: ranks whose streams share a hardware work queue
// (FIFO) cannot block each other, and implicit context synchronisations
// (cudaFree, module loading) by another rank always terminate.  (Measured:
// with the wait launched before the peers' raises were submitted, 2D/3D runs
// on one B200 stalled in about half the trials; scripts/diag_local.py.)
#pragma once

#include <condition_variable>
#include <functional>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "grid.hpp"
#include "sync.cuh"

namespace cagnet {

// 128-byte communicator id of a local world: magic, key, rank count, device.
constexpr char kLocalMagic[16] = "CAGNET-LOCAL-W1";
struct LocalId {
  char magic[16];
  uint64_t key;
  int32_t ranks;
  int32_t device;
  char pad[128 - 32];
};
static_assert(sizeof(LocalId) == 128, "LocalId must match ncclUniqueId's size");

bool is_local_id(const void* id128);

class LocalWorld {
 public:
  // Creates a world of `ranks` ranks on `device` and writes its id.
  static void create(int ranks, int device, LocalId* out);
  // Joins the world named by id (each rank once); the registry forgets the
  // world when the last rank joined.
  static std::shared_ptr<LocalWorld> attach(const LocalId& id, int rank);
  // Marks the world named by id failed: every blocked or future host wait
  // throws (a rank that raised must not leave its peers waiting).
  static void abort_id(const LocalId& id, const std::string& why);

  LocalWorld(int ranks, int device);
  ~LocalWorld();
  LocalWorld(const LocalWorld&) = delete;
  LocalWorld& operator=(const LocalWorld&) = delete;

  int ranks() const { return ranks_; }
  int device() const { return device_; }

  // Device flags of group g: arrive[S] | done[S] | seq[S] (uint64, zeroed on
  // first registration; every member registers its groups at construction).
  uint64_t* group_flags(const Group& g);

  // Host rendezvous on (channel, call): member m of a group of size S posts
  // `mine` and receives every member's payload in member order.
  std::vector<std::vector<char>> exchange(int channel, uint64_t call, int S, int m,
                                          std::vector<char> mine);
  // Monotone per-rank progress counters on a channel (peer-memory panels:
  // "rank r has issued its publish of stage s").
  void post(int channel, int rank, uint64_t value);
  void wait_posted(int channel, const std::vector<int>& ranks, uint64_t value);
  // All ranks of the world.
  void barrier(int rank);

  void abort(const std::string& why);
  WaitError* err_dev() const { return err_dev_; }
  // Throws NcclError if a device wait of this world timed out.
  void check() const;

 private:
  void wait_locked(std::unique_lock<std::mutex>& lk, const std::function<bool()>& pred,
                   const char* what);
  struct Slot {
    std::vector<std::vector<char>> entries;
    int posted = 0;
    int taken = 0;
  };
  int ranks_, device_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::pair<int, uint64_t>, Slot> slots_;
  std::map<int, std::vector<uint64_t>> posted_;
  std::map<int, uint64_t*> flags_;
  uint64_t barrier_gen_ = 0;
  int barrier_count_ = 0;
  bool aborted_ = false;
  std::string abort_why_;
  WaitError* err_host_ = nullptr;
  WaitError* err_dev_ = nullptr;
  cudaStream_t setup_ = nullptr;
};

// The data movement of Comm's collectives over a LocalWorld (the metering
// stays in comm.cu).  All calls are made by member `m` of group g on stream s.
class LocalCollectives {
 public:
  LocalCollectives(std::shared_ptr<LocalWorld> w, int rank) : w_(std::move(w)), rank_(rank) {}
  LocalWorld& world() { return *w_; }

  void bcast(const Group& g, int root_member, void* buf, size_t bytes, cudaStream_t s);
  // Three arrays of one root in one rendezvous.
  void bcast3(const Group& g, int root_member, void* a, size_t na, void* b, size_t nb, void* c,
              size_t nc, cudaStream_t s);
  // dtype: 0 = f32, 1 = f64.
  void all_reduce(const Group& g, void* buf, size_t count, int dtype, cudaStream_t s);
  void reduce_scatter(const Group& g, const void* send, void* recv, size_t slice, int dtype,
                      cudaStream_t s);
  void all_gather(const Group& g, const void* send, void* recv, size_t slice_bytes, cudaStream_t s);
  // Host-synchronous world all-gather of `bytes` per rank (setup metadata).
  void setup_all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s);

 private:
  // Raise + rendezvous (payload exchange) + arrive wait.
  std::vector<std::vector<char>> arrive(const Group& g, std::vector<char> mine, cudaStream_t s);
  // Rendezvous + arrive barrier; returns the members' (a, b) pointers.
  // sig: the call's shape (operation, root, sizes); every member must pass
  // the same one — a mismatch is a host-side bug and throws.
  std::vector<std::pair<const void*, void*>> enter(const Group& g, const void* a, void* b,
                                                   cudaStream_t s, uint64_t sig);
  void leave(const Group& g, cudaStream_t s);
  char* scratch(size_t bytes, cudaStream_t s);

  std::shared_ptr<LocalWorld> w_;
  int rank_;
  std::map<int, uint64_t> calls_;  // group id -> host call index
  std::map<int, uint64_t> dones_;  // group id -> done phases issued
  uint64_t setup_calls_ = 0;
  DevBuf<char> scratch_;
};

}  // namespace cagnet
