// In-process communication world (see comm_local.hpp).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>

#include "comm.hpp"
#include "comm_local.hpp"
#include "kernels.cuh"

namespace cagnet {

// ---- host-mapped wait-error word (shared with p2p.cu) ----------------------------------
WaitError* wait_error_alloc(WaitError** dev) {
  WaitError* h = nullptr;
  CG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h), sizeof(WaitError),
                        cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(const_cast<WaitError*>(h), 0, sizeof(WaitError));
  const char* e = std::getenv("CAGNET_WAIT_TIMEOUT_MS");
  const double ms = e ? std::atof(e) : 0.0;
  h->limit_ns = ms > 0 ? static_cast<uint64_t>(ms * 1e6) : kSpinLimitNs;
  CG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(dev), h, 0));
  return h;
}

void wait_error_free(WaitError* host) {
  if (host) cudaFreeHost(host);
}

std::string wait_error_message(const WaitError* e, const char* what) {
  if (!e || e->code == 0) return "";
  return std::string(what) + ": device wait timed out after " +
         std::to_string(e->limit_ns / 1000000ull) + " ms (channel " + std::to_string(e->channel) +
         ", member " + std::to_string(e->waiter) + " waiting for member " + std::to_string(e->peer) +
         ": flag " + std::to_string(e->seen) + " < " + std::to_string(e->want) +
         "); a peer never published — deadlock or a failed rank";
}

namespace {

constexpr int kMaxLocal = 64;
constexpr double kHostWaitSeconds = 300.0;

struct PtrPack {
  const void* p[kMaxLocal];
};

// Raise (phase 0 = arrive: bump this member's sequence first; phase 1 =
// done) this member's flag.  Never waits.
__global__ void lc_raise_kernel(uint64_t* f, int S, int m, int phase) {
  uint64_t* seq = f + 2 * S;
  uint64_t v = seq[m];
  if (phase == 0) {
    v += 1;
    seq[m] = v;
  }
  __threadfence_system();
  st_release_sys(f + (phase ? S : 0) + m, v);
}

// Waits until every member's phase flag reached this member's sequence.
__global__ void lc_wait_kernel(const uint64_t* f, int S, int m, int phase, WaitError* err, int channel) {
  const uint64_t target = f[2 * S + m];
  const uint64_t* flag = f + (phase ? S : 0);
  for (int q = threadIdx.x; q < S; q += blockDim.x)
    if (q != m) spin_until_geq(flag + q, target, err, channel, m, q);
  __syncthreads();
  __threadfence_system();
}

template <class T>
__global__ void lc_sum_kernel(PtrPack src, int S, size_t offset, T* __restrict__ out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(src.p[0])[offset + i];
    for (int q = 1; q < S; ++q) acc += static_cast<const T*>(src.p[q])[offset + i];  // member order
    out[i] = acc;
  }
}

template <class T>
void launch_sum(const std::vector<const void*>& src, size_t offset, T* out, size_t count, int device,
                cudaStream_t s) {
  if (count == 0) return;
  PtrPack pk{};
  for (size_t q = 0; q < src.size(); ++q) pk.p[q] = src[q];
  size_t blocks = (count + 255) / 256;
  const size_t cap = static_cast<size_t>(4 * num_sms(device));
  if (blocks > cap) blocks = cap;
  lc_sum_kernel<T><<<static_cast<unsigned>(blocks), 256, 0, s>>>(pk, static_cast<int>(src.size()), offset,
                                                                  out, count);
  CG_LAUNCH_CHECK();
}

struct Registry {
  std::mutex mu;
  struct Entry {
    std::shared_ptr<LocalWorld> strong;  // until every rank joined
    std::weak_ptr<LocalWorld> weak;
    int joined = 0;
  };
  std::map<uint64_t, Entry> worlds;
};
Registry& registry() {
  static Registry r;
  return r;
}

}  // namespace

bool is_local_id(const void* id128) {
  return id128 && std::memcmp(id128, kLocalMagic, sizeof(kLocalMagic)) == 0;
}

// ---- LocalWorld ------------------------------------------------------------------------
void LocalWorld::create(int ranks, int device, LocalId* out) {
  require(ranks >= 1 && ranks <= kMaxLocal,
          "local world: rank count " + std::to_string(ranks) + " outside [1, " + std::to_string(kMaxLocal) + "]");
  auto w = std::make_shared<LocalWorld>(ranks, device);
  static std::mt19937_64 gen(std::random_device{}());
  Registry& r = registry();
  std::lock_guard<std::mutex> lk(r.mu);
  for (auto it = r.worlds.begin(); it != r.worlds.end();)  // forget finished worlds
    it = (!it->second.strong && it->second.weak.expired()) ? r.worlds.erase(it) : std::next(it);
  uint64_t key = gen();
  while (key == 0 || r.worlds.count(key)) key = gen();
  r.worlds[key] = Registry::Entry{w, w, 0};
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->magic, kLocalMagic, sizeof(kLocalMagic));
  out->key = key;
  out->ranks = ranks;
  out->device = device;
}

std::shared_ptr<LocalWorld> LocalWorld::attach(const LocalId& id, int rank) {
  Registry& r = registry();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.worlds.find(id.key);
  std::shared_ptr<LocalWorld> w = it == r.worlds.end() ? nullptr : it->second.weak.lock();
  if (!w) throw NcclError("local world: unknown or finished communicator id");
  if (rank < 0 || rank >= w->ranks())
    throw std::invalid_argument("local world: rank " + std::to_string(rank) + " outside the world");
  if (++it->second.joined == w->ranks()) it->second.strong.reset();
  return w;
}

void LocalWorld::abort_id(const LocalId& id, const std::string& why) {
  std::shared_ptr<LocalWorld> w;
  {
    Registry& r = registry();
    std::lock_guard<std::mutex> lk(r.mu);
    auto it = r.worlds.find(id.key);
    if (it != r.worlds.end()) w = it->second.weak.lock();
  }
  if (w) w->abort(why);
}

LocalWorld::LocalWorld(int ranks, int device) : ranks_(ranks), device_(device) {
  CG_CUDA(cudaSetDevice(device));
  err_host_ = wait_error_alloc(&err_dev_);
  CG_CUDA(cudaStreamCreateWithFlags(&setup_, cudaStreamNonBlocking));
}

LocalWorld::~LocalWorld() {
  cudaSetDevice(device_);
  if (setup_) cudaStreamSynchronize(setup_);
  for (auto& kv : flags_) cudaFree(kv.second);
  if (setup_) cudaStreamDestroy(setup_);
  wait_error_free(err_host_);
}

uint64_t* LocalWorld::group_flags(const Group& g) {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = flags_.find(g.id);
  if (it != flags_.end()) return it->second;
  const size_t bytes = 3 * g.size() * sizeof(uint64_t);
  uint64_t* f = nullptr;
  CG_CUDA(cudaSetDevice(device_));
  CG_CUDA(cudaMalloc(reinterpret_cast<void**>(&f), bytes));
  CG_CUDA(cudaMemsetAsync(f, 0, bytes, setup_));
  CG_CUDA(cudaStreamSynchronize(setup_));
  flags_[g.id] = f;
  return f;
}

void LocalWorld::wait_locked(std::unique_lock<std::mutex>& lk, const std::function<bool()>& pred,
                             const char* what) {
  const auto deadline =
      std::chrono::steady_clock::now() + std::chrono::duration<double>(kHostWaitSeconds);
  while (!pred()) {
    if (aborted_) throw NcclError(std::string("local world aborted during ") + what + ": " + abort_why_);
    if (cv_.wait_until(lk, deadline) == std::cv_status::timeout && !pred()) {
      aborted_ = true;
      abort_why_ = std::string(what) + " timed out (a rank never arrived: deadlock or a failed rank)";
      cv_.notify_all();
      throw NcclError("local world: " + abort_why_);
    }
  }
  if (aborted_) throw NcclError(std::string("local world aborted during ") + what + ": " + abort_why_);
}

std::vector<std::vector<char>> LocalWorld::exchange(int channel, uint64_t call, int S, int m,
                                                    std::vector<char> mine) {
  std::unique_lock<std::mutex> lk(mu_);
  Slot& sl = slots_[{channel, call}];
  if (sl.entries.empty()) sl.entries.resize(static_cast<size_t>(S));
  sl.entries[static_cast<size_t>(m)] = std::move(mine);
  if (++sl.posted == S) cv_.notify_all();
  const std::string what = "collective rendezvous (group " + std::to_string(channel) + ", call " +
                           std::to_string(call) + ")";
  wait_locked(lk, [&] { return sl.posted == S; }, what.c_str());
  std::vector<std::vector<char>> out = sl.entries;
  if (++sl.taken == S) slots_.erase({channel, call});
  return out;
}

void LocalWorld::post(int channel, int rank, uint64_t value) {
  std::lock_guard<std::mutex> lk(mu_);
  std::vector<uint64_t>& v = posted_[channel];
  if (v.empty()) v.assign(static_cast<size_t>(ranks_), 0);
  if (value > v[static_cast<size_t>(rank)]) v[static_cast<size_t>(rank)] = value;
  cv_.notify_all();
}

void LocalWorld::wait_posted(int channel, const std::vector<int>& who, uint64_t value) {
  std::unique_lock<std::mutex> lk(mu_);
  std::vector<uint64_t>& v = posted_[channel];
  if (v.empty()) v.assign(static_cast<size_t>(ranks_), 0);
  const std::string what = "peer-panel exchange (channel " + std::to_string(channel) + ", stage " +
                           std::to_string(value) + ")";
  wait_locked(lk, [&] {
    for (int q : who)
      if (v[static_cast<size_t>(q)] < value) return false;
    return true;
  }, what.c_str());
}

void LocalWorld::barrier(int rank) {
  (void)rank;
  std::unique_lock<std::mutex> lk(mu_);
  const uint64_t gen = barrier_gen_;
  if (++barrier_count_ == ranks_) {
    barrier_count_ = 0;
    ++barrier_gen_;
    cv_.notify_all();
    return;
  }
  wait_locked(lk, [&] { return barrier_gen_ != gen; }, "world barrier");
}

void LocalWorld::abort(const std::string& why) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!aborted_) {
    aborted_ = true;
    abort_why_ = why;
  }
  cv_.notify_all();
}

void LocalWorld::check() const {
  const std::string msg = wait_error_message(err_host_, "local collective");
  if (!msg.empty()) throw NcclError(msg);
}

// ---- LocalCollectives --------------------------------------------------------------------
// Submission order is what makes the protocol safe on a shared GPU: every
// member launches the kernel that RAISES its flag before it posts to the host
// rendezvous, and launches the kernel that WAITS only after the rendezvous
// saw every member's post.  Each spinning kernel therefore waits only for
// kernels submitted before it, so even when two ranks' streams share one
// hardware work queue (FIFO), a spinning kernel can never sit ahead of the
// kernel it waits for, and implicit context synchronisations (cudaFree,
// module loading) always terminate.
std::vector<std::vector<char>> LocalCollectives::arrive(const Group& g, std::vector<char> mine,
                                                        cudaStream_t s) {
  const int S = static_cast<int>(g.size());
  const int m = g.index_of(rank_);
  uint64_t* f = w_->group_flags(g);
  lc_raise_kernel<<<1, 1, 0, s>>>(f, S, m, 0);
  CG_LAUNCH_CHECK();
  static const bool trace = std::getenv("CAGNET_LOCAL_TRACE") != nullptr;
  const uint64_t call = calls_[g.id]++;
  if (trace) fprintf(stderr, "[local] rank %d group %d call %llu\n", rank_, g.id, (unsigned long long)call);
  auto all = w_->exchange(g.id, call, S, m, std::move(mine));
  lc_wait_kernel<<<1, 32 * ((S + 31) / 32), 0, s>>>(f, S, m, 0, w_->err_dev(), g.id);
  CG_LAUNCH_CHECK();
  return all;
}

std::vector<std::pair<const void*, void*>> LocalCollectives::enter(const Group& g, const void* a, void* b,
                                                                   cudaStream_t s, uint64_t sig) {
  const int S = static_cast<int>(g.size());
  std::vector<char> mine(2 * sizeof(void*) + sizeof(uint64_t));
  std::memcpy(mine.data(), &a, sizeof(void*));
  std::memcpy(mine.data() + sizeof(void*), &b, sizeof(void*));
  std::memcpy(mine.data() + 2 * sizeof(void*), &sig, sizeof(uint64_t));
  auto all = arrive(g, std::move(mine), s);
  std::vector<std::pair<const void*, void*>> out(static_cast<size_t>(S));
  for (int q = 0; q < S; ++q) {
    std::memcpy(&out[q].first, all[q].data(), sizeof(void*));
    std::memcpy(&out[q].second, all[q].data() + sizeof(void*), sizeof(void*));
    uint64_t other = 0;
    std::memcpy(&other, all[q].data() + 2 * sizeof(void*), sizeof(uint64_t));
    if (other != sig)
      throw std::logic_error("local collective mismatch in group " + std::to_string(g.id) + ": rank " +
                             std::to_string(rank_) + " call signature " + std::to_string(sig) +
                             ", member " + std::to_string(q) + " " + std::to_string(other));
  }
  return out;
}

namespace {
uint64_t call_sig(uint64_t op, uint64_t root, uint64_t size) { return (op << 56) ^ (root << 48) ^ size; }
}  // namespace

void LocalCollectives::leave(const Group& g, cudaStream_t s) {
  const int S = static_cast<int>(g.size());
  const int m = g.index_of(rank_);
  uint64_t* f = w_->group_flags(g);
  lc_raise_kernel<<<1, 1, 0, s>>>(f, S, m, 1);
  CG_LAUNCH_CHECK();
  // Host side of the done phase: every member has launched its raise.
  const int channel = -(1 << 20) - g.id;
  const uint64_t n = ++dones_[g.id];
  w_->post(channel, rank_, n);
  w_->wait_posted(channel, g.members, n);
  lc_wait_kernel<<<1, 32 * ((S + 31) / 32), 0, s>>>(f, S, m, 1, w_->err_dev(), g.id);
  CG_LAUNCH_CHECK();
}

char* LocalCollectives::scratch(size_t bytes, cudaStream_t s) {
  if (scratch_.count < bytes) {
    // Captured nodes may already reference the current scratch: it can only
    // grow eagerly (the eager epoch before a capture reaches the maximum).
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    CG_CUDA(cudaStreamIsCapturing(s, &st));
    if (st != cudaStreamCaptureStatusNone)
      throw std::logic_error("local all_reduce: scratch growth inside a graph capture");
    scratch_.resize(bytes + (bytes >> 2));
  }
  return scratch_.get();
}

void LocalCollectives::bcast(const Group& g, int root_member, void* buf, size_t bytes, cudaStream_t s) {
  auto p = enter(g, buf, buf, s, call_sig(1, static_cast<uint64_t>(root_member), bytes));
  if (g.index_of(rank_) != root_member && bytes)
    kern::copy_bytes(buf, p[static_cast<size_t>(root_member)].first, bytes, s);
  leave(g, s);
}

void LocalCollectives::bcast3(const Group& g, int root_member, void* a, size_t na, void* b, size_t nb,
                              void* c, size_t nc, cudaStream_t s) {
  const int m = g.index_of(rank_);
  std::vector<char> mine(3 * sizeof(void*) + 3 * sizeof(size_t));
  std::memcpy(mine.data(), &a, sizeof(void*));
  std::memcpy(mine.data() + sizeof(void*), &b, sizeof(void*));
  std::memcpy(mine.data() + 2 * sizeof(void*), &c, sizeof(void*));
  const size_t sizes[3] = {na, nb, nc};
  std::memcpy(mine.data() + 3 * sizeof(void*), sizes, sizeof(sizes));
  auto all = arrive(g, std::move(mine), s);
  for (size_t q = 0; q < all.size(); ++q)
    if (std::memcmp(all[q].data() + 3 * sizeof(void*), sizes, sizeof(sizes)) != 0)
      throw std::logic_error("local bcast3 size mismatch in group " + std::to_string(g.id) + ": rank " +
                             std::to_string(rank_) + " vs member " + std::to_string(q));
  if (m != root_member) {
    const std::vector<char>& r = all[static_cast<size_t>(root_member)];
    void* src[3];
    std::memcpy(src, r.data(), sizeof(src));
    kern::copy_bytes(a, src[0], na, s);
    kern::copy_bytes(b, src[1], nb, s);
    kern::copy_bytes(c, src[2], nc, s);
  }
  leave(g, s);
}

void LocalCollectives::all_reduce(const Group& g, void* buf, size_t count, int dtype, cudaStream_t s) {
  const size_t es = dtype == 1 ? 8 : 4;
  char* tmp = scratch(count * es, s);
  auto p = enter(g, buf, buf, s, call_sig(2, static_cast<uint64_t>(dtype), count));
  std::vector<const void*> src;
  for (auto& e : p) src.push_back(e.first);
  if (dtype == 1)
    launch_sum<double>(src, 0, reinterpret_cast<double*>(tmp), count, w_->device(), s);
  else
    launch_sum<float>(src, 0, reinterpret_cast<float*>(tmp), count, w_->device(), s);
  leave(g, s);  // every member has read every buffer
  kern::copy_bytes(buf, tmp, count * es, s);
}

void LocalCollectives::reduce_scatter(const Group& g, const void* send, void* recv, size_t slice, int dtype,
                                      cudaStream_t s) {
  auto p = enter(g, send, recv, s, call_sig(3, static_cast<uint64_t>(dtype), slice));
  const int m = g.index_of(rank_);
  std::vector<const void*> src;
  for (auto& e : p) src.push_back(e.first);
  if (dtype == 1)
    launch_sum<double>(src, m * slice, static_cast<double*>(recv), slice, w_->device(), s);
  else
    launch_sum<float>(src, m * slice, static_cast<float*>(recv), slice, w_->device(), s);
  leave(g, s);
}

void LocalCollectives::all_gather(const Group& g, const void* send, void* recv, size_t slice_bytes,
                                  cudaStream_t s) {
  auto p = enter(g, send, recv, s, call_sig(4, 0, slice_bytes));
  for (size_t q = 0; q < p.size(); ++q) {
    char* dst = static_cast<char*>(recv) + q * slice_bytes;
    if (dst != p[q].first) kern::copy_bytes(dst, p[q].first, slice_bytes, s);
  }
  leave(g, s);
}

void LocalCollectives::setup_all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) {
  std::vector<char> mine(bytes);
  if (bytes) CG_CUDA(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  auto all = w_->exchange(-1, setup_calls_++, w_->ranks(), rank_, std::move(mine));
  std::vector<char> cat(bytes * all.size());
  for (size_t q = 0; q < all.size(); ++q)
    if (bytes) std::memcpy(cat.data() + q * bytes, all[q].data(), bytes);
  if (!cat.empty()) CG_CUDA(cudaMemcpyAsync(recv, cat.data(), cat.size(), cudaMemcpyHostToDevice, s));
  CG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace cagnet
