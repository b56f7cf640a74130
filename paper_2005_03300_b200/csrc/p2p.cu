// NVLink peer-memory panel exchange (see p2p.hpp).
#include <unistd.h>

#include <cstring>

#include "p2p.hpp"
#include "sync.cuh"

namespace cagnet {
namespace {

// Flag block of every rank (uint64): ready[P] | consumed[P] | ctr | arrivals.
//   ready[q]    = last stage rank q published into this rank's buffers
//   consumed[q] = last stage whose buffer rank q finished reading
//   ctr         = stages completed by this rank (advanced by consumed())
struct Flags {
  int P;
  __device__ uint64_t* ready(uint64_t* f) const { return f; }
  __device__ uint64_t* pub_ctr(uint64_t* f) const { return f + P; }
  __device__ uint64_t* wait_ctr(uint64_t* f) const { return f + P + 1; }
  __device__ uint64_t* arrivals(uint64_t* f) const { return f + P + 2; }
};

// Copies the panel into slot `rank` of every destination buffer; the last CTA
// to finish raises ready[rank] = s on every peer (s = this rank's publish count).
__global__ void publish_kernel(float* const* bufs, uint64_t* const* flags, int rank, int P,
                               bool skip_self, const float* __restrict__ src, int64_t ld_src,
                               uint32_t rows, uint32_t c4, int64_t slot_floats, int64_t ld_dst) {
  const Flags F{P};
  uint64_t* my = flags[rank];
  const uint64_t s = *F.pub_ctr(my) + 1;
  const uint32_t total = rows * c4;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t r = e / c4, c = e - r * c4;
    const float4 v = *reinterpret_cast<const float4*>(src + r * ld_src + 4 * c);
    const int64_t off = rank * slot_floats + r * ld_dst + 4 * c;
#pragma unroll 4
    for (int d = 1; d <= P; ++d) {
      const int q = (rank + d) % P;  // peers first, self last
      if (q == rank && skip_self) continue;
      *reinterpret_cast<float4*>(bufs[q] + off) = v;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev =
        atomicAdd(reinterpret_cast<unsigned long long*>(F.arrivals(my)), 1ull);
    if (prev == gridDim.x - 1) {
      *F.arrivals(my) = 0;
      *F.pub_ctr(my) = s;
      __threadfence_system();
      for (int q = 0; q < P; ++q)
        if (q != rank) st_release_sys(F.ready(flags[q]) + rank, s);
    }
  }
}

// One destination of a pipelined stage: the last CTA raises ready[rank] on q
// (and, for the stage's last destination, advances the publish count).
__global__ void publish_one_kernel(float* const* bufs, uint64_t* const* flags, int rank, int P, int q,
                                   bool last, const float* __restrict__ src, int64_t ld_src, uint32_t rows,
                                   uint32_t c4, int64_t slot_floats, int64_t ld_dst) {
  const Flags F{P};
  uint64_t* my = flags[rank];
  const uint64_t s = *F.pub_ctr(my) + 1;
  const uint32_t total = rows * c4;
  float* dst = bufs[q] + rank * slot_floats;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t r = e / c4, c = e - r * c4;
    *reinterpret_cast<float4*>(dst + r * ld_dst + 4 * c) = *reinterpret_cast<const float4*>(src + r * ld_src + 4 * c);
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev =
        atomicAdd(reinterpret_cast<unsigned long long*>(F.arrivals(my)), 1ull);
    if (prev == gridDim.x - 1) {
      *F.arrivals(my) = 0;
      if (last) *F.pub_ctr(my) = s;
      __threadfence_system();
      st_release_sys(F.ready(flags[q]) + rank, s);
    }
  }
}

__global__ void wait_slot_kernel(uint64_t* const* flags, int rank, int P, int q, WaitError* err) {
  const Flags F{P};
  uint64_t* my = flags[rank];
  const uint64_t s = *F.wait_ctr(my) + 1;
  if (threadIdx.x == 0) spin_until_geq(F.ready(my) + q, s, err, -2, rank, q);
  __threadfence_system();
}

__global__ void wait_ready_kernel(uint64_t* const* flags, int rank, int P, WaitError* err) {
  const Flags F{P};
  uint64_t* my = flags[rank];
  const uint64_t s = *F.wait_ctr(my) + 1;
  for (int q = threadIdx.x; q < P; q += blockDim.x)
    if (q != rank) spin_until_geq(F.ready(my) + q, s, err, -2, rank, q);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *F.wait_ctr(my) = s;
}

constexpr int kAllocs = PeerPanels::kBuffers + 1;  // panel buffers + flags

struct PeerInfo {
  cudaIpcMemHandle_t h[kAllocs];
  uint64_t ptr[kAllocs];
  uint64_t pid;
  int32_t device;
  int32_t ok;
};

}  // namespace

PeerPanels::~PeerPanels() {
  if (ranks_ <= 1) return;
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  for (float* b : base_)
    if (b) cudaFree(b);
  if (flags_) cudaFree(flags_);
  wait_error_free(err_host_);
}

void PeerPanels::check() const {
  const std::string msg = wait_error_message(err_host_, "peer-memory panel exchange");
  if (!msg.empty()) throw NcclError(msg);
}

void PeerPanels::post_issued() {
  if (local_) local_->post(channel_, rank_, ++host_pub_);
}

void PeerPanels::wait_issued(const std::vector<int>& who, uint64_t stage) {
  if (local_) local_->wait_posted(channel_, who, stage);
}

bool PeerPanels::init(Comm& comm, int rank, int ranks, int device, size_t bytes, cudaStream_t s) {
  rank_ = rank;
  ranks_ = ranks;
  device_ = device;
  if (ranks <= 1) return false;
  const int P = ranks;
  local_ = comm.local_world();
  if (local_) channel_ = comm.next_local_channel();
  host_pub_ = host_wait_ = 0;
  peers_.clear();
  for (int q = 0; q < P; ++q)
    if (q != rank) peers_.push_back(q);
  if (!err_host_) err_host_ = wait_error_alloc(&err_dev_);
  // Allocate first so every rank can advertise handles; freed again on fallback.
  for (int b = 0; b < kBuffers; ++b) {
    CG_CUDA(cudaMalloc(reinterpret_cast<void**>(&base_[b]), bytes));
    CG_CUDA(cudaMemset(base_[b], 0, bytes));
  }
  CG_CUDA(cudaMalloc(reinterpret_cast<void**>(&flags_), (P + 3) * sizeof(uint64_t)));
  CG_CUDA(cudaMemset(flags_, 0, (P + 3) * sizeof(uint64_t)));
  // Legacy-stream zeroing: finished before any peer (non-blocking streams) can write.
  CG_CUDA(cudaStreamSynchronize(nullptr));

  PeerInfo mine{};
  void* ptrs[kAllocs];
  for (int b = 0; b < kBuffers; ++b) ptrs[b] = base_[b];
  ptrs[kBuffers] = flags_;
  mine.ok = 1;
  for (int i = 0; i < kAllocs; ++i) {
    mine.ptr[i] = reinterpret_cast<uint64_t>(ptrs[i]);
    if (cudaIpcGetMemHandle(&mine.h[i], ptrs[i]) != cudaSuccess) {
      cudaGetLastError();
      mine.ok = 0;
    }
  }
  mine.pid = static_cast<uint64_t>(getpid());
  mine.device = device;
  const size_t words = (sizeof(PeerInfo) + 7) / 8;
  DevBuf<uint64_t> dsend(words), drecv(words * P);
  std::vector<uint64_t> hsend(words, 0), hrecv(words * P, 0);
  std::memcpy(hsend.data(), &mine, sizeof(PeerInfo));
  CG_CUDA(cudaMemcpy(dsend.get(), hsend.data(), words * 8, cudaMemcpyHostToDevice));
  CG_CUDA(cudaStreamSynchronize(nullptr));  // legacy-stream copy done before the non-blocking streams read it
  comm.setup_all_gather(dsend.get(), drecv.get(), words, ncclUint64, s);
  CG_CUDA(cudaStreamSynchronize(s));
  CG_CUDA(cudaMemcpy(hrecv.data(), drecv.get(), words * P * 8, cudaMemcpyDeviceToHost));
  std::vector<PeerInfo> all(static_cast<size_t>(P));
  for (int q = 0; q < P; ++q) std::memcpy(&all[q], hrecv.data() + q * words, sizeof(PeerInfo));

  // Map every peer; agree on the outcome (all ranks take the same path).
  bool ok = true;
  same_process_ = true;
  for (int q = 0; q < P; ++q) {
    ok = ok && all[q].ok;
    if (all[q].pid != mine.pid) same_process_ = false;
  }
  for (int b = 0; b < kBuffers; ++b) peer_buf_[b].assign(static_cast<size_t>(P), nullptr);
  peer_flags_.assign(static_cast<size_t>(P), nullptr);
  for (int q = 0; q < P && ok; ++q) {
    if (q == rank) {
      for (int b = 0; b < kBuffers; ++b) peer_buf_[b][q] = base_[b];
      peer_flags_[q] = flags_;
      continue;
    }
    if (same_process_ && all[q].device == device) {
      // Ranks sharing one GPU (in-process world): plain device pointers.
      for (int b = 0; b < kBuffers; ++b) peer_buf_[b][q] = reinterpret_cast<float*>(all[q].ptr[b]);
      peer_flags_[q] = reinterpret_cast<uint64_t*>(all[q].ptr[kBuffers]);
    } else if (same_process_) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, device, all[q].device);
      if (!can) {
        ok = false;
        break;
      }
      const cudaError_t e = cudaDeviceEnablePeerAccess(all[q].device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        ok = false;
        break;
      }
      cudaGetLastError();
      for (int b = 0; b < kBuffers; ++b) peer_buf_[b][q] = reinterpret_cast<float*>(all[q].ptr[b]);
      peer_flags_[q] = reinterpret_cast<uint64_t*>(all[q].ptr[kBuffers]);
    } else {
      void* p[kAllocs] = {};
      for (int i = 0; i < kAllocs && ok; ++i) {
        if (cudaIpcOpenMemHandle(&p[i], all[q].h[i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          ok = false;
        } else {
          opened_.push_back(p[i]);
        }
      }
      if (!ok) break;
      for (int b = 0; b < kBuffers; ++b) peer_buf_[b][q] = static_cast<float*>(p[b]);
      peer_flags_[q] = static_cast<uint64_t*>(p[kBuffers]);
    }
  }
  // Agreement: all-gather the per-rank verdicts.
  DevBuf<int32_t> vs(1), va(static_cast<size_t>(P));
  const int32_t v = ok ? 1 : 0;
  CG_CUDA(cudaMemcpy(vs.get(), &v, sizeof(v), cudaMemcpyHostToDevice));
  CG_CUDA(cudaStreamSynchronize(nullptr));  // legacy-stream copy done before the non-blocking streams read it
  comm.setup_all_gather(vs.get(), va.get(), 1, ncclInt32, s);
  CG_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> verdicts(static_cast<size_t>(P));
  CG_CUDA(cudaMemcpy(verdicts.data(), va.get(), P * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int32_t x : verdicts) ok = ok && x;
  if (!ok) {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    opened_.clear();
    for (float*& b : base_) {
      cudaFree(b);
      b = nullptr;
    }
    cudaFree(flags_);
    flags_ = nullptr;
    return false;
  }
  for (int b = 0; b < kBuffers; ++b) {
    d_bufs_[b].resize(static_cast<size_t>(P));
    CG_CUDA(cudaMemcpy(d_bufs_[b].get(), peer_buf_[b].data(), P * sizeof(float*), cudaMemcpyHostToDevice));
  }
  d_flags_.resize(static_cast<size_t>(P));
  CG_CUDA(cudaMemcpy(d_flags_.get(), peer_flags_.data(), P * sizeof(uint64_t*), cudaMemcpyHostToDevice));
  CG_CUDA(cudaStreamSynchronize(nullptr));  // legacy-stream copy done before the non-blocking streams read it
  return true;
}

void PeerPanels::publish(int b, const float* src, int64_t ld_src, int64_t rows, int64_t cols,
                         int64_t slot_floats, int64_t ld_dst, bool skip_self, cudaStream_t s) {
  require(ld_src % 4 == 0 && ld_dst % 4 == 0 && slot_floats % 4 == 0 &&
              reinterpret_cast<uintptr_t>(src) % 16 == 0,
          "PeerPanels::publish: rows must be 16 B aligned");
  const int64_t c4 = (cols + 3) / 4;
  require(c4 * 4 <= ld_src && c4 * 4 <= ld_dst, "PeerPanels::publish: padded width exceeds ld");
  const int64_t total = rows * c4;
  int blocks = static_cast<int>(ceil_div64(total > 0 ? total : 1, 256));
  const int cap = 2 * num_sms(device_);
  if (blocks > cap) blocks = cap;
  publish_kernel<<<blocks, 256, 0, s>>>(d_bufs_[b].get(), d_flags_.get(), rank_, ranks_, skip_self, src,
                                        ld_src, static_cast<uint32_t>(rows), static_cast<uint32_t>(c4),
                                        slot_floats, ld_dst);
  CG_LAUNCH_CHECK();
  post_issued();
}

void PeerPanels::publish_to(int b, int dest, const float* src, int64_t ld_src, int64_t rows, int64_t cols,
                            int64_t slot_floats, int64_t ld_dst, bool last, cudaStream_t s) {
  require(ld_src % 4 == 0 && ld_dst % 4 == 0 && slot_floats % 4 == 0 &&
              reinterpret_cast<uintptr_t>(src) % 16 == 0,
          "PeerPanels::publish_to: rows must be 16 B aligned");
  require(dest >= 0 && dest < ranks_ && dest != rank_, "PeerPanels::publish_to: bad destination");
  const int64_t c4 = (cols + 3) / 4;
  require(c4 * 4 <= ld_src && c4 * 4 <= ld_dst, "PeerPanels::publish_to: padded width exceeds ld");
  const int64_t total = rows * c4;
  int blocks = static_cast<int>(ceil_div64(total > 0 ? total : 1, 256));
  const int cap = 2 * num_sms(device_);
  if (blocks > cap) blocks = cap;
  publish_one_kernel<<<blocks, 256, 0, s>>>(d_bufs_[b].get(), d_flags_.get(), rank_, ranks_, dest, last, src,
                                            ld_src, static_cast<uint32_t>(rows), static_cast<uint32_t>(c4),
                                            slot_floats, ld_dst);
  CG_LAUNCH_CHECK();
  if (last) post_issued();  // the stage's pushes were issued back to back
}

void PeerPanels::signal(cudaStream_t s) {
  // A copy-free publish: one CTA fences and raises the flags (the rows were
  // stored by an earlier kernel on this stream, complete at its boundary).
  publish_kernel<<<1, 32, 0, s>>>(d_bufs_[0].get(), d_flags_.get(), rank_, ranks_, true, nullptr, 0, 0, 0, 0, 0);
  CG_LAUNCH_CHECK();
  post_issued();
}

void PeerPanels::wait_slot(int q, cudaStream_t s) {
  wait_issued({q}, host_wait_ + 1);
  wait_slot_kernel<<<1, 32, 0, s>>>(d_flags_.get(), rank_, ranks_, q, err_dev_);
  CG_LAUNCH_CHECK();
}

void PeerPanels::wait_ready(cudaStream_t s) {
  wait_issued(peers_, ++host_wait_);
  wait_ready_kernel<<<1, 32 * ((ranks_ + 31) / 32), 0, s>>>(d_flags_.get(), rank_, ranks_, err_dev_);
  CG_LAUNCH_CHECK();
}

}  // namespace cagnet
