// Shared helpers for the cagnet_b200 CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace cagnet {

// Error classes mirror the reference's exception types:
// std::invalid_argument → CAGNET_EINVAL, CUDA failures → CAGNET_ECUDA,
// NCCL failures → CAGNET_ENCCL, std::runtime_error → CAGNET_ERUNTIME.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                  std::to_string(line) + ")");
}

#define CG_CUDA(expr)                                                   \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) ::cagnet::throw_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)

// Number of hot-path kernel launches issued by this library (every launch
// site goes through CG_LAUNCH_CHECK), read by bench.py around its timed region.
inline std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}

#define CG_LAUNCH_CHECK()                               \
  do {                                                  \
    ::cagnet::launch_counter().fetch_add(1, std::memory_order_relaxed); \
    CG_CUDA(cudaGetLastError());                        \
  } while (0)

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}

inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div64(a, b) * b; }

// Leading dimension used for every device-resident dense matrix: rows padded
// to 16 bytes so rows can be moved with 128-bit loads.
inline int64_t padded_ld(int64_t cols) { return round_up(cols > 0 ? cols : 1, 4); }

inline int num_sms(int device) {
  static int cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int v = 0;
  CG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (device >= 0 && device < 64) cached[device] = v;
  return v;
}

inline int current_device() {
  int d = 0;
  CG_CUDA(cudaGetDevice(&d));
  return d;
}

// RAII device buffer.
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count) {
    o.ptr = nullptr;
    o.count = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      count = o.count;
      o.ptr = nullptr;
      o.count = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    count = 0;
  }
  // Grows (never shrinks) the allocation; contents are not preserved.
  void resize(size_t n) {
    if (n <= count && ptr) return;
    release();
    size_t bytes = (n ? n : 1) * sizeof(T);
    CG_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), bytes));
    count = n;
  }
  T* get() const { return ptr; }
};

// Per-stream device workspace (split-K partials, loss partials): grows on
// demand outside graph capture and is reused by every later call on the same
// stream (stream order makes the reuse safe), so eager epochs do no
// allocation churn and captured graphs reference a fixed address.  Never
// shrinks; lives until process exit.
void* stream_scratch(cudaStream_t s, size_t bytes);

}  // namespace cagnet
