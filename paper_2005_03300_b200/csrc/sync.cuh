// Device-side flag waits shared by the peer-memory panel exchange (p2p.cu)
// and the in-process collectives (comm_local.cu).
//
// A wait never traps: after kSpinLimitNs of spinning it records what it was
// waiting for in a host-mapped error word and returns, so the CUDA context
// stays usable and the host turns the record into a CAGNET_ENCCL status at
// its next synchronisation point (the reference's deadlock detector raises
// SimError instead of hanging, runtime.cpp:58-136).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace cagnet {

// Lives in pinned host memory mapped into the device address space, so the
// host can read it without synchronising any stream.
struct WaitError {
  volatile uint32_t code;         // 0 = none, 1 = wait timed out
  volatile int32_t channel;       // group id / panel channel of the failed wait
  volatile int32_t waiter;        // member that waited
  volatile int32_t peer;          // member it waited for
  volatile uint64_t want, seen;   // flag target and last value read
  uint64_t limit_ns;              // spin budget (CAGNET_WAIT_TIMEOUT_MS, default 20 s)
};

// Allocates a zeroed WaitError in mapped pinned memory with the spin budget
// set; *dev receives the device alias.
WaitError* wait_error_alloc(WaitError** dev);
void wait_error_free(WaitError* host);
// "" when no wait failed, else a one-line description.
std::string wait_error_message(const WaitError* host, const char* what);

constexpr uint64_t kSpinLimitNs = 20ull * 1000 * 1000 * 1000;  // default budget: 20 s

#ifdef __CUDACC__
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spins until *p >= target.  Returns false (after recording the failure in
// err, first failure wins) on timeout or when another wait already failed.
__device__ __forceinline__ bool spin_until_geq(const uint64_t* p, uint64_t target, WaitError* err,
                                               int channel, int waiter, int peer) {
  uint64_t v = ld_acquire_sys(p);
  if (v >= target) return true;
  const uint64_t t0 = globaltimer_ns();
  uint32_t it = 0;
  while ((v = ld_acquire_sys(p)) < target) {
    if ((++it & 1023u) == 0) {
      // Host-mapped reads only every 1024 polls (~0.1 ms).
      if (err && err->code != 0) return false;  // a peer already gave up: unwind fast
      if (globaltimer_ns() - t0 > (err ? err->limit_ns : kSpinLimitNs)) {
        // Plain stores (atomics on mapped host memory are not portable over
        // PCIe); concurrent failures may mix their fields, which only affects
        // the diagnostic text.
        if (err && err->code == 0) {
          err->channel = channel;
          err->waiter = waiter;
          err->peer = peer;
          err->want = target;
          err->seen = v;
          __threadfence_system();
          err->code = 1;
          __threadfence_system();
        }
        return false;
      }
    }
    __nanosleep(128);
  }
  return true;
}
#endif

}  // namespace cagnet
