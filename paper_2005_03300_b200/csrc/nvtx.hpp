// NVTX ranges (header-only nvtx3, no link dependency): host-side markers for
// the epoch phases and collectives, seen by nsys / `ncu --nvtx` when a tool is
// attached and a no-op otherwise.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace cagnet {

class NvtxRange {
 public:
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace cagnet
