// NVTX ranges per kernel family (header-only NVTX3: free unless a profiler
// such as nsys / ncu --nvtx is attached).  Ranges mark host-side launch
// sequences; inside a replayed CUDA graph they mark the capture.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace cprb {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace cprb
