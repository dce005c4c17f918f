// NVTX ranges around the host-visible phases (tracing).  nvtx3 is
// header-only and resolves its injection library lazily: without a profiler
// attached a push/pop is a null-pointer check.  Ranges named cssc.<phase> show
// pack / encrypt / cloud / decrypt on an Nsight Systems timeline next to the
// kernels they enqueue.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace cssc {

struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace cssc
