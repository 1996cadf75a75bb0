// NVTX ranges around the library's phases (tree levels and their batches,
// merge levels, streamed chunks, align_sequences steps), so an Nsight
// timeline or an ncu --nvtx filter sees the structure. Header-only NVTX v3:
// without an attached tool each push/pop is a branch on a null pointer.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace dm {

struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace dm
