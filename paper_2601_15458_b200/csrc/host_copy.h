// Bulk host->device copies of caller buffers (sequences, alignment inputs).
// A pageable source would go through the driver's own staging at a fraction
// of the bus rate; here it is copied by the host pool into a small pinned
// double buffer whose halves are uploaded while the next one fills. Pinned
// sources (and small copies) go straight to the copy engine.
#pragma once

#include <cstddef>

#include "dm_internal.h"

namespace dm {

// Enqueues the copy on `st`; when this returns a pageable `src` may be
// reused (staged: the last half has been uploaded; small direct copies: the
// driver has staged them). A pinned `src` must stay valid until `st` has
// executed the copy.
void upload_host(dm_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);

// The reverse for `rows` rows of `width` bytes at device pitch `pitch` into a
// dense host buffer; synchronous (returns with `dst` filled). Large copies
// into pageable memory go through the pinned double buffer, each half's
// spill to `dst` (host pool) overlapping the next half's download.
void download_rows(dm_ctx* ctx, void* dst, const void* src, size_t width, size_t pitch, size_t rows,
                   cudaStream_t st);
// Dense device -> host copy of `bytes` (same staging), synchronous.
void download_host(dm_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);

}  // namespace dm
