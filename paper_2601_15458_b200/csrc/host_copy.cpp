// Staged host->device copies (host_copy.h).
#include "host_copy.h"

#include <algorithm>
#include <cstring>

#include "host_pack.h"

namespace dm {

namespace {

bool is_pinned(const void* p) {
    cudaPointerAttributes pa{};
    const bool ok = cudaPointerGetAttributes(&pa, p) == cudaSuccess;
    cudaGetLastError();
    return ok && (pa.type == cudaMemoryTypeHost || pa.type == cudaMemoryTypeManaged);
}

}  // namespace

void upload_host(dm_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    constexpr size_t kHalf = 32ull << 20;  // bytes per staging half
    if (bytes == 0) return;
    if (bytes < (4ull << 20) || is_pinned(src)) {
        // (from pageable memory the driver has staged the bytes when this returns)
        DM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    uint8_t* ring = ctx->pin_stage.as<uint8_t>(2 * kHalf);
    if (!ctx->stage_ev[0])
        for (auto& e : ctx->stage_ev) DM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const uint8_t* s = static_cast<const uint8_t*>(src);
    uint8_t* d = static_cast<uint8_t*>(dst);
    bool used[2] = {false, false};
    for (size_t off = 0, k = 0; off < bytes; off += kHalf, ++k) {
        const int h = (int)(k & 1);
        const size_t len = std::min(kHalf, bytes - off);
        if (used[h]) DM_CUDA(cudaEventSynchronize(ctx->stage_ev[h]));  // this half's last upload is done
        uint8_t* buf = ring + h * kHalf;
        constexpr size_t piece = 1ull << 20;
        host_pool_run((len + piece - 1) / piece, [&](uint64_t t) {
            const size_t o = t * piece;
            std::memcpy(buf + o, s + off + o, std::min(piece, len - o));
        });
        DM_CUDA(cudaMemcpyAsync(d + off, buf, len, cudaMemcpyHostToDevice, st));
        DM_CUDA(cudaEventRecord(ctx->stage_ev[h], st));
        used[h] = true;
    }
    for (int h = 0; h < 2; ++h)
        if (used[h]) DM_CUDA(cudaEventSynchronize(ctx->stage_ev[h]));  // the ring is reusable by the next call
}

}  // namespace dm
