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

void download_rows(dm_ctx* ctx, void* dst, const void* src, size_t width, size_t pitch, size_t rows,
                   cudaStream_t st) {
    constexpr size_t kHalf = 32ull << 20;
    const size_t bytes = width * rows;
    if (bytes == 0) return;
    if (bytes < (4ull << 20) || is_pinned(dst) || width > kHalf) {
        DM_CUDA(cudaMemcpy2DAsync(dst, width, src, pitch, width, rows, cudaMemcpyDeviceToHost, st));
        DM_CUDA(cudaStreamSynchronize(st));
        return;
    }
    uint8_t* ring = ctx->pin_stage.as<uint8_t>(2 * kHalf);
    if (!ctx->stage_ev[0])
        for (auto& e : ctx->stage_ev) DM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t per = kHalf / width;  // rows per half
    const uint8_t* s = static_cast<const uint8_t*>(src);
    uint8_t* d = static_cast<uint8_t*>(dst);
    auto spill = [&](int h, size_t r0, size_t nr) {  // half h (rows r0..) -> dst, on the host pool
        DM_CUDA(cudaEventSynchronize(ctx->stage_ev[h]));
        const uint8_t* buf = ring + h * kHalf;
        const size_t len = nr * width;
        constexpr size_t piece = 1ull << 20;
        host_pool_run((len + piece - 1) / piece, [&](uint64_t t) {
            const size_t o = t * piece;
            std::memcpy(d + r0 * width + o, buf + o, std::min(piece, len - o));
        });
    };
    size_t prev_r0 = 0, prev_nr = 0;
    int prev_h = -1;
    for (size_t r0 = 0, k = 0; r0 < rows; r0 += per, ++k) {
        const int h = (int)(k & 1);
        const size_t nr = std::min(per, rows - r0);
        DM_CUDA(cudaMemcpy2DAsync(ring + h * kHalf, width, s + r0 * pitch, pitch, width, nr, cudaMemcpyDeviceToHost, st));
        DM_CUDA(cudaEventRecord(ctx->stage_ev[h], st));
        if (prev_h >= 0) spill(prev_h, prev_r0, prev_nr);  // overlaps this half's download
        prev_h = h;
        prev_r0 = r0;
        prev_nr = nr;
    }
    spill(prev_h, prev_r0, prev_nr);
}

void download_host(dm_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    constexpr size_t kRow = 1ull << 20;  // viewed as rows of 1 MB
    const size_t rows = bytes / kRow, tail = bytes - rows * kRow;
    if (rows) download_rows(ctx, dst, src, kRow, kRow, rows, st);
    if (tail) {
        DM_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + rows * kRow, static_cast<const uint8_t*>(src) + rows * kRow,
                                tail, cudaMemcpyDeviceToHost, st));
        DM_CUDA(cudaStreamSynchronize(st));
    }
}

}  // namespace dm
