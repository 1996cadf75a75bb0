// Streamed pair batches from host memory (the end-to-end path of the
// distance engine): pair i = (sequence 2i, sequence 2i+1) of a packed host
// buffer. The batch is cut into chunks that move through three streams:
//   copy stream     uploads of chunks c+1..c+3 (offsets, then residues)
//   planner stream  census/recode/bit-planes + pair planning of chunk c+1
//                   (one planner context per staging slot: own scratch)
//   ctx->stream     distance kernels of chunk c
// The planners' host syncs never wait on the distance kernels, and nothing
// but the bulk uploads uses the host->device copy engine (all per-chunk
// metadata is derived on the device), so upload, planning and compute
// overlap. Results land in one device array and come back in one copy.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "capi_guard.h"

namespace dm {
namespace {

__global__ void iota_pairs(uint32_t* ia, uint32_t* ib, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        ia[i] = (uint32_t)(2 * i);
        ib[i] = (uint32_t)(2 * i + 1);
    }
}

}  // namespace

namespace {

dm_ctx* prep_context(dm_ctx* ctx, int k) {
    if (!ctx->prep[k]) {
        auto* p = new dm_ctx;
        p->device = ctx->device;
        p->sm_count = ctx->sm_count;
        // planners run at high priority: their blocks take the first SM slots
        // the distance kernels free (the host waits on them)
        int least = 0, greatest = 0;
        DM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        if (cudaStreamCreateWithPriority(&p->stream, cudaStreamNonBlocking, greatest) != cudaSuccess) {
            delete p;
            throw cuda_error("cannot create a planner stream");
        }
        p->own_stream = p->stream;
        DM_CUDA(cudaEventCreate(&p->ev0));
        DM_CUDA(cudaEventCreate(&p->ev1));
        ctx->prep[k] = p;
    }
    return ctx->prep[k];
}

constexpr int NB = dm_ctx::kStreamSlots;  // chunks in flight: uploading (NB-1), planning/computing

struct ChunkEvents {
    cudaEvent_t copied[NB] = {}, recoded[NB] = {}, planned[NB] = {}, done[NB] = {}, ready = nullptr;
    ChunkEvents() {
        for (int b = 0; b < NB; ++b)
            for (cudaEvent_t* e : {&copied[b], &recoded[b], &planned[b], &done[b]})
                DM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        DM_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    }
    ~ChunkEvents() {
        for (int b = 0; b < NB; ++b)
            for (cudaEvent_t e : {copied[b], recoded[b], planned[b], done[b]})
                if (e) cudaEventDestroy(e);
        if (ready) cudaEventDestroy(ready);
    }
};

}  // namespace

void lev_pairs_packed(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint64_t npairs, uint32_t* out,
                      LevTotals* tot, bool timing) {
    (void)timing;
    if (npairs == 0) return;
    if (2 * npairs > 0xffffffffull) throw invalid_argument("too many sequences in one streamed batch");
    for (uint64_t i = 0; i < 2 * npairs; ++i)
        if (offsets[i + 1] < offsets[i]) throw invalid_argument("sequence offsets must be non-decreasing");
    // Chunk boundaries (pair indices). Sizes ramp up from `small` to `big`
    // residue bytes so the first kernels start after a short upload, and
    // halve again over the tail so little compute is left once the last
    // upload lands.
    uint64_t big = 256ull << 20, small = 32ull << 20;
    if (const char* env = std::getenv("DM_STREAM_CHUNK_BYTES"))
        big = small = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10));
    std::vector<uint64_t> cb{0};
    for (uint64_t lo = 0, k = 0; lo < npairs; ++k) {
        const uint64_t rem = offsets[2 * npairs] - offsets[2 * lo];
        uint64_t t = std::min(big, small << std::min<uint64_t>(k, 20));
        if (rem < 2 * t) t = std::max(small, rem / 2);
        // smallest hi > lo with offsets[2hi] - offsets[2lo] >= t
        uint64_t a = lo + 1, z = npairs;
        while (a < z) {
            const uint64_t mid = (a + z) / 2;
            if (offsets[2 * mid] - offsets[2 * lo] >= t) z = mid; else a = mid + 1;
        }
        lo = a;
        cb.push_back(lo);
    }
    const uint64_t nchunks = cb.size() - 1;
    uint64_t per = 1, maxbytes = 0;
    for (uint64_t c = 0; c < nchunks; ++c) {
        per = std::max(per, cb[c + 1] - cb[c]);
        maxbytes = std::max(maxbytes, offsets[2 * cb[c + 1]] - offsets[2 * cb[c]]);
    }
    const uint64_t oslot = 2 * per + 1;  // offsets per staging slot
    if (!ctx->copy_stream) DM_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    dm_ctx* prep[NB];
    for (int b = 0; b < NB; ++b) prep[b] = prep_context(ctx, b);
    ChunkEvents ev;
    dm_seqset* live[NB] = {};
    const bool trace = std::getenv("DM_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tl;
    std::vector<std::pair<cudaEvent_t, uint64_t>> tc;
    cudaEvent_t tl0 = nullptr;
    if (trace) {
        cudaEventCreate(&tl0);
        cudaEventRecord(tl0, ctx->stream);
    }
    auto now_ms = [&] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    };
    auto drain = [&] {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamSynchronize(ctx->stream);
        for (int b = 0; b < NB; ++b) {
            delete live[b];
            live[b] = nullptr;
            cudaStreamSynchronize(prep[b]->stream);
        }
    };
    try {
        // every buffer the side streams touch is (re)allocated on ctx->stream first
        uint8_t* stage[NB];
        for (int b = 0; b < NB; ++b) stage[b] = (uint8_t*)ctx->stage[b].get(maxbytes + 16);
        uint64_t* d_offs = ctx->stream_offs.as<uint64_t>(NB * oslot);
        uint64_t* h_offs = ctx->pin_items.as<uint64_t>(NB * oslot);
        uint32_t* d_ab = ctx->stream_pairs.as<uint32_t>(2 * per + 2);
        uint32_t* d_res = ctx->stream_out.as<uint32_t>(npairs);
        uint32_t* h_res = ctx->pin_out.as<uint32_t>(npairs);
        const int grid = (int)std::min<uint64_t>((per + 255) / 256, (uint64_t)ctx->sm_count * 4);
        iota_pairs<<<std::max(grid, 1), 256, 0, ctx->stream>>>(d_ab, d_ab + per, per);
        DM_CUDA(cudaGetLastError());
        DM_CUDA(cudaEventRecord(ev.ready, ctx->stream));
        DM_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev.ready, 0));
        auto issue_copy = [&](uint64_t c) {
            const int b = (int)(c % NB);
            const uint64_t lo = cb[c], hi = cb[c + 1];
            // chunk offsets go up from a pinned slot (a pageable copy would block
            // the host behind the bulk upload already queued)
            if (c >= NB) DM_CUDA(cudaEventSynchronize(ev.copied[b]));  // slot's last upload done
            std::memcpy(h_offs + b * oslot, offsets + 2 * lo, (2 * (hi - lo) + 1) * 8);
            if (c >= NB) DM_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev.recoded[b], 0));
            DM_CUDA(cudaMemcpyAsync(d_offs + b * oslot, h_offs + b * oslot, (2 * (hi - lo) + 1) * 8,
                                    cudaMemcpyHostToDevice, ctx->copy_stream));
            const uint64_t a0 = offsets[2 * lo], a1 = offsets[2 * hi];
            if (a1 > a0)
                DM_CUDA(cudaMemcpyAsync(stage[b], data + a0, a1 - a0, cudaMemcpyHostToDevice, ctx->copy_stream));
            DM_CUDA(cudaEventRecord(ev.copied[b], ctx->copy_stream));
            if (trace) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, ctx->copy_stream);
                tc.push_back({e, a1 - a0});
            }
        };
        for (uint64_t c = 0; c + 1 < NB && c < nchunks; ++c) issue_copy(c);
        for (uint64_t c = 0; c < nchunks; ++c) {
            const int b = (int)(c % NB);
            dm_ctx* P = prep[b];
            const uint64_t lo = cb[c], hi = cb[c + 1], cnt = hi - lo;
            DM_CUDA(cudaStreamWaitEvent(P->stream, ev.copied[b], 0));
            if (c >= NB) DM_CUDA(cudaStreamWaitEvent(P->stream, ev.done[b], 0));  // chunk c-NB's kernels
            delete live[b];  // stream-ordered frees behind that wait
            live[b] = nullptr;
            // census + recode + bit-planes on the planner stream (one host sync)
            const double t0 = trace ? now_ms() : 0.0;
            live[b] = seqset_create_device(P, stage[b], d_offs + b * oslot, offsets + 2 * lo, (uint32_t)(2 * cnt));
            DM_CUDA(cudaEventRecord(ev.recoded[b], P->stream));  // staging b free again
            const double t1 = trace ? now_ms() : 0.0;
            // keep NB-1 chunk uploads queued so the copy engine never idles
            if (c + NB - 1 < nchunks) issue_copy(c + NB - 1);
            // plan on the planner stream (second host sync), kernels on ctx->stream
            lev_plan_then_launch(P, ctx, live[b], d_ab, d_ab + per, cnt, d_res + lo, ev.planned[b], tot);
            DM_CUDA(cudaEventRecord(ev.done[b], ctx->stream));
            if (trace) {  // GPU-side timeline: when chunk c's planning and kernels finished
                cudaEvent_t a, k;
                cudaEventCreate(&a);
                cudaEventCreate(&k);
                cudaEventRecord(a, P->stream);
                cudaEventRecord(k, ctx->stream);
                tl.push_back({a, k});
            }
            if (trace)
                std::fprintf(stderr, "[stream] chunk %llu pairs %llu: census-wait+recode %.2f..%.2f ms, planned %.2f ms\n",
                             (unsigned long long)c, (unsigned long long)cnt, t0, t1, now_ms());
        }
        DM_CUDA(cudaMemcpyAsync(h_res, d_res, npairs * 4, cudaMemcpyDeviceToHost, ctx->stream));
        DM_CUDA(cudaStreamSynchronize(ctx->stream));
        if (trace) {
            std::fprintf(stderr, "[stream] all kernels done %.2f ms\n", now_ms());
            for (size_t i = 0; i < tl.size(); ++i) {
                float pa = 0, ka = 0;
                cudaEventElapsedTime(&pa, tl0, tl[i].first);
                cudaEventElapsedTime(&ka, tl0, tl[i].second);
                std::fprintf(stderr, "[stream] gpu: chunk %zu planned %.2f ms, kernels done %.2f ms\n", i, pa, ka);
                cudaEventDestroy(tl[i].first);
                cudaEventDestroy(tl[i].second);
            }
            for (size_t i = 0; i < tc.size(); ++i) {
                float ca = 0;
                cudaEventElapsedTime(&ca, tl0, tc[i].first);
                std::fprintf(stderr, "[stream] gpu: chunk %zu uploaded %.2f ms (%.1f MB)\n", i, ca, tc[i].second / 1e6);
                cudaEventDestroy(tc[i].first);
            }
            cudaEventDestroy(tl0);
        }
        std::memcpy(out, h_res, npairs * 4);
    } catch (...) {
        drain();
        throw;
    }
    drain();
}

}  // namespace dm

extern "C" int dm_lev_pairs_packed(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint64_t npairs,
                                   uint32_t* out, dm_stats* st) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && offsets && (out || npairs == 0), "null argument");
        cudaEvent_t t0, t1;
        DM_CUDA(cudaEventCreate(&t0));
        DM_CUDA(cudaEventCreate(&t1));
        DM_CUDA(cudaEventRecord(t0, ctx->stream));
        dm::LevTotals tot;
        dm::lev_pairs_packed(ctx, data, offsets, npairs, out, &tot, false);
        DM_CUDA(cudaEventRecord(t1, ctx->stream));
        DM_CUDA(cudaEventSynchronize(t1));
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->total_ms = ms;
            st->cells = tot.cells;
            st->cells_executed = tot.cells_exec;
            st->launches = tot.launches;
        }
    });
}
