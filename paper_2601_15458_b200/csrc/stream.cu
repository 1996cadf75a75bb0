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
//
// PCIe is the end-to-end bound of the raw bytes (2 GB per cfg1 batch), so a
// packer thread feeds the copy stream: a chunk that holds only A/C/G/T bytes
// is packed by the host pool, sequence by sequence, straight into the
// sequence set's 2-bit code layout (code_bytes()) in a pinned slot; a quarter
// of the bytes cross the bus and the uploaded buffer IS the chunk's code
// buffer. Knowing the alphabet and the lengths, that chunk's planner skips
// both host syncs (codes A0 C1 G2 T3; bucket histogram counted on the host,
// plan_hist_host) and has no recode pass. Any other chunk is uploaded as
// given and planned as before. DM_STREAM_PACK_FRAC < 1 packs only the head
// of each chunk (flat, expanded by unpack_acgt next to the raw tail), for
// hosts whose packing rate is below the bus rate.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "capi_guard.h"
#include "host_pack.h"

namespace dm {
namespace {

__global__ void iota_pairs(uint32_t* ia, uint32_t* ib, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        ia[i] = (uint32_t)(2 * i);
        ib[i] = (uint32_t)(2 * i + 1);
    }
}

// 4 codes (one packed byte) -> 4 residue bytes: the codes are PRMT selectors
// into the word "ACGT".
__device__ __forceinline__ uint32_t expand4(uint32_t b) {
    const uint32_t sel = (b & 3u) | ((b & 0xcu) << 2) | ((b & 0x30u) << 4) | ((b & 0xc0u) << 6);
    return __byte_perm(0x54474341u, 0u, sel);
}

// n residues from 2-bit codes (host_pack.h layout) back to bytes; 16
// residues (one 32-bit load, one 16-byte store) per thread.
__global__ void unpack_acgt(const uint32_t* __restrict__ src, uint64_t n, uint8_t* __restrict__ dst) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, groups = n / 16;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const uint32_t w = src[g];
        reinterpret_cast<uint4*>(dst)[g] =
            make_uint4(expand4(w & 0xffu), expand4((w >> 8) & 0xffu), expand4((w >> 16) & 0xffu), expand4(w >> 24));
    }
    if (blockIdx.x == 0 && threadIdx.x < n % 16) {
        const uint64_t j = groups * 16 + threadIdx.x;
        const uint32_t b = reinterpret_cast<const uint8_t*>(src)[j / 4];
        dst[j] = (uint8_t)(0x54474341u >> (8 * ((b >> (2 * (j % 4))) & 3u)));
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
    cudaEvent_t copied[NB] = {}, planned[NB] = {}, done[NB] = {}, ready = nullptr;
    ChunkEvents() {
        for (int b = 0; b < NB; ++b)
            for (cudaEvent_t* e : {&copied[b], &planned[b], &done[b]})
                DM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        DM_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    }
    ~ChunkEvents() {
        for (int b = 0; b < NB; ++b)
            for (cudaEvent_t e : {copied[b], planned[b], done[b]})
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
    if (const char* env = std::getenv("DM_STREAM_BIG_MB")) big = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10)) << 20;
    if (const char* env = std::getenv("DM_STREAM_SMALL_MB")) small = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10)) << 20;
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
    if (!ctx->copy_stream) {  // high priority: the unpack kernels take the first SM slots the distance kernels free
        int least = 0, greatest = 0;
        DM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        DM_CUDA(cudaStreamCreateWithPriority(&ctx->copy_stream, cudaStreamNonBlocking, greatest));
    }
    dm_ctx* prep[NB];
    for (int b = 0; b < NB; ++b) prep[b] = prep_context(ctx, b);
    ChunkEvents ev;
    dm_seqset* live[NB] = {};
    const bool trace = std::getenv("DM_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tl;
    std::vector<std::pair<cudaEvent_t, uint64_t>> tc;
    std::vector<cudaEvent_t> th;  // trace: residue bytes landed (before the unpack)
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
    // Hand-off between the packer thread (uploads) and this thread (planning,
    // kernels): chunk c may be planned once issued > c; chunk c + NB may be
    // uploaded into slot c % NB once launched > c, behind ev.done of chunk c
    // (a packed chunk's upload buffer is its code buffer, read by its kernels).
    struct Handoff {
        std::mutex mu;
        std::condition_variable cv;
        uint64_t issued = 0, launched = 0;
        bool abort = false;
        std::exception_ptr err;
    } hs;
    std::thread packer;
    auto stop_packer = [&] {
        if (!packer.joinable()) return;
        {
            std::lock_guard<std::mutex> g(hs.mu);
            hs.abort = true;
        }
        hs.cv.notify_all();
        packer.join();
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
        const char* pk = std::getenv("DM_STREAM_PACK");
        const bool pack = !(pk && pk[0] == '0');
        // per-sequence 2-bit layout (code_bytes): < L / 4 + 32 bytes per sequence
        const uint64_t packed_cap = maxbytes / 4 + 32 * (2 * per) + 64;
        uint8_t* d_pack[NB] = {};
        uint8_t* h_pack[NB] = {};
        if (pack)
            for (int b = 0; b < NB; ++b) {
                d_pack[b] = (uint8_t*)ctx->stage_packed[b].get(packed_cap);
                h_pack[b] = (uint8_t*)ctx->pin_pack[b].get(packed_cap);
            }
        const int grid = (int)std::min<uint64_t>((per + 255) / 256, (uint64_t)ctx->sm_count * 4);
        iota_pairs<<<std::max(grid, 1), 256, 0, ctx->stream>>>(d_ab, d_ab + per, per);
        DM_CUDA(cudaGetLastError());
        DM_CUDA(cudaEventRecord(ev.ready, ctx->stream));
        DM_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev.ready, 0));
        cudaEvent_t h2d_done[NB] = {};  // slot's pinned buffers read by the copy engine
        for (int b = 0; b < NB; ++b) DM_CUDA(cudaEventCreateWithFlags(&h2d_done[b], cudaEventDisableTiming));
        struct EvGuard {
            cudaEvent_t* e;
            ~EvGuard() {
                for (int b = 0; b < NB; ++b) cudaEventDestroy(e[b]);
            }
        } evg{h2d_done};
        uint64_t h2d_bytes = 0;
        std::vector<char> acgt(nchunks, 0);  // chunk c went up fully packed (set before issued > c)
        // Share of each chunk that is packed on the host (default all of it);
        // with f < 1 the rest goes up raw while the host packs (pack rate P,
        // bus rate B: f/P = (1 - 3f/4)/B balances them). Only a fully packed
        // chunk is known to be A/C/G/T, which lets its planner skip both host
        // syncs (census and bucket histogram).
        double frac = 1.0;
        if (const char* e = std::getenv("DM_STREAM_PACK_FRAC")) frac = std::min(1.0, std::max(0.0, std::atof(e)));
        auto issue_copy = [&](uint64_t c) {
            const int b = (int)(c % NB);
            const uint64_t lo = cb[c], hi = cb[c + 1];
            const uint64_t a0 = offsets[2 * lo], a1 = offsets[2 * hi], n = a1 - a0;
            if (c >= NB) DM_CUDA(cudaEventSynchronize(h2d_done[b]));  // slot's pinned buffers free
            // chunk offsets go up from a pinned slot (a pageable copy would block
            // the host behind the bulk upload already queued)
            std::memcpy(h_offs + b * oslot, offsets + 2 * lo, (2 * (hi - lo) + 1) * 8);
            if (c >= NB) {  // slot b's device buffers are free once chunk c - NB's kernels are done
                std::unique_lock<std::mutex> g(hs.mu);
                hs.cv.wait(g, [&] { return hs.abort || hs.launched > c - NB; });
                if (hs.abort) return false;
                DM_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev.done[b], 0));
            }
            DM_CUDA(cudaMemcpyAsync(d_offs + b * oslot, h_offs + b * oslot, (2 * (hi - lo) + 1) * 8,
                                    cudaMemcpyHostToDevice, ctx->copy_stream));
            h2d_bytes += (2 * (hi - lo) + 1) * 8;
            // head [0, m) packed, tail [m, n) raw; the tail's upload runs while the head is packed
            uint64_t m = !pack || n < 256 ? 0 : (frac >= 1.0 ? n : (uint64_t)(frac * (double)n) / 128 * 128);
            if (m < n) {
                DM_CUDA(cudaMemcpyAsync(stage[b] + m, data + a0 + m, n - m, cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d_bytes += n - m;
            }
            const double tp0 = trace ? now_ms() : 0.0;
            uint64_t pb = 0;  // packed bytes to upload
            bool packed = false;
            if (m == n && m > 0) {  // whole chunk: straight into the set's 2-bit code layout
                // (one upload per chunk: uploading pieces while packing measured slower,
                // the copy engine's host reads compete with the packers)
                packed = pack_acgt_seqs(data, offsets + 2 * lo, 2 * (hi - lo), h_pack[b], &pb);
            } else if (m > 0) {     // head only: flat 2-bit stream, expanded next to the raw tail
                packed = pack_acgt((const uint8_t*)data + a0, m, h_pack[b]);
                pb = (m + 15) / 16 * 4;
            }
            if (trace)
                std::fprintf(stderr, "[pack] chunk %llu: %.1f MB packed %.2f..%.2f ms\n", (unsigned long long)c, m / 1e6,
                             tp0, now_ms());
            acgt[c] = packed && m == n;
            if (packed) {
                DM_CUDA(cudaMemcpyAsync(d_pack[b], h_pack[b], pb, cudaMemcpyHostToDevice, ctx->copy_stream));
                DM_CUDA(cudaEventRecord(h2d_done[b], ctx->copy_stream));
                if (trace) {
                    cudaEvent_t e;
                    cudaEventCreate(&e);
                    cudaEventRecord(e, ctx->copy_stream);
                    th.push_back(e);
                }
                if (m < n) {
                    const int ug = (int)std::min<uint64_t>((m / 16 + 255) / 256 + 1, (uint64_t)ctx->sm_count * 8);
                    unpack_acgt<<<ug, 256, 0, ctx->copy_stream>>>((const uint32_t*)d_pack[b], m, stage[b]);
                    DM_CUDA(cudaGetLastError());
                }  // else d_pack[b] is the chunk's code buffer as it stands
                h2d_bytes += pb;
            } else {
                if (m) DM_CUDA(cudaMemcpyAsync(stage[b], data + a0, m, cudaMemcpyHostToDevice, ctx->copy_stream));
                DM_CUDA(cudaEventRecord(h2d_done[b], ctx->copy_stream));
                h2d_bytes += m;
            }
            DM_CUDA(cudaEventRecord(ev.copied[b], ctx->copy_stream));
            if (trace) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, ctx->copy_stream);
                tc.push_back({e, packed ? pb + (n - m) : n});
            }
            return true;
        };
        packer = std::thread([&] {
            try {
                DM_CUDA(cudaSetDevice(ctx->device));
                for (uint64_t c = 0; c < nchunks; ++c) {
                    if (!issue_copy(c)) return;
                    {
                        std::lock_guard<std::mutex> g(hs.mu);
                        hs.issued = c + 1;
                    }
                    hs.cv.notify_all();
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(hs.mu);
                hs.err = std::current_exception();
                hs.abort = true;
            }
            hs.cv.notify_all();
        });
        for (uint64_t c = 0; c < nchunks; ++c) {
            const int b = (int)(c % NB);
            dm_ctx* P = prep[b];
            const uint64_t lo = cb[c], hi = cb[c + 1], cnt = hi - lo;
            {
                std::unique_lock<std::mutex> g(hs.mu);
                hs.cv.wait(g, [&] { return hs.abort || hs.issued > c; });
                if (hs.err) std::rethrow_exception(hs.err);
                if (hs.issued <= c) throw cuda_error("streamed upload stopped");
            }
            DM_CUDA(cudaStreamWaitEvent(P->stream, ev.copied[b], 0));
            if (c >= NB) DM_CUDA(cudaStreamWaitEvent(P->stream, ev.done[b], 0));  // chunk c-NB's kernels
            delete live[b];  // stream-ordered frees behind that wait
            live[b] = nullptr;
            // census + recode + bit-planes on the planner stream (one host sync)
            const double t0 = trace ? now_ms() : 0.0;
            live[b] = seqset_create_device(P, stage[b], d_offs + b * oslot, offsets + 2 * lo, (uint32_t)(2 * cnt),
                                           acgt[c] != 0, acgt[c] ? d_pack[b] : nullptr);
            const double t1 = trace ? now_ms() : 0.0;
            // plan on the planner stream, kernels on ctx->stream
            lev_plan_then_launch(P, ctx, live[b], d_ab, d_ab + per, cnt, d_res + lo, ev.planned[b], tot,
                                 acgt[c] ? offsets + 2 * lo : nullptr);
            DM_CUDA(cudaEventRecord(ev.done[b], ctx->stream));
            {
                std::lock_guard<std::mutex> g(hs.mu);
                hs.launched = c + 1;
            }
            hs.cv.notify_all();
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
        packer.join();
        if (hs.err) std::rethrow_exception(hs.err);
        DM_CUDA(cudaMemcpyAsync(h_res, d_res, npairs * 4, cudaMemcpyDeviceToHost, ctx->stream));
        DM_CUDA(cudaStreamSynchronize(ctx->stream));
        if (tot) {
            tot->h2d_bytes += h2d_bytes;
            tot->d2h_bytes += npairs * 4;
        }
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
                float ha = -1;
                if (i < th.size()) {
                    cudaEventElapsedTime(&ha, tl0, th[i]);
                    cudaEventDestroy(th[i]);
                }
                std::fprintf(stderr, "[stream] gpu: chunk %zu h2d done %.2f ms, uploaded %.2f ms (%.1f MB)\n", i, ha, ca,
                             tc[i].second / 1e6);
                cudaEventDestroy(tc[i].first);
            }
            cudaEventDestroy(tl0);
        }
        std::memcpy(out, h_res, npairs * 4);
    } catch (...) {
        stop_packer();
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
            st->h2d_bytes = tot.h2d_bytes;
            st->d2h_bytes = tot.d2h_bytes;
        }
    });
}

extern "C" int dm_pack_nt_seqs(const char* data, const uint64_t* offsets, uint64_t n, uint8_t* dst,
                               uint64_t* bytes) {
    return dm::guard([&] {
        dm::require(offsets && bytes && (data || n == 0) && (dst || n == 0), "null argument");
        dm::require(((uintptr_t)dst & 31) == 0, "dst must be 32-byte aligned");
        for (uint64_t i = 0; i < n; ++i)
            if (offsets[i + 1] < offsets[i]) throw dm::invalid_argument("sequence offsets must be non-decreasing");
        if (!dm::pack_acgt_seqs(data, offsets, n, dst, bytes))
            throw dm::invalid_argument("not a nucleotide (A/C/G/T) buffer");
    });
}

extern "C" int dm_pack_nt(const char* src, uint64_t n, uint8_t* dst) {
    return dm::guard([&] {
        dm::require(src || n == 0, "null argument");
        dm::require(dst || n == 0, "null argument");
        if (!dm::pack_acgt(reinterpret_cast<const uint8_t*>(src), n, dst))
            throw dm::invalid_argument("not a nucleotide (A/C/G/T) buffer");
    });
}
