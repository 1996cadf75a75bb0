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
// plan_hist_host) and has no recode pass. Packing is bound by host memory
// bandwidth, which the copy engine can add to: with a pinned caller buffer,
// ~30 % of the bytes go up raw instead ("speculative" chunks), planned as
// A/C/G/T like packed ones and checked on the device (verify_acgt_kernel);
// a chunk that fails is recomputed on the exact path before the call
// returns. Any other chunk is uploaded as given and planned with the device
// census. DM_STREAM_PACK=0 / DM_STREAM_RAW_FRAC=x override the mix.
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
#include "nvtx.h"

namespace dm {
namespace {

__global__ void iota_pairs(uint32_t* ia, uint32_t* ib, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        ia[i] = (uint32_t)(2 * i);
        ib[i] = (uint32_t)(2 * i + 1);
    }
}

// Speculative chunks: flag = 1 if any of the n bytes is not A, C, G or T.
__global__ void verify_acgt_kernel(const uint8_t* __restrict__ raw, uint64_t n, uint32_t* __restrict__ flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, words = n / 16;
    bool bad = false;
    auto check4 = [](uint32_t x) {
        const uint32_t ok = __vcmpeq4(x, 0x41414141u) | __vcmpeq4(x, 0x43434343u) | __vcmpeq4(x, 0x47474747u) |
                            __vcmpeq4(x, 0x54545454u);
        return ok != 0xffffffffu;
    };
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) {
        const uint4 v = reinterpret_cast<const uint4*>(raw)[i];
        bad |= check4(v.x) | check4(v.y) | check4(v.z) | check4(v.w);
    }
    if (blockIdx.x == 0 && threadIdx.x < n % 16) {
        const uint8_t c = raw[words * 16 + threadIdx.x];
        bad |= !(c == 'A' || c == 'C' || c == 'G' || c == 'T');
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

namespace {

dm_ctx* prep_context(dm_ctx* ctx, int k) {
    if (!ctx->prep[k]) {
        auto* p = new dm_ctx;
        p->device = ctx->device;
        p->sm_count = ctx->sm_count;
        p->lev_wmax_cap = 16;
        if (const char* e = std::getenv("DM_STREAM_WSEL")) p->lev_wmax_cap = std::max(1, std::atoi(e));
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
                      LevTotals* tot, bool speculate, std::vector<std::pair<uint64_t, uint64_t>>* redo) {
    if (npairs == 0) return;
    NvtxRange nvtx_stream("dm streamed pair batch");
    if (2 * npairs > 0xffffffffull) throw invalid_argument("too many sequences in one streamed batch");
    for (uint64_t i = 0; i < 2 * npairs; ++i)
        if (offsets[i + 1] < offsets[i]) throw invalid_argument("sequence offsets must be non-decreasing");
    // Chunk boundaries (pair indices). Sizes ramp up from `small` to `big`
    // residue bytes so the first kernels start after a short upload, and
    // halve again over the tail so little compute is left once the last
    // upload lands.
    // 128 MB chunks and raw (speculative) chunks of at most 32 MB: the copy
    // engine alternates short raw uploads with the packed ones, so the GPU is
    // fed early (measured 27.1 vs 28.1 ms per cfg1 step at 256 / 128 MB,
    // tools/sweep_stream.sh)
    uint64_t big = 128ull << 20, small = 32ull << 20;
    if (const char* env = std::getenv("DM_STREAM_CHUNK_BYTES"))
        big = small = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10));
    if (const char* env = std::getenv("DM_STREAM_BIG_MB")) big = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10)) << 20;
    if (const char* env = std::getenv("DM_STREAM_SMALL_MB")) small = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10)) << 20;
    const char* pk = std::getenv("DM_STREAM_PACK");
    const bool pack = !(pk && pk[0] == '0');
    // Share of the residue bytes sent raw (speculative chunks, see the top):
    // the copy engine reads them from host memory while the host threads
    // pack the rest, which uses host memory bandwidth better than packing
    // everything (measured on the box: pack alone ~100 GB/s; pack + raw copy
    // 82 + 54 GB/s); at ~0.3 the bus and the packers finish together. Needs
    // a pinned `data`.
    double raw_frac = 0.0;
    if (speculate && pack) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, data) == cudaSuccess && pa.type == cudaMemoryTypeHost) raw_frac = 0.3;
        cudaGetLastError();
        if (const char* e = std::getenv("DM_STREAM_RAW_FRAC")) raw_frac = std::min(1.0, std::max(0.0, std::atof(e)));
    }
    // Raw chunks are small (DM_STREAM_RAW_MB): a raw chunk's upload (4x the
    // bytes of a packed one) should not hold the copy engine while packed
    // chunks wait.
    uint64_t raw_cap = 32ull << 20;
    if (const char* env = std::getenv("DM_STREAM_RAW_MB")) raw_cap = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10)) << 20;
    std::vector<uint64_t> cb{0};
    std::vector<char> spec;  // chunk k goes up raw (speculative)
    uint64_t raw_sofar = 0, all_sofar = 0;
    for (uint64_t lo = 0, k = 0; lo < npairs; ++k) {
        const uint64_t rem = offsets[2 * npairs] - offsets[2 * lo];
        uint64_t t = std::min(big, small << std::min<uint64_t>(k, 20));
        if (rem < 2 * t) t = std::max(small, rem / 2);
        const bool raw = (double)raw_sofar < raw_frac * (double)(all_sofar + t);
        if (raw) t = std::max<uint64_t>(std::min(t, raw_cap), 1);
        // smallest hi > lo with offsets[2hi] - offsets[2lo] >= t
        uint64_t a = lo + 1, z = npairs;
        while (a < z) {
            const uint64_t mid = (a + z) / 2;
            if (offsets[2 * mid] - offsets[2 * lo] >= t) z = mid; else a = mid + 1;
        }
        const uint64_t n = offsets[2 * a] - offsets[2 * lo];
        all_sofar += n;
        if (raw && n > 0) raw_sofar += n;
        spec.push_back(raw && n > 0);
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
    if (!ctx->copy_stream) {  // high priority, like the planners
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
    std::vector<cudaEvent_t> th;  // trace: residue bytes landed
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
        uint64_t issued = 0, launched = 0, planned = 0;
        bool abort = false;
        std::exception_ptr err;
    } hs;
    std::thread packer, planner;
    auto stop_packer = [&] {
        if (!packer.joinable() && !planner.joinable()) return;
        {
            std::lock_guard<std::mutex> g(hs.mu);
            hs.abort = true;
        }
        hs.cv.notify_all();
        if (packer.joinable()) packer.join();
        if (planner.joinable()) planner.join();
    };
    try {
        // every buffer the side streams touch is (re)allocated on ctx->stream first
        uint8_t* stage[NB];
        // +64: the raw-byte kernels read whole aligned words past a sequence's end
        for (int b = 0; b < NB; ++b) stage[b] = (uint8_t*)ctx->stage[b].get(maxbytes + 64);
        uint64_t* d_offs = ctx->stream_offs.as<uint64_t>(NB * oslot);
        uint64_t* h_offs = ctx->pin_items.as<uint64_t>(NB * oslot);
        uint32_t* d_ab = ctx->stream_pairs.as<uint32_t>(2 * per + 2);
        uint32_t* d_res = ctx->stream_out.as<uint32_t>(npairs);
        uint32_t* h_res = ctx->pin_out.as<uint32_t>(npairs);
        uint32_t* d_flags = ctx->stream_flags.as<uint32_t>(nchunks);  // speculative chunk c held a non-ACGT byte
        DM_CUDA(cudaMemsetAsync(d_flags, 0, nchunks * 4, ctx->stream));
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
        // Host-planned chunks (packed or speculative, all pairs within one
        // pass): the host orients, buckets and sorts the pairs and lays out
        // the chunk's per-sequence offsets and lengths; the plan goes up on the
        // copy stream just before the chunk's residues, and the chunk's
        // kernels (2-bit code / raw byte sources) wait only for the upload --
        // no planner kernels, no host sync. Plan slot layout: per-bucket
        // counters (zero) | items | lengths | offsets.
        constexpr uint64_t kPlanHead = 1024;
        static_assert(kLevBuckets * 4 <= kPlanHead, "plan header");
        auto plan_layout = [](uint64_t cnt, uint64_t& len_at, uint64_t& off_at) {
            len_at = kPlanHead + cnt * sizeof(LevItem);
            off_at = len_at + ((2 * cnt * 4 + 7) & ~uint64_t(7));
            return off_at + 2 * cnt * 8;
        };
        uint64_t l_at = 0, o_at = 0;
        const uint64_t plan_cap = plan_layout(per, l_at, o_at);
        uint8_t* d_plan[NB];
        uint8_t* h_plan[NB];
        for (int b = 0; b < NB; ++b) {
            d_plan[b] = (uint8_t*)ctx->stage_plan[b].get(plan_cap);
            h_plan[b] = (uint8_t*)ctx->pin_plan[b].get(plan_cap);
        }
        const bool host_plan = [] {
            const char* e = std::getenv("DM_STREAM_HOSTPLAN");
            return !(e && e[0] == '0');
        }();
        const int hwsel = [] {
            const char* e = std::getenv("DM_STREAM_HWSEL");
            return e ? std::max(1, std::atoi(e)) : 16;
        }();
        std::vector<char> hp_ok(nchunks, 0);
        std::vector<uint64_t> hp_bytes(nchunks, 0);
        std::vector<unsigned int> hp_hist(nchunks * kLevBuckets);
        std::vector<unsigned long long> hp_cells(2 * nchunks);
        std::vector<uint32_t> hp_tmp;
        cudaEvent_t plan_up[NB] = {};  // slot's pinned plan read by the copy engine
        for (int b = 0; b < NB; ++b) DM_CUDA(cudaEventCreateWithFlags(&plan_up[b], cudaEventDisableTiming));
        EvGuard evp{plan_up};
        auto plan_chunk = [&](uint64_t p) {  // planner thread, ahead of the packer
            NvtxRange nvtx_plan("dm host plan");
            const int b = (int)(p % NB);
            if (p >= NB) {  // chunk p - NB's plan has gone up from this slot
                {
                    std::unique_lock<std::mutex> g(hs.mu);
                    hs.cv.wait(g, [&] { return hs.abort || hs.issued > p - NB; });
                    if (hs.abort) return false;
                }
                DM_CUDA(cudaEventSynchronize(plan_up[b]));
            }
            const uint64_t lo = cb[p], hi = cb[p + 1], cnt = hi - lo;
            if (host_plan && (spec[p] || pack) && cnt > 0) {
                uint8_t* hb = h_plan[b];
                uint64_t la = 0, oa = 0;
                const uint64_t bytes = plan_layout(cnt, la, oa);
                std::memset(hb, 0, kPlanHead);
                if (lev_plan_host_pairs(offsets + 2 * lo, cnt, lo, ctx->sm_count, hwsel,
                                        reinterpret_cast<LevItem*>(hb + kPlanHead), &hp_hist[p * kLevBuckets],
                                        &hp_cells[2 * p], hp_tmp)) {
                    uint32_t* ln = reinterpret_cast<uint32_t*>(hb + la);
                    uint64_t* of = reinterpret_cast<uint64_t*>(hb + oa);
                    const uint64_t* o = offsets + 2 * lo;
                    uint64_t at = 0;
                    for (uint64_t k = 0; k < 2 * cnt; ++k) {
                        const uint64_t L = o[k + 1] - o[k];
                        ln[k] = (uint32_t)L;
                        if (spec[p]) {
                            of[k] = o[k] - o[0];  // raw bytes as uploaded
                        } else {
                            of[k] = at;  // host_pack.cpp's 2-bit layout
                            at += code_bytes(L, 2);
                        }
                    }
                    hp_ok[p] = 1;
                    hp_bytes[p] = bytes;
                }
            }
            {
                std::lock_guard<std::mutex> g(hs.mu);
                hs.planned = p + 1;
            }
            hs.cv.notify_all();
            return true;
        };
        // Chunk kinds (set before issued > c): kPacked — packed on the host,
        // the upload is its code buffer; kSpec — uploaded raw from the
        // caller's pinned buffer and planned as A/C/G/T, verified on the
        // device (a failed chunk is recomputed by the caller, see `redo`);
        // kRaw — uploaded raw, alphabet from the device census.
        enum : char { kRaw = 0, kPacked = 1, kSpec = 2 };
        std::vector<char> kind(nchunks, kRaw);
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
            const double tp0 = trace ? now_ms() : 0.0;
            bool pack_ok = false;
            uint64_t pb = 0;  // packed bytes
            if (spec[c]) {
                kind[c] = kSpec;
            } else if (pack && n >= 256 && (nvtxRangePushA("dm pack chunk"),
                                            pack_ok = pack_acgt_seqs(data, offsets + 2 * lo, 2 * (hi - lo), h_pack[b], &pb),
                                            nvtxRangePop(), pack_ok)) {
                kind[c] = kPacked;  // straight into the set's 2-bit code layout
            }
            if (trace)
                std::fprintf(stderr, "[pack] chunk %llu: %.1f MB kind %d %.2f..%.2f ms\n", (unsigned long long)c, n / 1e6,
                             (int)kind[c], tp0, now_ms());
            if (kind[c] == kPacked) {  // one upload per chunk: uploading pieces while packing measured slower
                DM_CUDA(cudaMemcpyAsync(d_pack[b], h_pack[b], pb, cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d_bytes += pb;
            } else {
                if (n) DM_CUDA(cudaMemcpyAsync(stage[b], data + a0, n, cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d_bytes += n;
            }
            DM_CUDA(cudaEventRecord(h2d_done[b], ctx->copy_stream));
            {  // chunk c's host plan goes up behind its residues (the main thread plans ahead)
                std::unique_lock<std::mutex> g(hs.mu);
                hs.cv.wait(g, [&] { return hs.abort || hs.planned > c; });
                if (hs.abort) return false;
            }
            if (hp_ok[c]) {
                DM_CUDA(cudaMemcpyAsync(d_plan[b], h_plan[b], hp_bytes[c], cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d_bytes += hp_bytes[c];
            }
            DM_CUDA(cudaEventRecord(plan_up[b], ctx->copy_stream));
            if (trace) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, ctx->copy_stream);
                th.push_back(e);
            }
            DM_CUDA(cudaEventRecord(ev.copied[b], ctx->copy_stream));
            if (trace) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, ctx->copy_stream);
                tc.push_back({e, kind[c] == kPacked ? pb : n});
            }
            return true;
        };
        planner = std::thread([&] {
            try {
                DM_CUDA(cudaSetDevice(ctx->device));
                for (uint64_t p = 0; p < nchunks; ++p)
                    if (!plan_chunk(p)) return;
            } catch (...) {
                std::lock_guard<std::mutex> g(hs.mu);
                if (!hs.err) hs.err = std::current_exception();
                hs.abort = true;
            }
            hs.cv.notify_all();
        });
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
                if (!hs.err) hs.err = std::current_exception();
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
            if (kind[c] != kRaw && hp_ok[c]) {
                // host-planned: the kernels wait for the upload alone
                const double t0 = trace ? now_ms() : 0.0;
                uint64_t la = 0, oa = 0;
                plan_layout(cnt, la, oa);
                if (kind[c] == kSpec) {  // the A/C/G/T assumption, checked on the device
                    DM_CUDA(cudaStreamWaitEvent(P->stream, ev.copied[b], 0));
                    const uint64_t nb = offsets[2 * hi] - offsets[2 * lo];
                    const int vg = (int)std::min<uint64_t>((nb + 4095) / 4096 + 1, (uint64_t)ctx->sm_count * 8);
                    verify_acgt_kernel<<<vg, 256, 0, P->stream>>>(stage[b], nb, d_flags + c);
                    DM_CUDA(cudaGetLastError());
                    DM_CUDA(cudaEventRecord(ev.planned[b], P->stream));
                }
                const int nl = lev_launch_host_planned(
                    ctx, reinterpret_cast<const LevItem*>(d_plan[b] + kPlanHead), reinterpret_cast<uint32_t*>(d_plan[b]),
                    &hp_hist[c * kLevBuckets], kind[c] == kPacked ? kLevSrcCodes : kLevSrcRaw,
                    kind[c] == kPacked ? d_pack[b] : stage[b], reinterpret_cast<const uint64_t*>(d_plan[b] + oa),
                    reinterpret_cast<const uint32_t*>(d_plan[b] + la), d_res, ev.copied[b]);
                // the slot's buffers are reused once its kernels (and check) are done
                if (kind[c] == kSpec) DM_CUDA(cudaStreamWaitEvent(ctx->stream, ev.planned[b], 0));
                DM_CUDA(cudaEventRecord(ev.done[b], ctx->stream));
                if (tot) {
                    tot->cells += hp_cells[2 * c];
                    tot->cells_exec += hp_cells[2 * c + 1];
                    tot->launches += nl + (kind[c] == kSpec ? 1 : 0);
                }
                {
                    std::lock_guard<std::mutex> g(hs.mu);
                    hs.launched = c + 1;
                }
                hs.cv.notify_all();
                if (trace) {
                    cudaEvent_t a, k;
                    cudaEventCreate(&a);
                    cudaEventCreate(&k);
                    cudaEventRecord(a, ctx->copy_stream);
                    cudaEventRecord(k, ctx->stream);
                    tl.push_back({a, k});
                    std::fprintf(stderr, "[stream] chunk %llu pairs %llu: host-planned kind %d, launched %.2f..%.2f ms\n",
                                 (unsigned long long)c, (unsigned long long)cnt, (int)kind[c], t0, now_ms());
                }
                continue;
            }
            DM_CUDA(cudaStreamWaitEvent(P->stream, ev.copied[b], 0));
            if (c >= NB) DM_CUDA(cudaStreamWaitEvent(P->stream, ev.done[b], 0));  // chunk c-NB's kernels
            delete live[b];  // stream-ordered frees behind that wait
            live[b] = nullptr;
            // census + recode + bit-planes on the planner stream (one host sync)
            const double t0 = trace ? now_ms() : 0.0;
            const bool known = kind[c] != kRaw;  // alphabet known (packed) or assumed (speculative)
            live[b] = seqset_create_device(P, stage[b], d_offs + b * oslot, offsets + 2 * lo, (uint32_t)(2 * cnt),
                                           known, kind[c] == kPacked ? d_pack[b] : nullptr);
            if (kind[c] == kSpec) {  // the assumption, checked on the device
                const uint64_t nb = offsets[2 * hi] - offsets[2 * lo];
                const int vg = (int)std::min<uint64_t>((nb + 4095) / 4096 + 1, (uint64_t)ctx->sm_count * 8);
                verify_acgt_kernel<<<vg, 256, 0, P->stream>>>(stage[b], nb, d_flags + c);
                DM_CUDA(cudaGetLastError());
            }
            const double t1 = trace ? now_ms() : 0.0;
            // plan on the planner stream, kernels on ctx->stream
            lev_plan_then_launch(P, ctx, live[b], d_ab, d_ab + per, cnt, d_res + lo, ev.planned[b], tot,
                                 known ? offsets + 2 * lo : nullptr);
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
        planner.join();
        if (hs.err) std::rethrow_exception(hs.err);
        DM_CUDA(cudaMemcpyAsync(h_res, d_res, npairs * 4, cudaMemcpyDeviceToHost, ctx->stream));
        std::vector<uint32_t> flags(nchunks);
        DM_CUDA(cudaMemcpyAsync(flags.data(), d_flags, nchunks * 4, cudaMemcpyDeviceToHost, ctx->stream));
        DM_CUDA(cudaStreamSynchronize(ctx->stream));
        for (uint64_t c = 0; c < nchunks; ++c)
            if (flags[c]) {
                if (!redo) throw cuda_error("internal error: unverified chunk without a redo list");
                redo->push_back({cb[c], cb[c + 1]});
            }
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
        std::vector<std::pair<uint64_t, uint64_t>> redo;
        dm::lev_pairs_packed(ctx, data, offsets, npairs, out, &tot, true, &redo);
        // speculative chunks that turned out not to be A/C/G/T only: again,
        // on the exact path (rare; results overwritten in place)
        for (const auto& r : redo) {
            dm::LevTotals again;  // the cells were counted once already; the extra traffic is real
            dm::lev_pairs_packed(ctx, data, offsets + 2 * r.first, r.second - r.first, out + r.first, &again, false,
                                 nullptr);
            tot.h2d_bytes += again.h2d_bytes;
            tot.d2h_bytes += again.d2h_bytes;
            tot.launches += again.launches;
        }
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
