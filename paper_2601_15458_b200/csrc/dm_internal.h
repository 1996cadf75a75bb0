// Internal declarations shared by the CUDA translation units of libdmb200.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dm_b200.h"

namespace dm {

// Internal errors are exceptions; capi.cpp maps them onto DM_* status codes.
struct invalid_argument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct runtime_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define DM_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::dm::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Growable device scratch buffer (never shrinks; reused across calls).
// Growable device scratch buffer (never shrinks; reused across calls).
// Stream-ordered on the owning context's stream (*sp) so growth never
// synchronises the device; the pool keeps freed blocks (dm_ctx_create).
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaStream_t* sp = nullptr;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) {
                if (sp) cudaFreeAsync(p, *sp);
                else cudaFree(p);
            }
            p = nullptr;
            size_t c = bytes + bytes / 4 + 256;
            if (sp) DM_CUDA(cudaMallocAsync(&p, c, *sp));
            else DM_CUDA(cudaMalloc(&p, c));
            cap = c;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
    // grow to exactly `bytes` (no slack): for large one-off reservations
    void reserve_exact(size_t bytes) {
        if (bytes <= cap) return;
        if (p) {
            if (sp) cudaFreeAsync(p, *sp);
            else cudaFree(p);
        }
        p = nullptr;
        if (sp) DM_CUDA(cudaMallocAsync(&p, bytes, *sp));
        else DM_CUDA(cudaMalloc(&p, bytes));
        cap = bytes;
    }
    DevBuf() = default;
    explicit DevBuf(cudaStream_t* s) : sp(s) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) {
            if (sp) cudaFreeAsync(p, *sp);
            else cudaFree(p);
        }
    }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            size_t c = bytes + bytes / 4 + 256;
            DM_CUDA(cudaMallocHost(&p, c));
            cap = c;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

}  // namespace dm

struct dm_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;      // stream every call is issued on
    cudaStream_t own_stream = nullptr;  // created by dm_ctx_create (null once replaced)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    uint64_t free_at_create = 0;  // device memory free when the context was created (sizes trace budgets)
    int rank = 0, world = 1;   // NCCL shard of this context (dm_ctx_attach_nccl)
    int sim_world = 1;         // >1: run the sharded path on this one GPU (tests)
    void* nccl = nullptr;      // ncclComm_t
    dm_allgather_fn host_allgather = nullptr;  // host-callback collectives (dm_ctx_attach_host_comm)
    void* host_comm_user = nullptr;
    dm::PinnedBuf* comm_pin = nullptr;         // staging for host-callback collectives
    // multi-rank counters (dm_ctx_comm_stats): collectives issued, bytes each
    // rank contributed, subtrees this rank owned in the tree / the merges
    uint64_t coll_calls = 0, coll_bytes = 0, own_tree = 0, own_msa = 0;
    // scratch for the distance engine
    dm::DevBuf items, out, counter, aux, aux2, aux3, lev_all, lev_items, comm_dev, shard_buf;
    // multi-pass distance jobs (lev.cu run_long): plain cudaMalloc (not
    // stream-ordered: they are used on the side streams)
    dm::DevBuf lev_long_off, lev_long_h;
    dm::PinnedBuf pin_long;
    cudaStream_t copy_stream = nullptr;  // host->device staging of streamed batches
    static constexpr int kStreamSlots = 6;  // chunks of a streamed batch in flight
    dm::DevBuf stage[kStreamSlots], stream_pairs, stream_out, stream_offs, stream_flags;
    dm::DevBuf stage_packed[kStreamSlots];  // 2-bit nucleotide chunks as uploaded
    dm::DevBuf ss_meta, ss_codes, ss_planes;  // planner contexts: the chunk's sequence set (reused)
    dm::PinnedBuf pin_pack[kStreamSlots];   // host side of the same
    dm::DevBuf stage_plan[kStreamSlots];    // host-planned chunks: counters, sorted items, lengths, offsets
    dm::PinnedBuf pin_plan[kStreamSlots];
    dm_ctx* prep[kStreamSlots] = {};  // planner contexts of the streamed path (own stream + scratch)
    // words per lane the lane count per pair is chosen for on this context
    // (0: the alphabet's maximum; patterns too long for it still use up to
    // the maximum); the streamed path's planners use 16 (DM_STREAM_WSEL) --
    // its chunks share the SMs with planning and uploads, where the
    // 2-block-per-SM kernels of 17-24 words measured slower end to end
    // (32.5 / 32.9 / 34.1 ms per cfg1 step at 16 / 20 / 24)
    int lev_wmax_cap = 0;
    static constexpr int kLevSide = 8;  // side streams the distance buckets fan out on
    int side_prio = 0;                  // their priority (dm_ctx_create: the greatest; 0 = default, the least)
    dm_ctx* tree_bg = nullptr;          // low-priority context for the tree's background batches (tree.cu)
    uint32_t lev_waves = 0;             // distance-kernel grids in waves of resident blocks (0: default 4)
    cudaStream_t lev_side[kLevSide] = {};
    int lev_rr = 0;
    cudaEvent_t lev_fork = nullptr, lev_join[kLevSide] = {};
    dm::PinnedBuf pin_items, pin_out;
    dm::PinnedBuf pin_stage;                 // host_copy.cpp: double buffer for pageable uploads
    cudaEvent_t stage_ev[2] = {};
    // scratch for the aligner / merge scheduler
    dm::DevBuf nw_in, nw_table, nw_jobs, nw_trace, nw_res, nw_gaps, nw_wrap, rows_a, rows_b, colmap, tree_buf,
        nw_seqtab, nw_shard, nw_shard_gaps;
    uint64_t launches = 0;
    // Every C ABI call on a context holds this lock (capi_guard.h), so one
    // context may be shared by host threads (the reference's functions are
    // reentrant and are called from parallel_for bodies).
    std::recursive_mutex mu;
    dm_ctx() { attach(&stream); }
    void detach_buffers() { attach(nullptr); }

private:
    void attach(cudaStream_t* s) {
        for (dm::DevBuf* b : {&items, &out, &counter, &aux, &aux2, &aux3, &lev_all, &lev_items, &comm_dev, &shard_buf,
                              &stream_pairs, &stream_out, &stream_offs, &stream_flags, &nw_in, &nw_table,
                              &nw_jobs, &nw_trace, &nw_wrap,
                              &nw_res, &nw_gaps, &rows_a, &rows_b, &colmap, &tree_buf, &nw_seqtab, &nw_shard, &nw_shard_gaps, &ss_meta,
                              &ss_codes,
                              &ss_planes})
            b->sp = s;
        for (dm::DevBuf& b : stage) b.sp = s;
        for (dm::DevBuf& b : stage_packed) b.sp = s;
        for (dm::DevBuf& b : stage_plan) b.sp = s;
    }
};

namespace dm {
// Bytes sequence i of length L occupies in a set's code buffer: with 2
// bit-planes (<= 4 symbols) the codes are stored 2 bits per residue, residue
// j at bits 2(j%16) of 32-bit word j/16, in whole 32-B blocks of 128 residues
// (zero past the end; the host packer writes each block with one aligned
// streaming store); otherwise one byte per residue in 16-B aligned runs with
// >= 1 pad byte. Host packer (host_pack.cpp), seqset builders and the
// distance kernel share this.
#if defined(__CUDACC__)
__host__ __device__
#endif
inline uint64_t code_bytes(uint64_t L, int planes) {
    return planes == 2 ? ((L + 127) >> 7) << 5 : (L + 16) & ~uint64_t(15);
}
}  // namespace dm

// Device-resident sequence store.
struct dm_seqset {
    dm_ctx* ctx = nullptr;
    uint32_t n = 0;
    int planes = 2;    // bit-planes per residue code: 2 (<=4 symbols), 5 (<=32), 8
    int nsym = 0;      // distinct residue bytes
    uint8_t code_of[256] = {};
    bool present[256] = {};  // bytes that occur in the set
    // host mirrors
    std::vector<uint32_t> len;     // residues per sequence
    std::vector<uint64_t> off;     // byte offset of sequence i in d_codes (16-B aligned)
    std::vector<uint64_t> blk_off; // first 64-row block of sequence i in d_planes
    std::vector<uint64_t> raw_off; // offset of sequence i in d_raw (as given by the caller)
    // device
    uint8_t* d_raw = nullptr;      // raw residue bytes (what NW scores and the MSA prints)
    bool owns_raw = true;
    uint64_t* d_raw_off = nullptr;
    uint8_t* d_codes = nullptr;    // dense codes 0..nsym-1, laid out by code_bytes()
    uint64_t* d_off = nullptr;
    uint32_t* d_len = nullptr;
    uint64_t* d_blk = nullptr;
    uint64_t* d_planes = nullptr; // [block][plane] 64-bit words
    uint64_t total_blocks = 0;
    bool owns_meta = true;        // false: the arrays above are a context's scratch (streamed chunks)
    ~dm_seqset();
};

// Result of align_all / dm_msa (host side).
struct dm_msa_out {
    uint64_t width = 0;
    uint64_t dev_pitch = 0;  // the rows also stay in ctx->rows_a at this pitch until the next call on ctx
    std::vector<char> rows;  // rows x width, tree order
    std::vector<uint32_t> row_seq;
    std::vector<dm_node> nodes;
    std::vector<uint32_t> order;
};

namespace dm {

// DM_TRACE_BYTES=1: one stderr line per launch of the memory-bound passes
// with its algorithmic bytes (read, written), matched against ncu's DRAM
// bytes by tools/prof_mem.py.
void trace_bytes(const char* kernel, uint64_t read, uint64_t written);

// Resident blocks per SM of `kern` at (threads, dynamic smem) on the current
// device, cached per (kernel, device, threads, smem) and thread-safe; opts the
// kernel into more than 48 KB of dynamic shared memory on that device when
// smem needs it (capi.cpp).
int occupancy(const void* kern, int threads, size_t smem);

struct NwScheme;

// One Levenshtein job: distance(seq pat, seq txt) -> out[slot].
struct LevItem {
    uint32_t pat;
    uint32_t txt;
    uint64_t slot;  // 64-bit: per-level candidate matrices can exceed 2^32 cells
};

// Device table of distances already computed in one guide-tree build
// (tree.cu): open addressing, key = min(a, b) << 32 | max(a, b) (sequence
// ids; Levenshtein is symmetric), linear probing. The tree asks for the same
// pair again across its phases -- a node's center is one of its median
// candidates, a child's median sample and a small subtree's all-pairs matrix
// overlap the parent's candidate matrix and pole sweeps -- and the planner
// answers those jobs (and a == b: 0) from here instead of launching them.
// Distances are deterministic, so a hit returns exactly what the kernel
// would. Lookups may run concurrently with inserts (the tree's background
// batches): a key whose value is still kCacheNone reads as a miss.
struct DistCache {
    unsigned long long* keys = nullptr;  // kCacheEmpty = free
    uint32_t* vals = nullptr;            // kCacheNone = not written yet
    unsigned int* fill = nullptr;        // inserted keys (device counter)
    uint64_t mask = 0;                   // capacity - 1 (power of two)
    unsigned int max_fill = 0;           // inserts stop here (load factor bound)
    bool insert = false;                 // this batch adds its results
    bool on() const { return keys != nullptr; }
};
constexpr unsigned long long kCacheEmpty = ~0ull;
constexpr uint32_t kCacheNone = 0xffffffffu;

struct LevTotals {
    uint64_t cells = 0, cells_exec = 0, launches = 0;
    uint64_t reused = 0, cells_reused = 0;  // jobs answered by a DistCache (or a == b)
    uint64_t h2d_bytes = 0, d2h_bytes = 0;  // streamed path: bytes actually copied
    float kernel_ms = 0.f;
    // timed batches whose event pairs are not read yet (no host sync per
    // batch): kernel_ms is complete after lev_finish_timing
    std::vector<cudaEvent_t> pend;
};
void lev_finish_timing(LevTotals& t);

// Run a batch of device-resident items (already oriented, bucket-sorted
// by the planner). d_out is indexed by item.slot.
// local: run the whole batch on this rank (subtrees it owns), never sharded.
void lev_run_host_items(dm_ctx* ctx, const dm_seqset* s, std::vector<LevItem>& items,
                        uint32_t* d_out, LevTotals* tot, bool time_kernels, bool local = false);
// Pairs (2i, 2i+1) of a packed HOST buffer, streamed in chunks (stream.cu).
// speculate: chunks may be sent raw and planned as A/C/G/T, verified on the
// device; the pair ranges of chunks that failed go to *redo (the caller runs
// them again with speculate = false).
void lev_pairs_packed(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint64_t npairs, uint32_t* out,
                      LevTotals* tot, bool speculate, std::vector<std::pair<uint64_t, uint64_t>>* redo);
// Streamed path: plan on `prep` (its stream and scratch), then launch the
// distance kernels on ctx->stream after `planned`. pair_offs (host, 2n+1
// offsets of pairs (2i, 2i+1)) given: the bucket histogram is counted on the
// host from the lengths and the planner never synchronises; null: it is read
// back from the device (one host sync).
void lev_plan_then_launch(dm_ctx* prep, dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                          const uint32_t* d_ib, uint64_t n, uint32_t* d_out, cudaEvent_t planned,
                          LevTotals* tot, const uint64_t* pair_offs = nullptr);
// Pairs given as device arrays (bench path): builds items on the device.
// Host-planned streamed chunks (stream.cu): pairs (2i, 2i+1) of `cnt`
// sequences with host offsets offs[0..2cnt]; items get slots slot0 + i.
// False when a pair needs the multi-pass bucket (the chunk then takes the
// device-planned path). `tmp` is scratch.
constexpr int kLevBuckets = 6 * 32;
constexpr int kLevSrcCodes = 1, kLevSrcRaw = 2;  // = kSrcCodes, kSrcRaw (lev_kernel.cuh)
bool lev_plan_host_pairs(const uint64_t* offs, uint64_t cnt, uint64_t slot0, int sm_count, int wsel_cap,
                         LevItem* items, unsigned int* hist, unsigned long long* cells, std::vector<uint32_t>& tmp);
// Launches a host-planned chunk (items + zeroed per-bucket counters already
// on the device) after `after`; src: 1 = 2-bit codes, 2 = raw A/C/G/T bytes.
int lev_launch_host_planned(dm_ctx* ctx, const LevItem* d_items, uint32_t* d_counters, const unsigned int* hist,
                            int src, const uint8_t* d_codes, const uint64_t* d_off, const uint32_t* d_len,
                            uint32_t* d_out, cudaEvent_t after);
struct LevArgs;
void lev_launch_bucket_src(int src, int w, const LevArgs& a, int sm_count, cudaStream_t st);
void lev_warm_src();
// Jobs already on the device (one rank: no sharding), e.g. generated by the
// tree builder's item kernels. cache (optional): jobs whose pair it holds,
// and a == b, are answered by the planner and never launched; with
// cache->insert the computed ones are added after the batch.
void lev_run_device_items(dm_ctx* ctx, const dm_seqset* s, const LevItem* d_items, uint64_t n, uint32_t* d_out,
                          LevTotals* tot, bool time_kernels, const DistCache* cache = nullptr);
void lev_run_device_pairs(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                          const uint32_t* d_ib, uint64_t n, uint32_t* d_out, LevTotals* tot,
                          bool time_kernels);

// d_raw_given: the residues already sit on the device at that address
// (offsets relative to it after subtracting offsets[0]); not owned.
dm_seqset* seqset_create(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                         const uint8_t* d_raw_given = nullptr);
// Sequence set over residues already on the device (d_raw) whose offsets are
// d_offs[first..first+n] (device, absolute) / h_offs[0..n] (host, same values):
// no host->device copies, so it never queues behind a bulk upload.
// Host mirrors (len/off/blk_off/raw_off) are left empty. The device arrays
// live in ctx's ss_* scratch (no allocation per chunk; valid until the next
// call on ctx, which must be stream-ordered after every use). acgt: the caller
// knows every byte is A/C/G/T (the streamed packer checked), so the census
// and its host sync are skipped (codes A0 C1 G2 T3, 2 bit-planes).
// d_codes_given (with acgt): the code buffer itself, already on the device
// in the code_bytes() layout (the streamed packer writes it on the host);
// d_raw is then unused and left null in the set.
dm_seqset* seqset_create_device(dm_ctx* ctx, const uint8_t* d_raw, const uint64_t* d_offs,
                                const uint64_t* h_offs, uint32_t n, bool acgt = false,
                                const uint8_t* d_codes_given = nullptr);

// Guide tree (tree.cu / tree_host.cpp).
void build_tree(dm_ctx* ctx, const dm_seqset* s, uint64_t seed, uint64_t exact_cap,
                std::vector<dm_node>& nodes, std::vector<uint32_t>& order, dm_stats* st);
double int32_peak(dm_ctx* ctx, int mode);
// The context's side streams (created once, at ctx->side_prio) and their fork/join events.
void ensure_side_streams(dm_ctx* ctx);
void lev_warm();
void nw_warm();
// progress (optional): called once per node as it completes (leaves when the
// rows are initialised, each merge when its level's results are known), as
// align_all's ProgressFn (msa_merge.cpp:121-129): done = 1..nodes.size().
dm_msa_out* align_all(dm_ctx* ctx, const dm_seqset* s, const std::vector<dm_node>& nodes,
                      const std::vector<uint32_t>& order, const NwScheme& sc, dm_stats* st,
                      dm_progress_fn progress = nullptr, void* progress_user = nullptr, bool host_rows = true);
// Rows sel[0..n) of the device row buffer `src` (pitch bytes per row), `width`
// bytes each, gathered on the device and copied densely into host `out`.
void gather_rows_to_host(dm_ctx* ctx, const uint8_t* src, uint64_t pitch, const uint32_t* sel, uint64_t n,
                         uint64_t width, char* out);
void insert_gap_columns(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, const uint32_t* pos,
                        uint64_t npos, char* out);
uint32_t geometric_median(dm_ctx* ctx, const dm_seqset* s, const uint32_t* members, uint64_t n,
                          uint64_t seed, uint64_t exact_cap);

}  // namespace dm
