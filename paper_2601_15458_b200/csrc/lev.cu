// Distance engine: batched exact Levenshtein distance,
// bit-parallel Myers/Hyyro recurrence, warp-cooperative.
//
// Replaces the two-row DP of distance.cpp:30-47 (called from
// cluster_tree.cpp:38 and :144-145). The value computed is the same
// uint32 edit distance; prefix/suffix trimming (distance.cpp:15-26) is an
// exact reduction the bit-parallel form does not need.
//
// Layout of one job (pattern p of m residues, text t of n residues):
//   * the pattern is the SHORTER string (distance is symmetric), cut into
//     B = ceil(m/32) 32-row words; a GROUP of G lanes (G | 32) owns the
//     pattern, lane g holding words [g*W, g*W+W) in registers as ONE
//     multi-precision bit-vector (W is a template parameter, so the state
//     never leaves the register file; carries run through the words of a
//     lane in one add chain and between lanes as the horizontal delta);
//   * the group sweeps the text column by column as a diagonal pipeline:
//     lane g works on column s-g at step s, receiving from lane g-1 (one
//     __shfl_up per column) the horizontal delta leaving the rows above and
//     the text code of that column. Lane 0 reads the text (four codes per
//     32-bit load in the steady state); the top boundary is D[0][j] = j,
//     i.e. h_in = +1;
//   * the match masks: DNA (<= 4 symbols) reads them from a per-thread
//     shared-memory table [code][word][thread]; larger alphabets rebuild Eq
//     from NP bit-planes with one IMAD per plane;
//   * the result needs no per-column bookkeeping: after the last column,
//     D[m][n] = D[0][n] + sum of vertical deltas = n + popc(Pv) - popc(Mv)
//     over the real rows, reduced across the group.
// Warps pull 32/G jobs at a time from an atomic counter (a bounded number
// of pulls per warp, so blocks turn over during a launch); the planner
// sorts jobs by (bucket, text length desc) so a warp's groups run the same
// number of steps, and the buckets' launches overlap on side streams.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "dm_internal.h"
#include "comm.h"
#include "lev_kernel.cuh"

namespace dm {
namespace {

// prefix offsets of the per-column delta buffers of the long jobs, and the
// longest pattern (passes needed): cnt slots + total + max pattern
__global__ void long_prep_kernel(const LevItem* __restrict__ items, uint32_t cnt, const uint32_t* __restrict__ len,
                                 unsigned long long* __restrict__ hoff) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const unsigned long long n = len[items[i].txt];
    hoff[i] = atomicAdd(&hoff[cnt], (n + 15ull) & ~15ull);
    atomicMax(&hoff[cnt + 1], (unsigned long long)len[items[i].pat]);
}

template <int NP>
void run_long_np(dm_ctx* ctx, const LevItem* items, uint32_t cnt, const dm_seqset* s, uint32_t* d_out,
                 cudaStream_t st) {
    constexpr int W = WMax<NP>::value;
    constexpr uint64_t kPassRows = 32ull * W * 32ull;
    uint64_t* hoff = ctx->lev_long_off.as<uint64_t>((uint64_t)cnt + 2 + 64);
    DM_CUDA(cudaMemsetAsync(hoff + cnt, 0, 2 * sizeof(uint64_t), st));
    long_prep_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(items, cnt, s->d_len, (unsigned long long*)hoff);
    DM_CUDA(cudaGetLastError());
    uint64_t* h = ctx->pin_long.as<uint64_t>(2);
    DM_CUDA(cudaMemcpyAsync(h, hoff + cnt, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    DM_CUDA(cudaStreamSynchronize(st));  // rare path: size the delta buffers
    const uint64_t total = h[0], maxm = h[1];
    const uint32_t passes = (uint32_t)((maxm + kPassRows - 1) / kPassRows);
    uint8_t* hbuf = ctx->lev_long_h.as<uint8_t>(total + 16);
    uint32_t* counters = reinterpret_cast<uint32_t*>(hoff + cnt + 2);
    if (passes > 128) throw invalid_argument("sequence too long for the distance engine");
    DM_CUDA(cudaMemsetAsync(counters, 0, passes * sizeof(uint32_t), st));
    LevArgs a{};
    a.items = items;
    a.nitems = cnt;
    a.lgG = 5;
    a.codes = s->d_codes;
    a.off = s->d_off;
    a.len = s->d_len;
    a.blk = s->d_blk;
    a.planes = s->d_planes;
    a.out = d_out;
    a.one = 1u;
    a.hbuf = hbuf;
    a.hoff = hoff;
    for (uint32_t p = 0; p < passes; ++p) {  // stream-ordered: pass p reads what pass p - 1 wrote
        a.pass = p;
        a.counter = counters + p;
        launch_one<NP, W, true>(a, ctx->sm_count, st);
        DM_CUDA(cudaGetLastError());
    }
    ctx->launches += passes + 1;
}

// Patterns longer than 32 lanes x WMax words: multi-pass (LONG kernels).
void run_long(dm_ctx* ctx, const LevItem* items, uint32_t cnt, const dm_seqset* s, uint32_t* d_out,
              cudaStream_t st) {
    if (s->planes == 2) run_long_np<2>(ctx, items, cnt, s, d_out, st);
    else if (s->planes == 5) run_long_np<5>(ctx, items, cnt, s, d_out, st);
    else run_long_np<8>(ctx, items, cnt, s, d_out, st);
}

void launch_bucket(int np, int w, const LevArgs& a, int sm, cudaStream_t st) {
    if (np == 2) dispatch_w<2, 1>(w, a, sm, st);
    else if (np == 5) dispatch_w<5, 1>(w, a, sm, st);
    else dispatch_w<8, 1>(w, a, sm, st);
}

constexpr int kBuckets = 6 * 32;  // (log2 G) * 32 + W
constexpr int kLevSide = dm_ctx::kLevSide;

// ---- DistCache (dm_internal.h): open addressing, linear probing
__device__ __forceinline__ unsigned long long cache_key(uint32_t a, uint32_t b) {
    return a < b ? ((unsigned long long)a << 32 | b) : ((unsigned long long)b << 32 | a);
}
__device__ __forceinline__ uint64_t cache_slot(unsigned long long k, uint64_t mask) {
    k ^= k >> 33;  // murmur3 finaliser
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k & mask;
}
constexpr int kCacheProbes = 64;  // bounded chains: a miss past them only costs the launch

__device__ bool cache_find(const DistCache& dc, uint32_t a, uint32_t b, uint32_t& d) {
    const unsigned long long key = cache_key(a, b);
    uint64_t h = cache_slot(key, dc.mask);
    for (int p = 0; p < kCacheProbes; ++p, h = (h + 1) & dc.mask) {
        const unsigned long long k = *(volatile const unsigned long long*)(dc.keys + h);
        if (k == kCacheEmpty) return false;
        if (k == key) {
            const uint32_t v = *(volatile const uint32_t*)(dc.vals + h);
            if (v == kCacheNone) return false;  // being inserted (background batch): a miss
            d = v;
            return true;
        }
    }
    return false;
}

__device__ void cache_put(const DistCache& dc, uint32_t a, uint32_t b, uint32_t d) {
    if (a == b || *(volatile unsigned int*)dc.fill >= dc.max_fill) return;
    const unsigned long long key = cache_key(a, b);
    uint64_t h = cache_slot(key, dc.mask);
    for (int p = 0; p < kCacheProbes; ++p, h = (h + 1) & dc.mask) {
        const unsigned long long prev = atomicCAS(dc.keys + h, kCacheEmpty, key);
        if (prev == kCacheEmpty || prev == key) {
            if (prev == kCacheEmpty) atomicAdd(dc.fill, 1u);
            dc.vals[h] = d;  // the same value whoever writes it
            return;
        }
    }
}

// Orient each job (shorter string = pattern), pick (G, R) and build the
// radix key (bucket << 32 | ~n) so one sort groups buckets and balances warps.
__global__ void plan_kernel(const uint32_t* __restrict__ ia, const uint32_t* __restrict__ ib,
                            const LevItem* __restrict__ in_items, uint64_t n,
                            const uint32_t* __restrict__ len, int lg_gpar, int wsel, int wmax,
                            LevItem* __restrict__ items, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ idx, unsigned int* __restrict__ hist,
                            unsigned long long* __restrict__ cells, const DistCache dc, uint32_t* __restrict__ out) {
    __shared__ unsigned int sh[kBuckets];
    __shared__ unsigned long long scells[3];
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) sh[i] = 0;
    if (threadIdx.x < 3) scells[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long c0 = 0, c1 = 0, c2 = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint32_t x, y;
        uint64_t slot;
        if (in_items) {
            x = in_items[i].pat;
            y = in_items[i].txt;
            slot = in_items[i].slot;
        } else {
            x = ia[i];
            y = ib[i];
            slot = i;
        }
        uint32_t lx = len[x], ly = len[y];
        if (lx > ly) {  // pattern = shorter
            const uint32_t t = x; x = y; y = t;
            const uint32_t tl = lx; lx = ly; ly = tl;
        }
        if (dc.keys) {  // answered without a launch: bucket 0 (never launched)
            uint32_t d = 0;
            if (x == y || cache_find(dc, x, y, d)) {
                out[slot] = d;
                items[i] = LevItem{x, y, slot};
                keys[i] = 0;
                idx[i] = (uint32_t)i;
                atomicAdd(&sh[0], 1u);
                c2 += (unsigned long long)lx * ly;
                continue;
            }
        }
        const uint32_t B = (lx + 31) >> 5;  // 32-row words of the pattern
        int lg = lg_gpar;
        while ((uint32_t)(wsel << lg) < B && lg < 5) ++lg;
        uint32_t R = (B + (1u << lg) - 1) >> lg;  // words per lane
        if (R < 1) R = 1;
        uint32_t bucket = (uint32_t)lg * 32 + R;
        unsigned long long rows = (unsigned long long)(R << lg) * 32ull;
        if (R > (uint32_t)wmax) {  // longer than one warp's rows: the multi-pass bucket
            bucket = kBuckets - 1;
            const unsigned long long pr = 1024ull * (unsigned)wmax;
            rows = (lx + pr - 1) / pr * pr;
        }
        items[i] = LevItem{x, y, slot};
        keys[i] = ((uint64_t)bucket << 32) | (uint64_t)(0xffffffffu - ly);
        idx[i] = (uint32_t)i;
        atomicAdd(&sh[bucket], 1u);
        c0 += (unsigned long long)lx * ly;
        c1 += rows * ly;
    }
    atomicAdd(&scells[0], c0);
    atomicAdd(&scells[1], c1);
    if (c2) atomicAdd(&scells[2], c2);
    __syncthreads();
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
    if (threadIdx.x == 0) {
        atomicAdd(&cells[0], scells[0]);
        atomicAdd(&cells[1], scells[1]);
        atomicAdd(&cells[2], scells[2]);
    }
}

// The computed jobs of a batch (planned items past bucket 0) into the cache.
__global__ void cache_insert_kernel(const LevItem* __restrict__ items, uint64_t n, const uint32_t* __restrict__ out,
                                    const DistCache dc) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const LevItem it = items[i];
        cache_put(dc, it.pat, it.txt, out[it.slot]);
    }
}

__global__ void gather_items(const LevItem* __restrict__ in, const uint32_t* __restrict__ idx,
                             uint64_t n, LevItem* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[idx[i]];
}

// A planned batch: bucket-sorted items plus the host copy of the histogram.
struct LevPlan {
    LevItem* items = nullptr;
    uint32_t* counters = nullptr;
    unsigned int h[kBuckets];
    unsigned long long hc[3];  // cells, cells executed, cells answered by the cache
};

// plan_kernel's histogram and cell counts for pairs (2i, 2i+1) of host
// offsets, counted on the host (same orientation and bucket rule).
void plan_hist_host(const uint64_t* offs, uint64_t n, int lg_gpar, int wsel, int wmax, LevPlan& P) {
    // lg per pattern word count B (beyond the table: 5); the per-pair body is
    // branch-free (random orientations would mispredict)
    const uint32_t bmax = (uint32_t)wsel << 5;
    std::vector<uint8_t> lgof(bmax + 2);
    for (uint32_t B = 0; B <= bmax + 1; ++B) {
        int lg = lg_gpar;
        while ((uint32_t)(wsel << lg) < B && lg < 5) ++lg;
        lgof[B] = (uint8_t)lg;
    }
    std::vector<unsigned int> h(4 * kBuckets, 0u);  // 4 interleaved copies: no store-forwarding chains
    unsigned long long c0 = 0, c1 = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t a = (uint32_t)(offs[2 * i + 1] - offs[2 * i]), b = (uint32_t)(offs[2 * i + 2] - offs[2 * i + 1]);
        const uint32_t m = 0u - (uint32_t)(a < b), lx = (a & m) | (b & ~m), ly = a ^ b ^ lx;
        const uint32_t B = (lx + 31) >> 5;
        const int lg = lgof[std::min(B, bmax + 1)];
        const uint32_t R = std::max((B + (1u << lg) - 1) >> lg, 1u);
        const bool lng = R > (uint32_t)wmax;
        const uint32_t bucket = lng ? kBuckets - 1 : (uint32_t)lg * 32 + R;
        ++h[(i & 3) * kBuckets + bucket];
        c0 += (unsigned long long)lx * ly;
        const unsigned long long pr = 1024ull * (unsigned)wmax;
        c1 += (lng ? (lx + pr - 1) / pr * pr : (unsigned long long)(R << lg) * 32ull) * ly;
    }
    for (int k = 0; k < kBuckets; ++k) P.h[k] = h[k] + h[kBuckets + k] + h[2 * kBuckets + k] + h[3 * kBuckets + k];
    P.hc[0] = c0;
    P.hc[1] = c1;
    P.hc[2] = 0;
}

// Planner phase on `ctx`'s stream (scratch from ctx): orient, bucket, sort,
// read the histogram back (the one host sync of a batch) -- or, given the
// host offsets of identity pairs (2i, 2i+1), count it on the host and stay
// asynchronous.
void plan_batch(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia, const uint32_t* d_ib,
                const LevItem* d_in_items, uint64_t n, LevPlan& P, const uint64_t* pair_offs = nullptr,
                const DistCache* dc = nullptr, uint32_t* d_out = nullptr) {
    if (n > 0xffffffffull) throw invalid_argument("too many distance jobs in one batch");
    cudaStream_t st = ctx->stream;
    const int np = s->planes;
    int wmax = wmax_for(np);
    if (const char* e = std::getenv("DM_LEV_WMAX")) {  // tuning knob: cap words per lane
        const int v = std::atoi(e);
        if (v >= 1 && v < wmax) wmax = v;
    }
    // lanes per pair are chosen for at most `wsel` words per lane; longer
    // patterns (lanes per pair maxed out) still go up to wmax
    const int wsel = ctx->lev_wmax_cap > 0 ? std::min(wmax, ctx->lev_wmax_cap) : wmax;
    const uint64_t target = (uint64_t)ctx->sm_count * 512;  // lanes wanted in flight
    int lg_gpar = 0;
    while (lg_gpar < 5 && (n << lg_gpar) < target) ++lg_gpar;
    if (const char* e = std::getenv("DM_LEV_GPAR")) {  // test knob: force the minimum lanes per pair (log2)
        const int v = std::atoi(e);
        if (v >= 0 && v <= 5) lg_gpar = v;
    }

    // scratch: items(2x), keys(2x), idx(2x), hist, cells, counters, cub temp
    const size_t item_b = n * sizeof(LevItem), key_b = n * 8, idx_b = n * 4;
    size_t cub_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_b, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 40, st);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t hist_b = al(kBuckets * 4 + 32 + kBuckets * 4);
    size_t total = al(item_b) * 2 + al(key_b) * 2 + al(idx_b) * 2 + hist_b + al(cub_b);
    char* base = (char*)ctx->items.get(total);
    LevItem* it0 = (LevItem*)base; base += al(item_b);
    LevItem* it1 = (LevItem*)base; base += al(item_b);
    uint64_t* k0 = (uint64_t*)base; base += al(key_b);
    uint64_t* k1 = (uint64_t*)base; base += al(key_b);
    uint32_t* i0 = (uint32_t*)base; base += al(idx_b);
    uint32_t* i1 = (uint32_t*)base; base += al(idx_b);
    unsigned int* hist = (unsigned int*)base;
    unsigned long long* cells = (unsigned long long*)(hist + kBuckets);
    uint32_t* counters = (uint32_t*)(cells + 4);
    base += hist_b;
    void* cub_tmp = base;

    DM_CUDA(cudaMemsetAsync(hist, 0, hist_b, st));
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 8);
    plan_kernel<<<grid, 256, 0, st>>>(d_ia, d_ib, d_in_items, n, s->d_len, lg_gpar, wsel, wmax, it0, k0, i0,
                                      hist, cells, dc ? *dc : DistCache{}, d_out);
    DM_CUDA(cudaGetLastError());
    DM_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_b, k0, k1, i0, i1, (int)n, 0, 40, st));
    gather_items<<<grid, 256, 0, st>>>(it0, i1, n, it1);
    DM_CUDA(cudaGetLastError());
    if (pair_offs) {
        plan_hist_host(pair_offs, n, lg_gpar, wsel, wmax, P);
    } else {
        DM_CUDA(cudaMemcpyAsync(P.h, hist, sizeof(P.h), cudaMemcpyDeviceToHost, st));
        DM_CUDA(cudaMemcpyAsync(P.hc, cells, sizeof(P.hc), cudaMemcpyDeviceToHost, st));
        DM_CUDA(cudaStreamSynchronize(st));
    }
    P.items = it1;
    P.counters = counters;
    ctx->launches += 2;
}

// Kernel phase: one persistent launch per non-empty bucket. A bucket's launch
// drains with a tail (its last warp tasks run while SMs empty out), so the
// buckets go out on side streams, largest per-task work first: the next
// bucket's blocks take the SMs the previous one frees. `after` (optional) is
// the event the launches must follow; by default they follow `st`. `st`
// waits for all of them on return.
// Residue source of a launch (lev_kernel.cuh): a resident / planner-built
// sequence set (bit-planes), or a host-planned streamed chunk (2-bit codes or
// raw A/C/G/T bytes, with uploaded per-sequence offsets and lengths).
struct LevSrc {
    int np = 2, src = kSrcPlanes;
    const uint8_t* codes = nullptr;
    const uint64_t* off = nullptr;
    const uint32_t* len = nullptr;
    const uint64_t* blk = nullptr;
    const uint64_t* planes = nullptr;
    const dm_seqset* set = nullptr;  // multi-pass bucket (bit-plane sources only)
};

LevSrc src_of(const dm_seqset* s) {
    LevSrc r;
    r.np = s->planes;
    r.codes = s->d_codes;
    r.off = s->d_off;
    r.len = s->d_len;
    r.blk = s->d_blk;
    r.planes = s->d_planes;
    r.set = s;
    return r;
}

int launch_plan(dm_ctx* ctx, const LevPlan& P, const LevSrc& S, uint32_t* d_out, cudaStream_t st,
                cudaEvent_t after = nullptr) {
    uint64_t starts[kBuckets];
    int order[kBuckets], nb = 0;
    uint64_t start = 0;
    for (int b = 0; b < kBuckets; ++b) {
        starts[b] = start;
        start += P.h[b];
        if (P.h[b] && b != 0) order[nb++] = b;  // bucket 0: answered by the planner (DistCache)
    }
    // the multi-pass bucket (largest work per job) is first in `order`:
    // it goes to the first side stream and syncs that stream once to size
    // its buffers (run_long)
    // largest per-task work first: lanes per pair x words per lane
    std::stable_sort(order, order + nb, [](int x, int y) { return ((x % 32) << (x / 32)) > ((y % 32) << (y / 32)); });
    // (a context with prioritised side streams always fans out: its batches
    // then take SM slots ahead of default-priority work, e.g. the tree's
    // background batches)
    const bool fork = nb > 1 || after != nullptr || ctx->side_prio != 0;
    int used[kLevSide], nused = 0;
    if (fork) {
        ensure_side_streams(ctx);
        if (!after) {
            DM_CUDA(cudaEventRecord(ctx->lev_fork, st));
            after = ctx->lev_fork;
        }
        // rotate through the side streams across calls, so back-to-back
        // batches (streamed chunks) do not queue behind each other's tails
        for (int i = 0; i < std::min(nb, kLevSide); ++i) {
            used[nused] = (ctx->lev_rr + i) % kLevSide;
            DM_CUDA(cudaStreamWaitEvent(ctx->lev_side[used[nused]], after, 0));
            ++nused;
        }
        ctx->lev_rr = (ctx->lev_rr + nused) % kLevSide;
    }
    for (int i = 0; i < nb; ++i) {
        const int b = order[i];
        if (b == kBuckets - 1) {
            if (!S.set) throw runtime_error("internal error: multi-pass distance jobs in a host-planned chunk");
            // rare path, on `st` itself: its delta buffers and pass counters are
            // context scratch allocated in `st`'s order, so the multi-pass jobs of
            // overlapping batches (streamed chunks) must not run concurrently
            if (after) DM_CUDA(cudaStreamWaitEvent(st, after, 0));
            run_long(ctx, P.items + starts[b], P.h[b], S.set, d_out, st);
            continue;
        }
        LevArgs a{};
        a.items = P.items + starts[b];
        a.nitems = P.h[b];
        a.lgG = b / 32;
        a.codes = S.codes;
        a.off = S.off;
        a.len = S.len;
        a.blk = S.blk;
        a.planes = S.planes;
        a.out = d_out;
        a.counter = P.counters + b;
        a.one = 1u;
        a.waves = ctx->lev_waves;
        cudaStream_t ls = fork ? ctx->lev_side[used[i % nused]] : st;
        if (S.src == kSrcPlanes) launch_bucket(S.np, b % 32, a, ctx->sm_count, ls);
        else lev_launch_bucket_src(S.src, b % 32, a, ctx->sm_count, ls);
        DM_CUDA(cudaGetLastError());
    }
    for (int i = 0; i < nused; ++i) {
        DM_CUDA(cudaEventRecord(ctx->lev_join[used[i]], ctx->lev_side[used[i]]));
        DM_CUDA(cudaStreamWaitEvent(st, ctx->lev_join[used[i]], 0));
    }
    return nb;
}

void run_planned(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia, const uint32_t* d_ib,
                 const LevItem* d_in_items, uint64_t n, uint32_t* d_out, LevTotals* tot,
                 bool time_kernels, const DistCache* dc = nullptr) {
    if (n == 0) return;
    LevPlan P;
    plan_batch(ctx, s, d_ia, d_ib, d_in_items, n, P, nullptr, dc, d_out);
    cudaStream_t st = ctx->stream;
    const bool timed = time_kernels && tot;  // event pairs read later (lev_finish_timing): no sync here
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        DM_CUDA(cudaEventCreate(&e0));
        DM_CUDA(cudaEventCreate(&e1));
        tot->pend.push_back(e0);
        tot->pend.push_back(e1);
        DM_CUDA(cudaEventRecord(e0, st));
    }
    int launches = launch_plan(ctx, P, src_of(s), d_out, st);
    if (timed) DM_CUDA(cudaEventRecord(e1, st));
    if (dc && dc->insert && n > P.h[0]) {
        const uint64_t m = n - P.h[0];
        const int grid = (int)std::min<uint64_t>((m + 255) / 256, (uint64_t)ctx->sm_count * 8);
        cache_insert_kernel<<<grid, 256, 0, st>>>(P.items + P.h[0], m, d_out, *dc);
        DM_CUDA(cudaGetLastError());
        ++launches;
    }
    ctx->launches += launches;
    if (tot) {
        tot->cells += P.hc[0];
        tot->cells_exec += P.hc[1];
        tot->reused += P.h[0];
        tot->cells_reused += P.hc[2];
        tot->launches += launches + 2;
    }
}

}  // namespace

void ensure_side_streams(dm_ctx* ctx) {
    if (ctx->lev_fork) return;
    DM_CUDA(cudaEventCreateWithFlags(&ctx->lev_fork, cudaEventDisableTiming));
    for (int k = 0; k < dm_ctx::kLevSide; ++k) {
        DM_CUDA(cudaStreamCreateWithPriority(&ctx->lev_side[k], cudaStreamNonBlocking, ctx->side_prio));
        DM_CUDA(cudaEventCreateWithFlags(&ctx->lev_join[k], cudaEventDisableTiming));
    }
}

void lev_finish_timing(LevTotals& t) {
    for (size_t i = 0; i + 1 < t.pend.size(); i += 2) {
        DM_CUDA(cudaEventSynchronize(t.pend[i + 1]));
        float ms = 0;
        DM_CUDA(cudaEventElapsedTime(&ms, t.pend[i], t.pend[i + 1]));
        t.kernel_ms += ms;
    }
    for (cudaEvent_t e : t.pend) cudaEventDestroy(e);
    t.pend.clear();
}

// Loads every kernel instance up front (lazy module loading would otherwise
// charge the first batch that hits a new bucket).
void lev_warm() {
    warm_np<2, 1>();
    warm_np<5, 1>();
    warm_np<8, 1>();
    lev_warm_src();
}

namespace {
// all[r * maxc + k] holds job bounds[r] + k of shard r; route it to its slot.
__global__ void scatter_shards(const uint32_t* __restrict__ all, const LevItem* __restrict__ items, uint64_t n,
                               const uint64_t* __restrict__ bounds, int w, uint64_t maxc, uint32_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int r = 0;
        while (r + 1 < w && bounds[r + 1] <= i) ++r;
        out[items[i].slot] = all[(uint64_t)r * maxc + (i - bounds[r])];
    }
}
}  // namespace

void lev_run_host_items(dm_ctx* ctx, const dm_seqset* s, std::vector<LevItem>& items,
                        uint32_t* d_out, LevTotals* tot, bool time_kernels, bool local) {
    if (items.empty()) return;
    const uint64_t n = items.size();
    const int w = local ? 1 : shard_world(ctx);
    if (w == 1) {
        LevItem* d_items = ctx->aux3.as<LevItem>(n);
        DM_CUDA(cudaMemcpyAsync(d_items, items.data(), n * sizeof(LevItem), cudaMemcpyHostToDevice, ctx->stream));
        run_planned(ctx, s, nullptr, nullptr, d_items, n, d_out, tot, time_kernels);
        return;
    }
    // Sharded batch: rank r computes the cost-balanced range [bounds[r],
    // bounds[r+1]) (cost |a| * |b|) into its row of `all`, the rows are
    // all-gathered, and every rank scatters the full result to the slots
    // (decisions stay replicated).
    std::vector<uint64_t> cost(n), bounds;
    for (uint64_t i = 0; i < n; ++i) cost[i] = (uint64_t)s->len[items[i].pat] * s->len[items[i].txt];
    shard_bounds(cost.data(), n, w, bounds);
    uint64_t maxc = 1;
    for (int r = 0; r < w; ++r) maxc = std::max(maxc, bounds[r + 1] - bounds[r]);
    uint32_t* d_all = ctx->lev_all.as<uint32_t>((uint64_t)w * maxc + 1);
    LevItem* d_global = ctx->lev_items.as<LevItem>(n);
    uint64_t* d_bounds = ctx->shard_buf.as<uint64_t>((uint64_t)w + 1);
    DM_CUDA(cudaMemcpyAsync(d_global, items.data(), n * sizeof(LevItem), cudaMemcpyHostToDevice, ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_bounds, bounds.data(), (w + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    const bool real = comm_real(ctx);
    std::vector<LevItem> sub;
    for (int r = 0; r < w; ++r) {
        if (real && r != ctx->rank) continue;
        const uint64_t lo = bounds[r], hi = bounds[r + 1];
        if (hi == lo) continue;
        sub.assign(items.begin() + lo, items.begin() + hi);
        for (uint64_t k = 0; k < sub.size(); ++k) sub[k].slot = k;
        LevItem* d_items = ctx->aux3.as<LevItem>(sub.size());
        DM_CUDA(cudaMemcpyAsync(d_items, sub.data(), sub.size() * sizeof(LevItem), cudaMemcpyHostToDevice,
                                ctx->stream));
        run_planned(ctx, s, nullptr, nullptr, d_items, sub.size(), d_all + (uint64_t)r * maxc, tot, time_kernels);
        DM_CUDA(cudaStreamSynchronize(ctx->stream));  // host `sub` reused / shard done before the exchange
    }
    if (real) comm_allgather(ctx, d_all + (uint64_t)ctx->rank * maxc, d_all, maxc * sizeof(uint32_t));
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 8);
    scatter_shards<<<std::max(grid, 1), 256, 0, ctx->stream>>>(d_all, d_global, n, d_bounds, w, maxc, d_out);
    DM_CUDA(cudaGetLastError());
    ctx->launches += 1;
}

void lev_run_device_items(dm_ctx* ctx, const dm_seqset* s, const LevItem* d_items, uint64_t n, uint32_t* d_out,
                          LevTotals* tot, bool time_kernels, const DistCache* cache) {
    run_planned(ctx, s, nullptr, nullptr, d_items, n, d_out, tot, time_kernels, cache);
}

void lev_run_device_pairs(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                          const uint32_t* d_ib, uint64_t n, uint32_t* d_out, LevTotals* tot,
                          bool time_kernels) {
    run_planned(ctx, s, d_ia, d_ib, nullptr, n, d_out, tot, time_kernels);
}

void lev_plan_then_launch(dm_ctx* prep, dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                          const uint32_t* d_ib, uint64_t n, uint32_t* d_out, cudaEvent_t planned,
                          LevTotals* tot, const uint64_t* pair_offs) {
    if (n == 0) return;
    LevPlan P;
    const bool tr = std::getenv("DM_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    plan_batch(prep, s, d_ia, d_ib, nullptr, n, P, pair_offs);
    auto t1 = std::chrono::steady_clock::now();
    DM_CUDA(cudaEventRecord(planned, prep->stream));
    // the kernels follow the planner directly, not ctx->stream: this batch's
    // buckets start while the previous batch's tails still drain
    const int launches = launch_plan(ctx, P, src_of(s), d_out, ctx->stream, planned);
    auto t2 = std::chrono::steady_clock::now();
    if (tr)
        std::fprintf(stderr, "[plan] plan_batch %.2f ms, launch_plan %.2f ms (%d launches)\n",
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(t2 - t1).count(), launches);
    ctx->launches += launches;
    if (tot) {
        tot->cells += P.hc[0];
        tot->cells_exec += P.hc[1];
        tot->launches += launches + 2;
    }
}

// ---- host-planned chunks of identity pairs (the streamed path, stream.cu)


bool lev_plan_host_pairs(const uint64_t* offs, uint64_t cnt, uint64_t slot0, int sm_count, int wsel_cap,
                         LevItem* items, unsigned int* hist, unsigned long long* cells, std::vector<uint32_t>& tmp) {
    // the same orientation / bucket rule as plan_kernel; the order (bucket asc,
    // text length desc in 8-residue bins, stable) by two counting sorts
    // (order only matters for warp balance)
    int wmax = wmax_for(2);
    if (const char* e = std::getenv("DM_LEV_WMAX")) {
        const int v = std::atoi(e);
        if (v >= 1 && v < wmax) wmax = v;
    }
    const int wsel = wsel_cap > 0 ? std::min(wmax, wsel_cap) : wmax;
    const uint64_t target = (uint64_t)sm_count * 512;
    int lg_gpar = 0;
    while (lg_gpar < 5 && (cnt << lg_gpar) < target) ++lg_gpar;
    if (const char* e = std::getenv("DM_LEV_GPAR")) {
        const int v = std::atoi(e);
        if (v >= 0 && v <= 5) lg_gpar = v;
    }
    const uint32_t bmax = (uint32_t)wsel << 5;
    uint8_t lgof[32 * 32 + 2];
    for (uint32_t B = 0; B <= bmax + 1; ++B) {
        int lg = lg_gpar;
        while ((uint32_t)(wsel << lg) < B && lg < 5) ++lg;
        lgof[B] = (uint8_t)lg;
    }
    std::memset(hist, 0, kBuckets * sizeof(unsigned int));
    // one counting sort over (bucket, text length desc in 8-residue bins):
    // pass 1 keys every pair, pass 2 scatters the items (order only matters
    // for warp balance; within a key the pairs keep their order)
    constexpr uint32_t kLenBins = 1u << 13;
    tmp.resize(cnt);
    uint32_t* key = tmp.data();  // bucket << 13 | length bin (bin 0 = longest)
    uint32_t lbmin = kLenBins, lbmax = 0;
    unsigned long long c0 = 0, c1 = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint32_t a = (uint32_t)(offs[2 * i + 1] - offs[2 * i]), b = (uint32_t)(offs[2 * i + 2] - offs[2 * i + 1]);
        const uint32_t lx = std::min(a, b), ly = std::max(a, b);
        const uint32_t B = (lx + 31) >> 5;
        const int lg = lgof[std::min(B, bmax + 1)];
        const uint32_t R = std::max((B + (1u << lg) - 1) >> lg, 1u);
        if (R > (uint32_t)wmax) return false;  // multi-pass bucket: the chunk takes the device-planned path
        const uint32_t bucket = (uint32_t)lg * 32 + R;
        ++hist[bucket];
        const uint32_t lb = kLenBins - 1 - std::min(ly >> 3, kLenBins - 1);
        lbmin = std::min(lbmin, lb);
        lbmax = std::max(lbmax, lb);
        key[i] = bucket << 13 | lb;
        c0 += (unsigned long long)lx * ly;
        c1 += (unsigned long long)(R << lg) * 32ull * ly;
    }
    int dense[kBuckets], nd = 0;
    for (int bk = 0; bk < kBuckets; ++bk) dense[bk] = hist[bk] ? nd++ : -1;  // ascending bucket ids
    const uint32_t range = lbmax - lbmin + 1;
    thread_local std::vector<uint32_t> pos;  // counting-sort table, per planning thread
    pos.assign((size_t)nd * range + 1, 0u);
    for (uint64_t i = 0; i < cnt; ++i)
        ++pos[(size_t)dense[key[i] >> 13] * range + ((key[i] & (kLenBins - 1)) - lbmin) + 1];
    for (size_t k = 1; k < pos.size(); ++k) pos[k] += pos[k - 1];
    for (uint64_t i = 0; i < cnt; ++i) {
        const bool swap = offs[2 * i + 1] - offs[2 * i] > offs[2 * i + 2] - offs[2 * i + 1];  // plan_kernel's orientation
        const uint32_t at = pos[(size_t)dense[key[i] >> 13] * range + ((key[i] & (kLenBins - 1)) - lbmin)]++;
        items[at] = LevItem{2 * (uint32_t)i + (swap ? 1u : 0u), 2 * (uint32_t)i + (swap ? 0u : 1u), slot0 + i};
    }
    cells[0] = c0;
    cells[1] = c1;
    return true;
}

int lev_launch_host_planned(dm_ctx* ctx, const LevItem* d_items, uint32_t* d_counters, const unsigned int* hist,
                            int src, const uint8_t* d_codes, const uint64_t* d_off, const uint32_t* d_len,
                            uint32_t* d_out, cudaEvent_t after) {
    LevPlan P;
    P.items = const_cast<LevItem*>(d_items);
    P.counters = d_counters;
    std::memcpy(P.h, hist, sizeof(P.h));
    P.hc[0] = P.hc[1] = 0;
    LevSrc S;
    S.np = 2;
    S.src = src;
    S.codes = d_codes;
    S.off = d_off;
    S.len = d_len;
    const int launches = launch_plan(ctx, P, S, d_out, ctx->stream, after);
    ctx->launches += launches;
    return launches;
}

}  // namespace dm
