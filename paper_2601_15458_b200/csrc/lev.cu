// Distance engine: batched exact Levenshtein distance,
// bit-parallel Myers/Hyyro recurrence over 64-bit blocks, warp-cooperative.
//
// Replaces the two-row DP of distance.cpp:30-47 (called from
// cluster_tree.cpp:38 and :144-145). The value computed is the same
// uint32 edit distance; prefix/suffix trimming (distance.cpp:15-26) is an
// exact reduction the bit-parallel form does not need.
//
// Layout of one job (pattern p of m residues, text t of n residues):
//   * the pattern is the SHORTER string (distance is symmetric), cut into
//     B = ceil(m/64) blocks of 64 rows; a GROUP of G lanes (G | 32) owns the
//     pattern, lane g holding blocks [g*R, g*R+R) in registers (R is a
//     template parameter, so the block state never leaves the register file);
//   * the group sweeps the text column by column as a diagonal pipeline:
//     lane g works on column s-g at step s, receiving from lane g-1 (one
//     __shfl_up per column) the horizontal delta leaving the block above and
//     the text code of that column. Lane 0 reads the text; the top boundary
//     is D[0][j] = j, i.e. h_in = +1;
//   * the match mask of a residue code c is built from NP bit-planes of the
//     pattern: Eq = AND_k (bit_k(c) ? P_k : ~P_k) — one LOP per plane, no
//     shared-memory table;
//   * the result needs no per-column bookkeeping: after the last column,
//     D[m][n] = D[0][n] + sum of vertical deltas = n + popc(Pv) - popc(Mv)
//     over the real rows, reduced across the group.
// Every warp is persistent and pulls 32/G jobs at a time from an atomic
// counter; the planner sorts jobs by (bucket, text length desc) so a warp's
// groups run the same number of steps.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>

#include "dm_internal.h"

namespace dm {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// Register budget per lane: 4R words of Pv/Mv state + 2*NP*R words of planes.
template <int NP>
struct RMax;
template <>
struct RMax<2> { static constexpr int value = 12; };
template <>
struct RMax<5> { static constexpr int value = 6; };
template <>
struct RMax<8> { static constexpr int value = 4; };

int rmax_for(int np) { return np == 2 ? RMax<2>::value : (np == 5 ? RMax<5>::value : RMax<8>::value); }

struct LevArgs {
    const LevItem* items;
    uint32_t nitems;
    int lgG;
    const uint8_t* codes;
    const uint64_t* off;
    const uint32_t* len;
    const uint64_t* blk;
    const uint64_t* planes;
    uint32_t* out;
    uint32_t* counter;
};

template <int NP, int R>
__global__ void __launch_bounds__(256) lev_kernel(const LevArgs a) {
    const int lane = threadIdx.x & 31;
    const int lgG = a.lgG;
    const int G = 1 << lgG;
    const int g = lane & (G - 1);
    const int grp = lane >> lgG;
    const uint32_t gpw = 32u >> lgG;

    for (;;) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(a.counter, gpw);
        base = __shfl_sync(FULL, base, 0);
        if (base >= a.nitems) break;
        const uint32_t it = base + grp;
        const bool valid = it < a.nitems;
        LevItem item{0, 0, 0};
        if (valid) item = a.items[it];
        const uint32_t m = valid ? a.len[item.pat] : 0;
        const uint32_t n = valid ? a.len[item.txt] : 0;
        const uint32_t nb = (m + 63) >> 6;

        uint64_t P[R][NP];
        uint64_t Pv[R], Mv[R];
        const uint64_t* pp = a.planes + a.blk[item.pat] * NP;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t b = (uint32_t)g * R + r;
#pragma unroll
            for (int k = 0; k < NP; ++k) P[r][k] = (valid && b < nb) ? __ldg(pp + (uint64_t)b * NP + k) : 0ull;
            Pv[r] = ~0ull;
            Mv[r] = 0ull;
        }
        // rows this lane owns that are real pattern rows
        const int first_row = g * R * 64;
        const int own = max(0, min((int)m - first_row, R * 64));
        int partial = own;  // sum of vertical deltas at column 0 (all +1)

        uint32_t steps = valid ? n + (uint32_t)G - 1u : 0u;
        steps = __reduce_max_sync(FULL, steps);
        const uint8_t* tp = a.codes + a.off[item.txt];
        uint32_t word = 0;
        for (uint32_t s = 0; s < steps; ++s) {
            const uint32_t recv = __shfl_up_sync(FULL, word, 1, G);
            uint32_t c, hp, hm;
            if (g == 0) {
                c = (s < n) ? (uint32_t)tp[s] : 0u;
                hp = 1u;
                hm = 0u;
            } else {
                c = recv >> 2;
                hp = recv & 1u;
                hm = (recv >> 1) & 1u;
            }
            const uint32_t j = s - (uint32_t)g;
            if (j < n) {
                uint64_t msk[NP];
#pragma unroll
                for (int k = 0; k < NP; ++k) msk[k] = 0ull - (uint64_t)((c >> k) & 1u);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    uint64_t eq = ~(P[r][0] ^ msk[0]);
#pragma unroll
                    for (int k = 1; k < NP; ++k) eq &= ~(P[r][k] ^ msk[k]);
                    const uint64_t pv = Pv[r], mv = Mv[r];
                    const uint64_t xv = eq | mv;
                    const uint64_t e = eq | (uint64_t)hm;
                    const uint64_t xh = (((e & pv) + pv) ^ pv) | e;
                    uint64_t ph = mv | ~(xh | pv);
                    uint64_t mh = pv & xh;
                    const uint32_t hpo = (uint32_t)(ph >> 63);
                    const uint32_t hmo = (uint32_t)(mh >> 63);
                    ph = (ph << 1) | (uint64_t)hp;
                    mh = (mh << 1) | (uint64_t)hm;
                    Pv[r] = mh | ~(xv | ph);
                    Mv[r] = ph & xv;
                    hp = hpo;
                    hm = hmo;
                }
                if (j == n - 1) {
                    int acc = 0;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int lo = first_row + r * 64;
                        const int cnt = max(0, min((int)m - lo, 64));
                        const uint64_t rm = cnt >= 64 ? ~0ull : ((1ull << cnt) - 1ull);
                        acc += __popcll(Pv[r] & rm) - __popcll(Mv[r] & rm);
                    }
                    partial = acc;
                }
            }
            word = (c << 2) | (hm << 1) | hp;
        }
        for (int o = G >> 1; o > 0; o >>= 1) partial += __shfl_down_sync(FULL, partial, o, G);
        if (valid && g == 0) a.out[item.slot] = n + (uint32_t)partial;
    }
}

template <int NP, int R>
void launch_one(const LevArgs& a, int sm_count, cudaStream_t st) {
    static int occ = -1;
    if (occ < 0) {
        DM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lev_kernel<NP, R>, 256, 0));
        occ = std::max(occ, 1);
    }
    const uint64_t lanes = (uint64_t)a.nitems << a.lgG;
    const uint64_t want = (lanes + 255) / 256;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)occ * sm_count));
    lev_kernel<NP, R><<<grid, 256, 0, st>>>(a);
}

template <int NP, int R>
void dispatch_r(int r, const LevArgs& a, int sm, cudaStream_t st) {
    if constexpr (R <= RMax<NP>::value) {
        if (r == R) {
            launch_one<NP, R>(a, sm, st);
            return;
        }
        dispatch_r<NP, R + 1>(r, a, sm, st);
    } else {
        throw runtime_error("distance engine: unsupported block count");
    }
}

void launch_bucket(int np, int r, const LevArgs& a, int sm, cudaStream_t st) {
    if (np == 2) dispatch_r<2, 1>(r, a, sm, st);
    else if (np == 5) dispatch_r<5, 1>(r, a, sm, st);
    else dispatch_r<8, 1>(r, a, sm, st);
}

constexpr int kBuckets = 6 * 16;

// Orient each job (shorter string = pattern), pick (G, R) and build the
// radix key (bucket << 32 | ~n) so one sort groups buckets and balances warps.
__global__ void plan_kernel(const uint32_t* __restrict__ ia, const uint32_t* __restrict__ ib,
                            const LevItem* __restrict__ in_items, uint64_t n,
                            const uint32_t* __restrict__ len, int lg_gpar, int rmax,
                            LevItem* __restrict__ items, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ idx, unsigned int* __restrict__ hist,
                            unsigned long long* __restrict__ cells) {
    __shared__ unsigned int sh[kBuckets];
    __shared__ unsigned long long scells[2];
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) sh[i] = 0;
    if (threadIdx.x < 2) scells[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long c0 = 0, c1 = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint32_t x, y, slot;
        if (in_items) {
            x = in_items[i].pat;
            y = in_items[i].txt;
            slot = in_items[i].slot;
        } else {
            x = ia[i];
            y = ib[i];
            slot = (uint32_t)i;
        }
        uint32_t lx = len[x], ly = len[y];
        if (lx > ly) {  // pattern = shorter
            const uint32_t t = x; x = y; y = t;
            const uint32_t tl = lx; lx = ly; ly = tl;
        }
        const uint32_t B = (lx + 63) >> 6;
        int lg = lg_gpar;
        while ((uint32_t)(rmax << lg) < B && lg < 5) ++lg;
        uint32_t R = (B + (1u << lg) - 1) >> lg;
        if (R < 1) R = 1;
        uint32_t bucket = (uint32_t)lg * 16 + R;
        if (R > (uint32_t)rmax) bucket = kBuckets - 1;  // too long: flagged below
        items[i] = LevItem{x, y, slot};
        keys[i] = ((uint64_t)bucket << 32) | (uint64_t)(0xffffffffu - ly);
        idx[i] = (uint32_t)i;
        atomicAdd(&sh[bucket], 1u);
        c0 += (unsigned long long)lx * ly;
        c1 += (unsigned long long)(R << lg) * 64ull * ly;
    }
    atomicAdd(&scells[0], c0);
    atomicAdd(&scells[1], c1);
    __syncthreads();
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
    if (threadIdx.x == 0) {
        atomicAdd(&cells[0], scells[0]);
        atomicAdd(&cells[1], scells[1]);
    }
}

__global__ void gather_items(const LevItem* __restrict__ in, const uint32_t* __restrict__ idx,
                             uint64_t n, LevItem* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[idx[i]];
}

void run_planned(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia, const uint32_t* d_ib,
                 const LevItem* d_in_items, uint64_t n, uint32_t* d_out, LevTotals* tot,
                 bool time_kernels) {
    if (n == 0) return;
    if (n > 0xffffffffull) throw invalid_argument("too many distance jobs in one batch");
    cudaStream_t st = ctx->stream;
    const int np = s->planes;
    const int rmax = rmax_for(np);
    const uint64_t target = (uint64_t)ctx->sm_count * 512;  // lanes wanted in flight
    int lg_gpar = 0;
    while (lg_gpar < 5 && (n << lg_gpar) < target) ++lg_gpar;

    // scratch: items(2x), keys(2x), idx(2x), hist, cells, counters, cub temp
    const size_t item_b = n * sizeof(LevItem), key_b = n * 8, idx_b = n * 4;
    size_t cub_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_b, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 40, st);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t hist_b = al(kBuckets * 4 + 16 + kBuckets * 4);
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
    uint32_t* counters = (uint32_t*)(cells + 2);
    base += hist_b;
    void* cub_tmp = base;

    DM_CUDA(cudaMemsetAsync(hist, 0, hist_b, st));
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 8);
    plan_kernel<<<grid, 256, 0, st>>>(d_ia, d_ib, d_in_items, n, s->d_len, lg_gpar, rmax, it0, k0, i0,
                                      hist, cells);
    DM_CUDA(cudaGetLastError());
    DM_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_b, k0, k1, i0, i1, (int)n, 0, 40, st));
    gather_items<<<grid, 256, 0, st>>>(it0, i1, n, it1);
    DM_CUDA(cudaGetLastError());
    unsigned int h[kBuckets];
    unsigned long long hc[2];
    DM_CUDA(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, st));
    DM_CUDA(cudaMemcpyAsync(hc, cells, sizeof(hc), cudaMemcpyDeviceToHost, st));
    DM_CUDA(cudaStreamSynchronize(st));
    if (h[kBuckets - 1])
        throw invalid_argument("sequence too long for the distance engine (max " +
                               std::to_string(32 * rmax * 64) + " residues for this alphabet)");
    if (time_kernels) DM_CUDA(cudaEventRecord(ctx->ev0, st));
    uint64_t start = 0;
    int launches = 0;
    for (int b = 0; b < kBuckets; ++b) {
        if (!h[b]) continue;
        LevArgs a;
        a.items = it1 + start;
        a.nitems = h[b];
        a.lgG = b / 16;
        a.codes = s->d_codes;
        a.off = s->d_off;
        a.len = s->d_len;
        a.blk = s->d_blk;
        a.planes = s->d_planes;
        a.out = d_out;
        a.counter = counters + b;
        launch_bucket(np, b % 16, a, ctx->sm_count, st);
        DM_CUDA(cudaGetLastError());
        start += h[b];
        ++launches;
    }
    if (time_kernels) DM_CUDA(cudaEventRecord(ctx->ev1, st));
    ctx->launches += launches + 2;
    if (tot) {
        tot->cells += hc[0];
        tot->cells_exec += hc[1];
        tot->launches += launches + 2;
        if (time_kernels) {
            DM_CUDA(cudaEventSynchronize(ctx->ev1));
            float ms = 0;
            DM_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            tot->kernel_ms += ms;
        }
    }
}

}  // namespace

void lev_run_host_items(dm_ctx* ctx, const dm_seqset* s, std::vector<LevItem>& items,
                        uint32_t* d_out, LevTotals* tot, bool time_kernels) {
    if (items.empty()) return;
    LevItem* d_items = ctx->aux3.as<LevItem>(items.size());
    DM_CUDA(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(LevItem),
                            cudaMemcpyHostToDevice, ctx->stream));
    run_planned(ctx, s, nullptr, nullptr, d_items, items.size(), d_out, tot, time_kernels);
}

void lev_run_device_pairs(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                          const uint32_t* d_ib, uint64_t n, uint32_t* d_out, LevTotals* tot,
                          bool time_kernels) {
    run_planned(ctx, s, d_ia, d_ib, nullptr, n, d_out, tot, time_kernels);
}

}  // namespace dm
