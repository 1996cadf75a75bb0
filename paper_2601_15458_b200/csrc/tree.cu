// Guide tree (SURVEY.md §2.2 K3/K4 + the level scheduler): divisive
// clustering of cluster_tree.cpp:168-235 with every distance on the GPU.
//
// Per level of the reference's BFS frontier the work is four dependent
// batches: median all-pairs -> center sweep -> pole_l sweep -> pole_r sweep
// (cluster_tree.cpp:76-109). Here:
//   * "big" nodes (more members than the small-subtree threshold T) are run
//     level by level; each phase is ONE distance-engine batch over all big
//     nodes of the level, followed by a reduction kernel (median argmin, sweep
//     argmax, stable partition) that keeps the decision on the device;
//   * a node with 2 <= |C| <= T (T = min(exact_cap, 128)) has every distance
//     its whole subtree will ever ask for inside its own |C|x|C| matrix: the
//     median of a node this small uses all members as candidates
//     (cluster_tree.cpp:128-129) and every descendant works on a subset. So
//     the matrix is computed once (one batch over all such roots) and
//     subtree_kernel resolves the whole subtree in shared memory, one CTA
//     per root. This is exact: no distance is approximated or skipped, only
//     recomputation of identical pairs is avoided.
// Seeds stay on the host, bit-identical: FNV-1a over the current member
// slice (:18-27) -> combine_seed -> mt19937_64 -> Floyd's sample_distinct,
// sorted (rng.hpp:14-59). Ties: argmin/argmax go to the lowest SEQUENCE index
// (:48-50, :159-163); the partition is stable (:98-109); children are numbered
// left then right in frontier order (:212-231) by a final BFS renumbering.
//
// Several attached ranks: the top levels (few nodes with many
// members) shard every distance batch across the ranks (cost-balanced
// ranges, results all-gathered, decisions replicated); once a level holds
// enough nodes (>= DM_OWN_MIN x world, none larger than 1/(DM_OWN_BAL x
// world) of the members) the nodes -- with their whole subtrees -- are assigned to ranks
// (largest first to the least loaded), each rank builds its subtrees with no
// collective, and the ranks exchange the finished subtrees once (node
// records and order slices). Pool ids may differ between ranks; the final
// BFS renumbering depends only on the tree's links, so every rank returns
// the same nodes and order.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <condition_variable>
#include <deque>
#include <functional>
#include <exception>
#include <mutex>
#include <random>
#include <thread>
#include <unordered_set>

#include "comm.h"
#include "dm_internal.h"
#include "nvtx.h"
#include "rng.h"

namespace dm {
namespace {

constexpr uint32_t kNo = 0xffffffffu;
constexpr int kSubMax = 128;  // largest subtree resolved in shared memory

// ---------------------------------------------------------------- host rng (rng.h)
using rng::bounded_draw;
using rng::combine_seed;
using rng::sample_distinct;

uint64_t hash_members(const uint32_t* m, size_t n) {
    uint64_t h = 14695981039346656037ULL;
    for (size_t i = 0; i < n; ++i) {
        h ^= m[i];
        h *= 1099511628211ULL;
    }
    return h;
}

// ------------------------------------------------------------ reductions
// lexicographic (primary, id) keys; argmin prefers smaller, argmax larger
// primary, both prefer the LOWER id on ties.
struct Key {
    uint64_t v;
    uint32_t id;
    uint32_t idx;
};
__device__ __forceinline__ bool better_min(const Key& a, const Key& b) {
    return a.v < b.v || (a.v == b.v && a.id < b.id);
}
__device__ __forceinline__ bool better_max(const Key& a, const Key& b) {
    return a.v > b.v || (a.v == b.v && a.id < b.id);
}
template <bool MIN>
__device__ Key block_reduce(Key k, Key* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        Key t;
        t.v = __shfl_down_sync(0xffffffffu, k.v, o);
        t.id = __shfl_down_sync(0xffffffffu, k.id, o);
        t.idx = __shfl_down_sync(0xffffffffu, k.idx, o);
        if (MIN ? better_min(t, k) : better_max(t, k)) k = t;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
            if (MIN ? better_min(sh[i], k) : better_max(sh[i], k)) k = sh[i];
        sh[0] = k;
    }
    __syncthreads();
    return sh[0];
}

// K3: median of each big node from its k x k candidate matrix (upper triangle
// filled at slot i*k+j, i<j): argmin of uint64 row sums (cluster_tree.cpp:152-165).
__global__ void median_argmin_kernel(const uint32_t* __restrict__ mat, const uint64_t* __restrict__ mat_off,
                                     const uint32_t* __restrict__ kk, const uint32_t* __restrict__ cand,
                                     const uint64_t* __restrict__ cand_off, uint32_t* __restrict__ center) {
    __shared__ Key sh[32];
    const uint32_t v = blockIdx.x;
    const uint32_t k = kk[v];
    const uint32_t* M = mat + mat_off[v];
    const uint32_t* C = cand + cand_off[v];
    Key best{~0ull, kNo, 0};
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        uint64_t s = 0;
        for (uint32_t j = 0; j < k; ++j) {
            if (j == i) continue;
            s += i < j ? M[(uint64_t)i * k + j] : M[(uint64_t)j * k + i];
        }
        Key c{s, C[i], i};
        if (better_min(c, best)) best = c;
    }
    best = block_reduce<true>(best, sh);
    if (threadIdx.x == 0) center[v] = best.id;
}

// K4: radius = max distance, argmax with ties to the lowest sequence index
// (cluster_tree.cpp:44-54, :83-84) over each node's slice of a sweep.
__global__ void sweep_argmax_kernel(const uint32_t* __restrict__ dist, const uint32_t* __restrict__ order,
                                    const uint32_t* __restrict__ nb, const uint32_t* __restrict__ ne,
                                    uint32_t* __restrict__ maxv, uint32_t* __restrict__ argid) {
    __shared__ Key sh[32];
    const uint32_t v = blockIdx.x;
    Key best{0, kNo, 0};
    bool any = false;
    for (uint32_t p = nb[v] + threadIdx.x; p < ne[v]; p += blockDim.x) {
        Key c{dist[p], order[p], p};
        if (!any || better_max(c, best)) best = c;
        any = true;
    }
    if (!any) best = Key{0, kNo, 0};
    best = block_reduce<false>(best, sh);
    if (threadIdx.x == 0) {
        maxv[v] = (uint32_t)best.v;
        argid[v] = best.id;
    }
}

// Stable partition of each node slice: d_l <= d_r to the left
// (cluster_tree.cpp:98-109). One CTA per node; ballot-scan over warps.
__global__ void partition_kernel(uint32_t* __restrict__ order, uint32_t* __restrict__ tmp,
                                 const uint32_t* __restrict__ dl, const uint32_t* __restrict__ dr,
                                 const uint32_t* __restrict__ nb, const uint32_t* __restrict__ ne,
                                 uint32_t* __restrict__ mid) {
    __shared__ uint32_t wcnt[32];
    __shared__ uint32_t base_l, base_r, total_l;
    const uint32_t v = blockIdx.x;
    const uint32_t b = nb[v], e = ne[v];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    // pass 1: count lefts
    uint32_t cnt = 0;
    for (uint32_t p = b + threadIdx.x; p < e; p += blockDim.x) cnt += dl[p] <= dr[p];
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    if (l == 0) wcnt[w] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int i = 0; i < nw; ++i) t += wcnt[i];
        total_l = t;
        base_l = 0;
        base_r = 0;
    }
    __syncthreads();
    const uint32_t L = total_l;
    // pass 2: chunked stable scatter (chunk = blockDim)
    for (uint32_t c0 = b; c0 < e; c0 += blockDim.x) {
        const uint32_t p = c0 + threadIdx.x;
        const bool in = p < e;
        const bool left = in && dl[p] <= dr[p];
        const unsigned ml = __ballot_sync(0xffffffffu, left);
        const unsigned mr = __ballot_sync(0xffffffffu, in && !left);
        __syncthreads();
        if (l == 0) wcnt[w] = __popc(ml) | (__popc(mr) << 16);
        __syncthreads();
        uint32_t pl = 0, pr = 0;
        for (int i = 0; i < w; ++i) {
            pl += wcnt[i] & 0xffff;
            pr += wcnt[i] >> 16;
        }
        const unsigned lt = (1u << l) - 1u;
        if (left) tmp[b + base_l + pl + __popc(ml & lt)] = order[p];
        else if (in) tmp[b + L + base_r + pr + __popc(mr & lt)] = order[p];
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t sl = 0, sr = 0;
            for (int i = 0; i < nw; ++i) {
                sl += wcnt[i] & 0xffff;
                sr += wcnt[i] >> 16;
            }
            base_l += sl;
            base_r += sr;
        }
        __syncthreads();
    }
    for (uint32_t p = b + threadIdx.x; p < e; p += blockDim.x) order[p] = tmp[p];
    if (threadIdx.x == 0) mid[v] = L;
}

// Record of one node of a small subtree; links are local ids.
struct SubRec {
    uint32_t b, e, center, radius, pole_l, pole_r;
    int32_t left, right, parent;
    uint32_t depth;
};

// Resolves a whole subtree of <= kSubMax members from its distance matrix.
__global__ void __launch_bounds__(128) subtree_kernel(
    uint32_t* __restrict__ order, const uint32_t* __restrict__ root_begin, const uint32_t* __restrict__ root_k,
    const uint64_t* __restrict__ mat_off, const uint32_t* __restrict__ mats, const uint64_t* __restrict__ rec_off,
    SubRec* __restrict__ recs, int* __restrict__ err) {
    extern __shared__ uint32_t smem[];
    __shared__ Key sh[32];
    __shared__ uint32_t qb[2 * kSubMax], qe[2 * kSubMax], qd[2 * kSubMax];
    __shared__ int32_t qp[2 * kSubMax];
    __shared__ uint32_t ids[kSubMax], ord[kSubMax], tmp[kSubMax];
    __shared__ uint32_t s_tail, s_bad, s_L;
    const uint32_t r = blockIdx.x;
    const uint32_t k = root_k[r];
    const uint32_t kp = k | 1u;  // odd stride: conflict-free column walks
    uint32_t* D = smem;          // kp * k
    const uint32_t* M = mats + mat_off[r];
    const uint32_t base = root_begin[r];
    SubRec* out = recs + rec_off[r];
    for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
        ids[t] = order[base + t];
        ord[t] = t;
    }
    for (uint32_t x = threadIdx.x; x < k * k; x += blockDim.x) {
        const uint32_t i = x / k, j = x % k;
        D[i * kp + j] = i < j ? M[(uint64_t)i * k + j] : (i > j ? M[(uint64_t)j * k + i] : 0u);
    }
    if (threadIdx.x == 0) {
        qb[0] = 0;
        qe[0] = k;
        qp[0] = -1;
        qd[0] = 0;
        s_tail = 1;
        s_bad = 0;
    }
    __syncthreads();
    for (uint32_t h = 0; h < s_tail; ++h) {
        const uint32_t b = qb[h], e = qe[h], m = e - b;
        if (m == 1) {
            if (threadIdx.x == 0)
                out[h] = SubRec{b, e, ids[ord[b]], 0, kNo, kNo, -1, -1, qp[h], qd[h]};
            __syncthreads();
            continue;
        }
        // median: all members are candidates (m <= exact_cap)
        Key best{~0ull, kNo, 0};
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
            const uint32_t* row = D + ord[b + i] * kp;
            uint64_t s = 0;
            for (uint32_t j = 0; j < m; ++j) s += row[ord[b + j]];
            Key c{s, ids[ord[b + i]], ord[b + i]};
            if (better_min(c, best)) best = c;
        }
        const Key cen = block_reduce<true>(best, sh);
        // radius + pole_l
        Key far{0, kNo, 0};
        bool any = false;
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
            const uint32_t x = ord[b + i];
            Key c{D[cen.idx * kp + x], ids[x], x};
            if (!any || better_max(c, far)) far = c;
            any = true;
        }
        if (!any) far = Key{0, kNo, 0};
        const Key pl = block_reduce<false>(far, sh);
        Key far2{0, kNo, 0};
        any = false;
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
            const uint32_t x = ord[b + i];
            Key c{D[pl.idx * kp + x], ids[x], x};
            if (!any || better_max(c, far2)) far2 = c;
            any = true;
        }
        if (!any) far2 = Key{0, kNo, 0};
        const Key pr = block_reduce<false>(far2, sh);
        if (pr.id == pl.id) {
            if (threadIdx.x == 0) s_bad = 1;
            __syncthreads();
            break;
        }
        // stable partition on warp 0
        if (threadIdx.x < 32) {
            const int l = threadIdx.x;
            const unsigned lt = (1u << l) - 1u;
            uint32_t nl = 0;
            for (uint32_t c0 = 0; c0 < m; c0 += 32) {
                const uint32_t i = c0 + l;
                const uint32_t x = i < m ? ord[b + i] : 0;
                const bool f = i < m && D[pl.idx * kp + x] <= D[pr.idx * kp + x];
                const unsigned msk = __ballot_sync(0xffffffffu, f);
                if (f) tmp[nl + __popc(msk & lt)] = x;
                nl += __popc(msk);
            }
            uint32_t nr = nl;
            for (uint32_t c0 = 0; c0 < m; c0 += 32) {
                const uint32_t i = c0 + l;
                const uint32_t x = i < m ? ord[b + i] : 0;
                const bool f = i < m && !(D[pl.idx * kp + x] <= D[pr.idx * kp + x]);
                const unsigned msk = __ballot_sync(0xffffffffu, f);
                if (f) tmp[nr + __popc(msk & lt)] = x;
                nr += __popc(msk);
            }
            if (l == 0) s_L = nl;
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) ord[b + i] = tmp[i];
        if (threadIdx.x == 0) {
            const uint32_t L = s_L, t = s_tail;
            uint32_t radius = D[cen.idx * kp + pl.idx];
            out[h] = SubRec{b, e, cen.id, radius, pl.id, pr.id, (int32_t)t, (int32_t)t + 1, qp[h], qd[h]};
            qb[t] = b; qe[t] = b + L; qp[t] = (int32_t)h; qd[t] = qd[h] + 1;
            qb[t + 1] = b + L; qe[t + 1] = e; qp[t + 1] = (int32_t)h; qd[t + 1] = qd[h] + 1;
            s_tail = t + 2;
        }
        __syncthreads();
    }
    if (s_bad) {
        if (threadIdx.x == 0) atomicExch(err, 1);
        return;
    }
    for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) order[base + t] = ids[ord[t]];
}

// ------------------------------------------------------------ distance jobs on the device
// All-pairs jobs (i < j) of each node's member list src[src_off[v] .. + k[v]),
// result slot mat_off[v] + i k + j; node v's jobs start at item_off[v],
// row i at i (2k - i - 1) / 2 -- the order the host loops produced.
__global__ void pair_items_kernel(const uint32_t* __restrict__ src, const uint64_t* __restrict__ src_off,
                                  const uint32_t* __restrict__ kk, const uint64_t* __restrict__ mat_off,
                                  const uint64_t* __restrict__ item_off, LevItem* __restrict__ items) {
    const uint32_t v = blockIdx.x, k = kk[v];
    const uint32_t* c = src + src_off[v];
    const uint64_t mo = mat_off[v];
    for (uint32_t i = 0; i + 1 < k; ++i) {
        LevItem* row = items + item_off[v] + (uint64_t)i * (2ull * k - i - 1) / 2 - (i + 1);
        const uint32_t ci = c[i];
        for (uint32_t j = i + 1 + threadIdx.x; j < k; j += blockDim.x)
            row[j] = LevItem{ci, c[j], mo + (uint64_t)i * k + j};
    }
}

// Sweep jobs: from[v] against every member of node v's slice of `order`,
// result slot = the member's position (cluster_tree.cpp:31-41).
__global__ void sweep_items_kernel(const uint32_t* __restrict__ from, const uint32_t* __restrict__ order,
                                   const uint32_t* __restrict__ nb, const uint32_t* __restrict__ ne,
                                   const uint64_t* __restrict__ item_off, LevItem* __restrict__ items) {
    const uint32_t v = blockIdx.x, f = from[v], b = nb[v];
    LevItem* out = items + item_off[v] - b;
    for (uint32_t p = b + threadIdx.x; p < ne[v]; p += blockDim.x) out[p] = LevItem{f, order[p], p};
}

// ------------------------------------------------------------ host side
struct PNode {
    uint32_t begin = 0, end = 0, center = kNo, radius = 0, pole_l = kNo, pole_r = kNo;
    int32_t left = -1, right = -1, parent = -1;
    uint32_t depth = 0;
};

template <class T>
T* upload(dm_ctx* ctx, DevBuf& buf, const std::vector<T>& v) {
    T* d = buf.as<T>(std::max<size_t>(v.size(), 1));
    if (!v.empty()) DM_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return d;
}
template <class T>
void download(dm_ctx* ctx, std::vector<T>& v, const T* d, size_t n) {
    v.resize(n);
    if (n) DM_CUDA(cudaMemcpyAsync(v.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
}

struct TreeScratch {
    DevBuf order, tmp, dc, dl, dr, mat, matoff, kk, cand, candoff, nb, ne, res1, res2, res3, res4, res5, res6, sub_begin,
        sub_k, sub_mat, sub_matoff, sub_recoff, sub_recs, err, items, itemoff, ckeys, cvals, cfill;
    explicit TreeScratch(cudaStream_t* s) {
        for (DevBuf* b : {&order, &tmp, &dc, &dl, &dr, &mat, &matoff, &kk, &cand, &candoff, &nb, &ne, &res1, &res2,
                          &res3, &res4, &res5, &res6, &sub_begin, &sub_k, &sub_mat, &sub_matoff, &sub_recoff, &sub_recs, &err,
                          &items, &itemoff, &ckeys, &cvals, &cfill})
            b->sp = s;
    }
};

const char* kDedupMsg = "cluster contains identical sequences; input was not de-duplicated";

// Subtree ownership exchange (several ranks): rank blobs hold
//   [n_roots u64][n_new u64] { root pool id u32, PNode } x n_roots
//   PNode x n_new { order slice of each root } x n_roots
// with node links < P0 global pool ids and >= P0 the sender's local ids.
void put(std::vector<uint8_t>& b, const void* p, size_t n) {
    const uint8_t* c = static_cast<const uint8_t*>(p);
    b.insert(b.end(), c, c + n);
}
template <class T>
T take(const std::vector<uint8_t>& b, size_t& at) {
    T v;
    std::memcpy(&v, b.data() + at, sizeof(T));
    at += sizeof(T);
    return v;
}

void exchange_subtrees(dm_ctx* ctx, std::vector<PNode>& pool, std::vector<uint32_t>& order, uint32_t P0,
                       const std::vector<uint32_t>& roots, const std::vector<int>& owner) {
    std::vector<uint8_t> mine;
    uint64_t nr = 0;
    for (size_t i = 0; i < roots.size(); ++i) nr += owner[i] == ctx->rank;
    const uint64_t nn = pool.size() - P0;
    put(mine, &nr, 8);
    put(mine, &nn, 8);
    for (size_t i = 0; i < roots.size(); ++i)
        if (owner[i] == ctx->rank) {
            put(mine, &roots[i], 4);
            put(mine, &pool[roots[i]], sizeof(PNode));
        }
    if (nn) put(mine, &pool[P0], nn * sizeof(PNode));
    for (size_t i = 0; i < roots.size(); ++i)
        if (owner[i] == ctx->rank) {
            const PNode& p = pool[roots[i]];
            put(mine, order.data() + p.begin, (size_t)(p.end - p.begin) * 4);
        }
    std::vector<std::vector<uint8_t>> all;
    comm_allgatherv_host(ctx, mine, all);
    for (int r = 0; r < ctx->world; ++r) {
        if (r == ctx->rank) continue;
        const std::vector<uint8_t>& b = all[r];
        size_t at = 0;
        const uint64_t rn = take<uint64_t>(b, at), rnew = take<uint64_t>(b, at);
        const uint32_t base = (uint32_t)pool.size();
        auto remap = [&](int32_t l) -> int32_t { return l < (int32_t)P0 ? l : (int32_t)(base + (uint32_t)l - P0); };
        auto fix = [&](PNode p) {
            p.left = p.left < 0 ? -1 : remap(p.left);
            p.right = p.right < 0 ? -1 : remap(p.right);
            p.parent = p.parent < 0 ? -1 : remap(p.parent);
            return p;
        };
        std::vector<uint32_t> rid(rn);
        for (uint64_t k = 0; k < rn; ++k) {
            rid[k] = take<uint32_t>(b, at);
            pool[rid[k]] = fix(take<PNode>(b, at));
        }
        for (uint64_t k = 0; k < rnew; ++k) pool.push_back(fix(take<PNode>(b, at)));
        for (uint64_t k = 0; k < rn; ++k) {
            const PNode& p = pool[rid[k]];
            std::memcpy(order.data() + p.begin, b.data() + at, (size_t)(p.end - p.begin) * 4);
            at += (size_t)(p.end - p.begin) * 4;
        }
    }
}

}  // namespace

// Low-priority context for the tree's background batches (one per context,
// kept for reuse; destroyed with it): own stream, scratch and side streams at
// the default (least) priority, while the context's own distance batches run
// on side streams of the greatest priority.
dm_ctx* tree_bg_context(dm_ctx* ctx) {
    if (!ctx->tree_bg) {
        auto* p = new dm_ctx;
        p->device = ctx->device;
        p->sm_count = ctx->sm_count;
        int least = 0, greatest = 0;
        DM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        if (cudaStreamCreateWithPriority(&p->stream, cudaStreamNonBlocking, least) != cudaSuccess) {
            delete p;
            throw cuda_error("cannot create the tree's background stream");
        }
        p->own_stream = p->stream;
        p->side_prio = 0;
        // short-lived blocks: the foreground batches' kernels (higher priority)
        // take SM slots as soon as a background block retires -- there is no
        // preemption, and 4-wave blocks held slots for ~1/4 of a batch
        p->lev_waves = 32;
        DM_CUDA(cudaEventCreate(&p->ev0));
        DM_CUDA(cudaEventCreate(&p->ev1));
        ctx->tree_bg = p;
    }
    return ctx->tree_bg;
}

void build_tree(dm_ctx* ctx, const dm_seqset* s, uint64_t seed, uint64_t exact_cap_in,
                std::vector<dm_node>& nodes_out, std::vector<uint32_t>& order, dm_stats* st) {
    NvtxRange nvtx_tree("dm build_tree");
    const uint32_t n = s->n;
    if (n == 0) throw runtime_error("cannot build a cluster tree from zero sequences");
    const uint64_t exact_cap = std::max<uint64_t>(2, exact_cap_in);
    const uint32_t T = (uint32_t)std::min<uint64_t>(exact_cap, kSubMax);
    cudaStream_t stream = ctx->stream;
    TreeScratch sc(&ctx->stream);
    LevTotals tot;
    const bool timing = st != nullptr;

    order.resize(n);
    std::iota(order.begin(), order.end(), 0u);
    std::vector<PNode> pool(1);
    pool[0].begin = 0;
    pool[0].end = n;
    std::vector<uint32_t> big, small;
    if (n == 1) pool[0].center = 0;
    else if (n <= T) small.push_back(0);
    else big.push_back(0);

    uint32_t* d_order = upload(ctx, sc.order, order);
    uint32_t* d_tmp = sc.tmp.as<uint32_t>(n);
    uint32_t* d_dc = sc.dc.as<uint32_t>(n);
    uint32_t* d_dl = sc.dl.as<uint32_t>(n);
    uint32_t* d_dr = sc.dr.as<uint32_t>(n);
    std::vector<LevItem> items;

    // Distances already computed in this build (DistCache, dm_internal.h):
    // the device-item batches (one rank, or subtrees a rank owns) look their
    // pairs up and add their results; ~30 % of the tree's cells are pairs it
    // asked for before (a center is a median candidate, a child's sample and
    // a small subtree's matrix overlap the parent's matrix and pole sweeps).
    // Sized for ~256 inserts per sequence (cfg4: ~135); inserts stop at a
    // 5/8 load, lookups never fail.
    // DM_TREE_CACHE=0 turns it off; =k (10 <= k <= 30) forces 2^k slots (tests:
    // a full table, long probe chains).
    DistCache cache, cache_ins;
    const int cache_env = [] {
        const char* e = std::getenv("DM_TREE_CACHE");
        return e ? std::atoi(e) : 1;
    }();
    if (n > T && cache_env != 0) {
        uint64_t cap = 1ull << 12;
        while (cap < (uint64_t)n * 256 && cap < (1ull << 28)) cap <<= 1;
        if (cache_env >= 10 && cache_env <= 30) cap = 1ull << cache_env;
        cache.keys = sc.ckeys.as<unsigned long long>(cap);
        cache.vals = sc.cvals.as<uint32_t>(cap);
        cache.fill = sc.cfill.as<unsigned int>(1);
        cache.mask = cap - 1;
        cache.max_fill = (unsigned int)(cap / 8 * 5);
        DM_CUDA(cudaMemsetAsync(cache.keys, 0xff, cap * sizeof(unsigned long long), stream));
        DM_CUDA(cudaMemsetAsync(cache.vals, 0xff, cap * sizeof(uint32_t), stream));
        DM_CUDA(cudaMemsetAsync(cache.fill, 0, sizeof(unsigned int), stream));
        cache_ins = cache;
        cache_ins.insert = true;
    }
    const DistCache* dc_look = cache.on() ? &cache : nullptr;       // lookups only
    const DistCache* dc_ins = cache.on() ? &cache_ins : nullptr;    // lookups + inserts

    const bool trace = std::getenv("DM_TRACE") != nullptr;
    auto tnow = [&] {
        if (trace) DM_CUDA(cudaStreamSynchronize(stream));
        return std::chrono::steady_clock::now();
    };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    // subtree ownership (several attached ranks), see the header
    const bool real = comm_real(ctx);
    const int wr = ctx->world;
    const uint64_t own_min = [] {
        const char* e = std::getenv("DM_OWN_MIN");
        return e ? (uint64_t)std::max(1, std::atoi(e)) : (uint64_t)4;
    }();
    // no owned node may exceed 1/(DM_OWN_BAL x world) of the level's members (0: no limit)
    const uint64_t own_bal = [] {
        const char* e = std::getenv("DM_OWN_BAL");
        return e ? (uint64_t)std::max(0, std::atoi(e)) : (uint64_t)2;
    }();
    bool owned = false;
    uint32_t P0 = 0;
    std::vector<uint32_t> own_roots;
    std::vector<int> own_of;
    auto try_own = [&] {
        if (!real || owned) return;
        uint64_t members = 0, mx = 0;
        for (uint32_t id : big) {
            const uint64_t m = pool[id].end - pool[id].begin;
            members += m;
            mx = std::max(mx, m);
        }
        if (big.size() < own_min * (uint64_t)wr || mx * own_bal * (uint64_t)wr > members) return;
        own_roots.assign(big.begin(), big.end());
        own_roots.insert(own_roots.end(), small.begin(), small.end());
        std::vector<uint64_t> cost(own_roots.size());
        for (size_t i = 0; i < own_roots.size(); ++i) {
            const uint64_t m = pool[own_roots[i]].end - pool[own_roots[i]].begin;
            uint64_t lg = 0;
            while ((m >> lg) > 128) ++lg;
            cost[i] = m * (64 + 3 * lg);  // sweeps per level + median/all-pairs work, per member
        }
        assign_lpt(cost.data(), cost.size(), wr, own_of);
        std::vector<uint32_t> nb2, ns2;
        for (size_t i = 0; i < own_roots.size(); ++i)
            if (own_of[i] == ctx->rank) (i < big.size() ? nb2 : ns2).push_back(own_roots[i]);
        big.swap(nb2);
        small.swap(ns2);
        owned = true;
        ctx->own_tree += big.size() + small.size();
        P0 = (uint32_t)pool.size();
        if (trace)
            std::fprintf(stderr, "[dm tree] rank %d/%d owns %zu + %zu of %zu subtrees\n", ctx->rank, wr, big.size(),
                         small.size(), own_roots.size());
    };
    int level = 0;
    int err_flag = 0;

    // Background batches (one rank): the all-pairs matrices of the small
    // subtrees a level creates are computed on a low-priority context while
    // the later levels run, filling the SM slots their batches' tails leave
    // idle; subtree_kernel resolves them all at the end. Every small
    // subtree's matrix lies at its offset in one buffer (sum k^2 <= n T).
    const bool bg_on = shard_world(ctx) == 1 && [] {
        const char* e = std::getenv("DM_TREE_BG");
        return !(e && e[0] == '0');
    }();
    dm_ctx* bg = bg_on ? tree_bg_context(ctx) : nullptr;
    uint32_t* d_submat = bg_on ? sc.sub_mat.as<uint32_t>((uint64_t)n * T + 1) : nullptr;
    struct BgJob {
        cudaEvent_t ready = nullptr;
        std::vector<uint64_t> soff, moff, ioff;
        std::vector<uint32_t> sk;
        uint64_t itot = 0;
    };
    struct BgState {
        std::mutex mu;
        std::condition_variable cv;
        std::deque<BgJob> q;
        bool done = false;
        std::exception_ptr err;
        LevTotals tot;
    } bgs;
    std::thread bg_thread;
    size_t bg_sent = 0;
    uint64_t bg_mtot = 0;
    std::vector<cudaEvent_t> bg_events;
    if (bg_on)
        bg_thread = std::thread([&] {
            try {
                DM_CUDA(cudaSetDevice(ctx->device));
                DevBuf b_soff(&bg->stream), b_sk(&bg->stream), b_moff(&bg->stream), b_ioff(&bg->stream),
                    b_items(&bg->stream);
                for (;;) {
                    BgJob job;
                    {
                        std::unique_lock<std::mutex> g(bgs.mu);
                        bgs.cv.wait(g, [&] { return bgs.done || !bgs.q.empty(); });
                        if (bgs.q.empty()) return;
                        job = std::move(bgs.q.front());
                        bgs.q.pop_front();
                    }
                    DM_CUDA(cudaStreamWaitEvent(bg->stream, job.ready, 0));  // the level's partition is done
                    const size_t S = job.sk.size();
                    LevItem* d_items = b_items.as<LevItem>(std::max<uint64_t>(job.itot, 1));
                    pair_items_kernel<<<(unsigned)S, 128, 0, bg->stream>>>(
                        d_order, upload(bg, b_soff, job.soff), upload(bg, b_sk, job.sk), upload(bg, b_moff, job.moff),
                        upload(bg, b_ioff, job.ioff), d_items);
                    DM_CUDA(cudaGetLastError());
                    lev_run_device_items(bg, s, d_items, job.itot, d_submat, &bgs.tot, false, dc_look);
                    bgs.tot.launches += 1;
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(bgs.mu);
                bgs.err = std::current_exception();
            }
        });
    auto stop_bg = [&] {
        if (!bg_thread.joinable()) return;
        {
            std::lock_guard<std::mutex> g(bgs.mu);
            bgs.done = true;
        }
        bgs.cv.notify_all();
        bg_thread.join();
    };
    struct BgGuard {  // error paths: the worker is stopped before the scratch it uses goes away
        std::function<void()> f;
        ~BgGuard() { f(); }
    } bg_guard{[&] {
        stop_bg();
        for (cudaEvent_t e : bg_events) cudaEventDestroy(e);
        if (bg) cudaStreamSynchronize(bg->stream);
    }};
    // the small subtrees made so far go to the background worker (their slices
    // of d_order are final once the work queued on `stream` so far is done)
    auto dispatch_bg = [&] {
        if (!bg_on || bg_sent == small.size()) return;
        BgJob job;
        for (size_t r = bg_sent; r < small.size(); ++r) {
            const PNode& nd = pool[small[r]];
            const uint32_t k = nd.end - nd.begin;
            job.soff.push_back(nd.begin);
            job.sk.push_back(k);
            job.moff.push_back(bg_mtot);
            job.ioff.push_back(job.itot);
            job.itot += (uint64_t)k * (k - 1) / 2;
            bg_mtot += (uint64_t)k * k;
        }
        DM_CUDA(cudaEventCreateWithFlags(&job.ready, cudaEventDisableTiming));
        bg_events.push_back(job.ready);
        DM_CUDA(cudaEventRecord(job.ready, stream));
        {
            std::lock_guard<std::mutex> g(bgs.mu);
            bgs.q.push_back(std::move(job));
        }
        bgs.cv.notify_all();
        bg_sent = small.size();
    };
    try_own();
    while (!big.empty()) {
        NvtxRange nvtx_level("dm tree level");
        const size_t B = big.size();
        const auto t0 = tnow();
        if (trace) lev_finish_timing(tot);
        const float k0 = tot.kernel_ms;
        // One rank (or an owned subtree): the jobs of every batch are generated
        // on the device from the candidate lists / node slices and the level's
        // decisions stay there until one download at the end of the level.
        // Several ranks sharing the level: host job lists, sharded by cost.
        const bool dev = owned || shard_world(ctx) == 1;
        // ---- phase 1: median candidates (host seeds) + all-pairs batch
        std::vector<uint64_t> mat_off(B), cand_off(B), item_off(B);
        std::vector<uint32_t> kk(B), cand, nb(B), ne(B);
        uint64_t mtot = 0, itot = 0;
        items.clear();
        for (size_t v = 0; v < B; ++v) {
            const PNode& nd = pool[big[v]];
            const uint32_t m = nd.end - nd.begin;
            nb[v] = nd.begin;
            ne[v] = nd.end;
            cand_off[v] = cand.size();
            const uint32_t* mem = order.data() + nd.begin;
            if (m <= exact_cap) {
                cand.insert(cand.end(), mem, mem + m);
            } else {
                const uint64_t node_seed = combine_seed(seed, hash_members(mem, m));
                std::mt19937_64 g(node_seed);
                for (uint64_t p : sample_distinct(g, m, exact_cap)) cand.push_back(mem[p]);
            }
            const uint32_t k = (uint32_t)(cand.size() - cand_off[v]);
            kk[v] = k;
            mat_off[v] = mtot;
            item_off[v] = itot;
            itot += (uint64_t)k * (k - 1) / 2;
            if (!dev) {
                const uint32_t* c = cand.data() + cand_off[v];
                for (uint32_t i = 0; i < k; ++i)
                    for (uint32_t j = i + 1; j < k; ++j)
                        items.push_back(LevItem{c[i], c[j], mtot + (uint64_t)i * k + j});
            }
            mtot += (uint64_t)k * k;
        }
        uint32_t* d_mat = sc.mat.as<uint32_t>(mtot);
        const uint32_t* d_cand = upload(ctx, sc.cand, cand);
        const uint64_t* d_candoff = upload(ctx, sc.candoff, cand_off);
        const uint32_t* d_kk = upload(ctx, sc.kk, kk);
        const uint64_t* d_matoff = upload(ctx, sc.matoff, mat_off);
        if (dev) {
            LevItem* d_items = sc.items.as<LevItem>(std::max<uint64_t>(itot, 1));
            pair_items_kernel<<<(unsigned)B, 128, 0, stream>>>(d_cand, d_candoff, d_kk, d_matoff,
                                                               upload(ctx, sc.itemoff, item_off), d_items);
            DM_CUDA(cudaGetLastError());
            lev_run_device_items(ctx, s, d_items, itot, d_mat, &tot, timing, dc_ins);
        } else {
            lev_run_host_items(ctx, s, items, d_mat, &tot, timing, owned);
        }
        const auto t_med = tnow();
        uint32_t* d_center = sc.res1.as<uint32_t>(B);
        median_argmin_kernel<<<(unsigned)B, 128, 0, stream>>>(d_mat, d_matoff, d_kk, d_cand, d_candoff, d_center);
        DM_CUDA(cudaGetLastError());
        std::vector<uint32_t> center, radius, pole_l, pole_r, mids;
        if (!dev) {
            download(ctx, center, d_center, B);
            DM_CUDA(cudaStreamSynchronize(stream));
        }
        uint32_t* d_nb = upload(ctx, sc.nb, nb);
        uint32_t* d_ne = upload(ctx, sc.ne, ne);
        std::vector<uint64_t> sweep_off(B);
        uint64_t nsweep = 0;
        for (size_t v = 0; v < B; ++v) {
            sweep_off[v] = nsweep;
            nsweep += ne[v] - nb[v];
        }
        const uint64_t* d_sweepoff = dev ? upload(ctx, sc.itemoff, sweep_off) : nullptr;

        // ---- phases 2-4: sweeps from center, pole_l, pole_r
        double sw_build = 0, sw_run = 0;
        auto sweep = [&](const uint32_t* d_from, const std::vector<uint32_t>& from, uint32_t* d_dist) {
            const auto a0 = tnow();
            if (dev) {
                LevItem* d_items = sc.items.as<LevItem>(std::max<uint64_t>(nsweep, 1));
                sweep_items_kernel<<<(unsigned)B, 256, 0, stream>>>(d_from, d_order, d_nb, d_ne, d_sweepoff, d_items);
                DM_CUDA(cudaGetLastError());
                const auto a1 = tnow();
                lev_run_device_items(ctx, s, d_items, nsweep, d_dist, &tot, timing, dc_ins);
                sw_build += ms(a0, a1);
                sw_run += ms(a1, tnow());
                return;
            }
            items.clear();
            for (size_t v = 0; v < B; ++v)
                for (uint32_t p = nb[v]; p < ne[v]; ++p) items.push_back(LevItem{from[v], order[p], p});
            const auto a1 = tnow();
            lev_run_host_items(ctx, s, items, d_dist, &tot, timing, owned);
            const auto a2 = tnow();
            sw_build += ms(a0, a1);
            sw_run += ms(a1, a2);
        };
        uint32_t* d_max = sc.res2.as<uint32_t>(B);
        uint32_t* d_pl = sc.res3.as<uint32_t>(B);
        uint32_t* d_pr = sc.res4.as<uint32_t>(B);
        uint32_t* d_max2 = sc.res6.as<uint32_t>(B);
        sweep(d_center, center, d_dc);
        sweep_argmax_kernel<<<(unsigned)B, 256, 0, stream>>>(d_dc, d_order, d_nb, d_ne, d_max, d_pl);
        DM_CUDA(cudaGetLastError());
        if (!dev) {
            download(ctx, radius, d_max, B);
            download(ctx, pole_l, d_pl, B);
            DM_CUDA(cudaStreamSynchronize(stream));
        }
        sweep(d_pl, pole_l, d_dl);
        sweep_argmax_kernel<<<(unsigned)B, 256, 0, stream>>>(d_dl, d_order, d_nb, d_ne, d_max2, d_pr);
        DM_CUDA(cudaGetLastError());
        auto dup_found = [&] {
            bool dup = false;
            for (size_t v = 0; v < B; ++v) dup = dup || pole_r[v] == pole_l[v];
            return dup;
        };
        if (!dev) {
            download(ctx, pole_r, d_pr, B);
            DM_CUDA(cudaStreamSynchronize(stream));
            if (dup_found()) {
                if (!owned) throw runtime_error(kDedupMsg);
                err_flag = 1;  // reported by every rank after the exchange
                break;
            }
        }
        // (one rank: with identical poles the last sweep and the partition are
        // wasted work, the error is raised below before any node is made)
        sweep(d_pr, pole_r, d_dr);
        uint32_t* d_mid = sc.res5.as<uint32_t>(B);
        partition_kernel<<<(unsigned)B, 256, 0, stream>>>(d_order, d_tmp, d_dl, d_dr, d_nb, d_ne, d_mid);
        DM_CUDA(cudaGetLastError());
        if (dev) {
            download(ctx, center, d_center, B);
            download(ctx, radius, d_max, B);
            download(ctx, pole_l, d_pl, B);
            download(ctx, pole_r, d_pr, B);
        }
        download(ctx, mids, d_mid, B);
        DM_CUDA(cudaMemcpyAsync(order.data(), d_order, (size_t)n * 4, cudaMemcpyDeviceToHost, stream));
        DM_CUDA(cudaStreamSynchronize(stream));
        if (dev && dup_found()) {
            if (!owned) throw runtime_error(kDedupMsg);
            err_flag = 1;  // reported by every rank after the exchange
            break;
        }
        ctx->launches += 4 + (dev ? 4 : 0);
        tot.launches += 4 + (dev ? 4 : 0);

        // ---- children (cluster_tree.cpp:201-231)
        std::vector<uint32_t> next;
        for (size_t v = 0; v < B; ++v) {
            const uint32_t id = big[v];
            pool[id].center = center[v];
            pool[id].radius = radius[v];
            pool[id].pole_l = pole_l[v];
            pool[id].pole_r = pole_r[v];
            const uint32_t b = pool[id].begin, e = pool[id].end, mid = b + mids[v];
            const uint32_t depth = pool[id].depth + 1;
            for (int side = 0; side < 2; ++side) {
                PNode c;
                c.begin = side ? mid : b;
                c.end = side ? e : mid;
                c.parent = (int32_t)id;
                c.depth = depth;
                const uint32_t cid = (uint32_t)pool.size();
                (side ? pool[id].right : pool[id].left) = (int32_t)cid;
                const uint32_t m = c.end - c.begin;
                if (m == 1) c.center = order[c.begin];
                pool.push_back(c);
                if (m >= 2) (m <= T ? small : next).push_back(cid);
            }
        }
        if (trace) {
            const auto t5 = tnow();
            lev_finish_timing(tot);
            uint64_t mem = 0;
            for (size_t v = 0; v < B; ++v) mem += ne[v] - nb[v];
            std::fprintf(stderr,
                         "[dm tree] level %d big %zu members %llu median %.3f ms sweeps %.3f ms (items %.3f, distance "
                         "batches %.3f) total %.3f ms, distance kernels %.3f ms\n",
                         level, B, (unsigned long long)mem, ms(t0, t_med), ms(t_med, t5), sw_build, sw_run, ms(t0, t5),
                         tot.kernel_ms - k0);
        }
        ++level;
        big.swap(next);
        dispatch_bg();
        try_own();
    }
    if (bg_on && !err_flag) {
        dispatch_bg();  // the rest (e.g. a root small enough from the start)
        stop_bg();
        if (bgs.err) std::rethrow_exception(bgs.err);
        DM_CUDA(cudaEventRecord(bg->ev1, bg->stream));
        DM_CUDA(cudaStreamWaitEvent(stream, bg->ev1, 0));
        if (trace) {
            const auto w0 = std::chrono::steady_clock::now();
            DM_CUDA(cudaEventSynchronize(bg->ev1));
            std::fprintf(stderr, "[dm tree] background all-pairs: %zu small subtrees, waited %.3f ms after the levels\n",
                         small.size(), ms(w0, std::chrono::steady_clock::now()));
        }
        tot.cells += bgs.tot.cells;
        tot.cells_exec += bgs.tot.cells_exec;
        tot.reused += bgs.tot.reused;
        tot.cells_reused += bgs.tot.cells_reused;
        tot.launches += bgs.tot.launches;
        ctx->launches += bg->launches;
        bg->launches = 0;
    }

    // ---- small subtrees: one all-pairs matrix each, resolved on the device
    if (!small.empty() && !err_flag) {
        NvtxRange nvtx_small("dm tree small subtrees");
        const size_t S = small.size();
        const bool dev = owned || shard_world(ctx) == 1;  // jobs generated on the device (see the level loop)
        std::vector<uint32_t> sb(S), sk(S);
        std::vector<uint64_t> moff(S), roff(S), ioff(S), soff(S);
        uint64_t mtot = 0, rtot = 0, itot = 0;
        items.clear();
        for (size_t r = 0; r < S; ++r) {
            const PNode& nd = pool[small[r]];
            const uint32_t k = nd.end - nd.begin;
            sb[r] = nd.begin;
            soff[r] = nd.begin;
            sk[r] = k;
            moff[r] = mtot;
            roff[r] = rtot;
            ioff[r] = itot;
            itot += (uint64_t)k * (k - 1) / 2;
            if (!dev && !bg_on) {
                const uint32_t* mem = order.data() + nd.begin;
                for (uint32_t i = 0; i < k; ++i)
                    for (uint32_t j = i + 1; j < k; ++j)
                        items.push_back(LevItem{mem[i], mem[j], mtot + (uint64_t)i * k + j});
            }
            mtot += (uint64_t)k * k;
            rtot += 2ull * k - 1;
        }
        const auto s0 = tnow();
        uint32_t* d_mat = bg_on ? d_submat : sc.sub_mat.as<uint32_t>(mtot);
        const uint32_t* d_sk = upload(ctx, sc.sub_k, sk);
        const uint64_t* d_smatoff = upload(ctx, sc.sub_matoff, moff);
        if (bg_on) {
            // computed in the background (same order, same offsets)
        } else if (dev) {
            LevItem* d_items = sc.items.as<LevItem>(std::max<uint64_t>(itot, 1));
            pair_items_kernel<<<(unsigned)S, 128, 0, stream>>>(d_order, upload(ctx, sc.candoff, soff), d_sk, d_smatoff,
                                                               upload(ctx, sc.itemoff, ioff), d_items);
            DM_CUDA(cudaGetLastError());
            lev_run_device_items(ctx, s, d_items, itot, d_mat, &tot, timing, dc_look);
            ctx->launches += 1;
            tot.launches += 1;
        } else {
            lev_run_host_items(ctx, s, items, d_mat, &tot, timing, owned);
        }
        const auto s1 = tnow();
        if (trace)
            std::fprintf(stderr, "[dm tree] small subtrees %zu pairs %llu all-pairs %.3f ms\n", S,
                         (unsigned long long)itot, ms(s0, s1));
        SubRec* d_recs = sc.sub_recs.as<SubRec>(rtot);
        int* d_err = sc.err.as<int>(1);
        DM_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), stream));
        const size_t smem = (size_t)(T | 1u) * T * 4;
        DM_CUDA(cudaFuncSetAttribute(subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        subtree_kernel<<<(unsigned)S, 128, smem, stream>>>(d_order, upload(ctx, sc.sub_begin, sb), d_sk, d_smatoff,
                                                           d_mat, upload(ctx, sc.sub_recoff, roff), d_recs, d_err);
        DM_CUDA(cudaGetLastError());
        ctx->launches += 1;
        tot.launches += 1;
        std::vector<SubRec> recs;
        download(ctx, recs, d_recs, rtot);
        int err = 0;
        DM_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, stream));
        DM_CUDA(cudaMemcpyAsync(order.data(), d_order, (size_t)n * 4, cudaMemcpyDeviceToHost, stream));
        DM_CUDA(cudaStreamSynchronize(stream));
        if (err && !owned) throw runtime_error(kDedupMsg);
        if (err) err_flag = 1;
        for (size_t r = 0; r < S; ++r) {
            const uint32_t root = small[r];
            const uint32_t k = sk[r];
            const SubRec* R = recs.data() + roff[r];
            const uint32_t nloc = 2 * k - 1;
            std::vector<uint32_t> gid(nloc);
            gid[0] = root;
            for (uint32_t h = 1; h < nloc; ++h) {
                gid[h] = (uint32_t)pool.size();
                pool.emplace_back();
            }
            const uint32_t b0 = pool[root].begin, d0 = pool[root].depth;
            const int32_t par0 = pool[root].parent;
            for (uint32_t h = 0; h < nloc; ++h) {
                PNode& p = pool[gid[h]];
                p.begin = b0 + R[h].b;
                p.end = b0 + R[h].e;
                p.center = R[h].center;
                p.radius = R[h].radius;
                p.pole_l = R[h].pole_l;
                p.pole_r = R[h].pole_r;
                p.left = R[h].left < 0 ? -1 : (int32_t)gid[R[h].left];
                p.right = R[h].right < 0 ? -1 : (int32_t)gid[R[h].right];
                p.parent = h == 0 ? par0 : (int32_t)gid[R[h].parent];
                p.depth = d0 + R[h].depth;
            }
        }
    }

    if (owned) {
        int bad = err_flag;  // a duplicate found by any rank fails every rank
        std::vector<int> allbad((size_t)wr);
        comm_allgather_host(ctx, &bad, allbad.data(), sizeof(int));
        for (int b : allbad)
            if (b) throw runtime_error(kDedupMsg);
        exchange_subtrees(ctx, pool, order, P0, own_roots, own_of);
    }

    // ---- BFS renumbering = the reference's level-synchronous numbering
    nodes_out.clear();
    nodes_out.reserve(pool.size());
    std::vector<uint32_t> q{0};
    std::vector<int32_t> newid(pool.size(), -1);
    newid[0] = 0;
    for (size_t h = 0; h < q.size(); ++h) {
        const PNode& p = pool[q[h]];
        if (p.left >= 0) {
            newid[p.left] = (int32_t)q.size();
            q.push_back((uint32_t)p.left);
            newid[p.right] = (int32_t)q.size();
            q.push_back((uint32_t)p.right);
        }
    }
    for (uint32_t id : q) {
        const PNode& p = pool[id];
        dm_node d;
        d.begin = p.begin;
        d.end = p.end;
        d.center = p.center;
        d.radius = p.radius;
        d.pole_l = p.pole_l;
        d.pole_r = p.pole_r;
        d.left = p.left < 0 ? -1 : newid[p.left];
        d.right = p.right < 0 ? -1 : newid[p.right];
        d.parent = p.parent < 0 ? -1 : newid[p.parent];
        d.depth = p.depth;
        nodes_out.push_back(d);
    }
    if (trace)
        std::fprintf(stderr, "[dm tree] distance cache: %llu jobs / %.3e cells answered without a launch, %.3e computed\n",
                     (unsigned long long)tot.reused, (double)tot.cells_reused, (double)tot.cells);
    if (st) {
        st->cells += tot.cells;
        st->cells_executed += tot.cells_exec;
        st->cells_reused += tot.cells_reused;
        st->launches += tot.launches;
        lev_finish_timing(tot);
        st->kernel_ms += tot.kernel_ms;
    }
}

uint32_t geometric_median(dm_ctx* ctx, const dm_seqset* s, const uint32_t* members, uint64_t n,
                          uint64_t seed, uint64_t exact_cap) {
    // cluster_tree.cpp:115-166
    if (n == 0) throw invalid_argument("geometric_median of an empty member set");
    for (uint64_t i = 0; i < n; ++i)
        if (members[i] >= s->n) throw invalid_argument("sequence index out of range");
    if (n == 1) return members[0];
    exact_cap = std::max<uint64_t>(2, exact_cap);
    std::vector<uint32_t> cand;
    if (n <= exact_cap) {
        cand.assign(members, members + n);
    } else {
        std::mt19937_64 g(seed);
        for (uint64_t p : sample_distinct(g, n, exact_cap)) cand.push_back(members[p]);
    }
    const uint32_t k = (uint32_t)cand.size();
    std::vector<LevItem> items;
    for (uint32_t i = 0; i < k; ++i)
        for (uint32_t j = i + 1; j < k; ++j) items.push_back(LevItem{cand[i], cand[j], (uint64_t)i * k + j});
    uint32_t* d = ctx->out.as<uint32_t>((size_t)k * k);
    lev_run_host_items(ctx, s, items, d, nullptr, false);
    std::vector<uint32_t> mat((size_t)k * k);
    DM_CUDA(cudaMemcpyAsync(mat.data(), d, mat.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    size_t best = 0;
    uint64_t best_sum = UINT64_MAX;
    for (uint32_t i = 0; i < k; ++i) {
        uint64_t sum = 0;
        for (uint32_t j = 0; j < k; ++j)
            if (i != j) sum += i < j ? mat[(size_t)i * k + j] : mat[(size_t)j * k + i];
        if (sum < best_sum || (sum == best_sum && cand[i] < cand[best])) {
            best_sum = sum;
            best = i;
        }
    }
    return cand[best];
}

}  // namespace dm
