// MSA builder (SURVEY.md §2.2 K7/K8 + the per-level merge scheduler):
// align_all (msa_merge.cpp:107-158) as level-synchronous batches.
//
// The rows of every subtree are contiguous in tree.order (cluster_tree.cpp:
// 212-231), so the alignment lives in ONE device row buffer: row r carries
// sequence order[r] (test_msa_merge.cpp:198) and the block of node v is rows
// [v.begin, v.end) x columns [0, W_v). Internal nodes are merged deepest
// level first; all merges of a level are independent:
//   1. NW of the children's CENTER rows, read in place from the row buffer
//      (msa_merge.cpp:82-84: left.row_of(left_child.center) etc.) — one
//      batched nw_run;
//   2. a column map per (merge, side) from the gap lists: original column c
//      moves to c + #{gap positions <= c}; gap k lands at p_k + k
//      (msa_merge.cpp:31-70);
//   3. every row of both children is rewritten in place through its map
//      (one CTA per row, staged through shared memory). Parent rows are
//      left rows then right rows by construction (:94-104).
// The result is schedule-independent exactly as the reference's task DAG
// (:119-122).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "comm.h"
#include "dm_internal.h"
#include "nvtx.h"
#include "host_copy.h"
#include "nw.h"

namespace dm {
namespace {

// Side descriptor: rows [r0, r1) of the buffer, old width -> new width via map.
struct SideDesc {
    uint32_t r0, r1;
    uint32_t w_old, w_new;
    uint64_t map_off;   // into the column-map buffer (w_new entries)
    uint64_t gap_off;   // gap list, DESCENDING (path order)
    uint32_t ngaps;
    uint32_t pad;
};

__global__ void init_rows_kernel(const uint8_t* __restrict__ raw, const uint64_t* __restrict__ raw_off,
                                 const uint32_t* __restrict__ order, uint32_t n, uint8_t* __restrict__ rows,
                                 uint64_t pitch) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = warp; r < n; r += nw) {
        const uint32_t s = order[r];
        const uint64_t a = raw_off[s], e = raw_off[s + 1];
        uint8_t* dst = rows + (uint64_t)r * pitch;
        for (uint64_t i = a + lane; i < e; i += 32) dst[i - a] = raw[i];
    }
}

// One CTA per side: map[o] = source column, or -1 for an inserted gap column.
__global__ void colmap_kernel(const SideDesc* __restrict__ sides, const uint32_t* __restrict__ gaps,
                              int32_t* __restrict__ maps) {
    const SideDesc d = sides[blockIdx.x];
    int32_t* map = maps + d.map_off;
    const uint32_t* g = gaps + d.gap_off;  // descending: asc[k] = g[ng-1-k]
    const uint32_t ng = d.ngaps;
    for (uint32_t k = threadIdx.x; k < ng; k += blockDim.x) map[g[ng - 1 - k] + k] = -1;
    for (uint32_t c = threadIdx.x; c < d.w_old; c += blockDim.x) {
        // count of gap positions <= c  (upper_bound over the ascending view)
        uint32_t lo = 0, hi = ng;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (g[ng - 1 - mid] <= c) lo = mid + 1;
            else hi = mid;
        }
        map[c + lo] = (int32_t)c;
    }
}

// Rows of all sides of a level; row -> side by binary search on prefix sums.
__global__ void insert_rows_kernel(const SideDesc* __restrict__ sides, const uint32_t* __restrict__ side_rows_prefix,
                                   uint32_t nsides, uint32_t total_rows, const int32_t* __restrict__ maps,
                                   uint8_t* __restrict__ rows, uint64_t pitch) {
    extern __shared__ __align__(16) uint8_t srow[];
    for (uint32_t t = blockIdx.x; t < total_rows; t += gridDim.x) {
        uint32_t lo = 0, hi = nsides;  // largest s with prefix[s] <= t
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (side_rows_prefix[mid] <= t) lo = mid;
            else hi = mid;
        }
        const SideDesc d = sides[lo];
        const uint32_t r = d.r0 + (t - side_rows_prefix[lo]);
        uint8_t* row = rows + (uint64_t)r * pitch;  // 64-byte aligned, pitch >= round64(w_new)
        __syncthreads();
        // the old row into shared memory, 16 bytes per thread (bytes past w_old are never mapped)
        for (uint32_t c = threadIdx.x * 16; c < d.w_old; c += blockDim.x * 16)
            *reinterpret_cast<uint4*>(srow + c) = *reinterpret_cast<const uint4*>(row + c);
        __syncthreads();
        // the new row, 4 bytes per thread per store (bytes past w_new up to the next
        // multiple of 4 are padding no reader looks at)
        const int32_t* map = maps + d.map_off;
        for (uint32_t o = threadIdx.x * 4; o < d.w_new; o += blockDim.x * 4) {
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t src = o + k < d.w_new ? map[o + k] : -1;
                v |= (uint32_t)(src < 0 ? (uint8_t)'-' : srow[src]) << (8 * k);
            }
            *reinterpret_cast<uint32_t*>(row + o) = v;
        }
    }
}

void grow_rows(dm_ctx* ctx, DevBuf& buf, uint64_t& pitch, uint32_t n, uint64_t need) {
    if (need <= pitch) return;
    const uint64_t np = ((need + need / 4) + 63) & ~uint64_t(63);
    DevBuf nb(&ctx->stream);
    uint8_t* dst = (uint8_t*)nb.get((uint64_t)n * np);
    DM_CUDA(cudaMemcpy2DAsync(dst, np, buf.p, pitch, pitch, n, cudaMemcpyDeviceToDevice, ctx->stream));
    std::swap(buf.p, nb.p);
    std::swap(buf.cap, nb.cap);
    pitch = np;
}

// Apply one batch of sides (their gap lists already on the device).
void apply_sides(dm_ctx* ctx, std::vector<SideDesc>& sides, const uint32_t* d_gaps, uint8_t* d_rows, uint64_t pitch,
                 uint64_t max_w_old) {
    if (sides.empty()) return;
    uint64_t mtot = 0;
    std::vector<uint32_t> prefix(sides.size() + 1, 0);
    for (size_t i = 0; i < sides.size(); ++i) {
        sides[i].map_off = mtot;
        mtot += sides[i].w_new;
        prefix[i + 1] = prefix[i] + (sides[i].r1 - sides[i].r0);
    }
    int32_t* d_maps = ctx->colmap.as<int32_t>(std::max<uint64_t>(mtot, 1));
    SideDesc* d_sides = ctx->tree_buf.as<SideDesc>(sides.size());
    uint32_t* d_prefix = ctx->aux3.as<uint32_t>(prefix.size());
    DM_CUDA(cudaMemcpyAsync(d_sides, sides.data(), sides.size() * sizeof(SideDesc), cudaMemcpyHostToDevice,
                            ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_prefix, prefix.data(), prefix.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    colmap_kernel<<<(unsigned)sides.size(), 256, 0, ctx->stream>>>(d_sides, d_gaps, d_maps);
    DM_CUDA(cudaGetLastError());
    {
        uint64_t g = 0, rd = 0, wr = 0;
        for (const SideDesc& d : sides) {
            g += d.ngaps;
            rd += (uint64_t)(d.r1 - d.r0) * d.w_old;
            wr += (uint64_t)(d.r1 - d.r0) * d.w_new;
        }
        trace_bytes("colmap_kernel", g * 4 * 2, mtot * 4);
        trace_bytes("insert_rows_kernel", rd, wr);
    }
    const uint32_t total = prefix.back();
    const size_t smem = std::max<uint64_t>((max_w_old + 15) & ~uint64_t(15), 16);
    if (smem > 48 * 1024)
        DM_CUDA(cudaFuncSetAttribute(insert_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::max<uint32_t>(1, std::min<uint32_t>(total, (uint32_t)ctx->sm_count * 16));
    insert_rows_kernel<<<grid, 128, smem, ctx->stream>>>(d_sides, d_prefix, (uint32_t)sides.size(), total, d_maps,
                                                         d_rows, pitch);
    DM_CUDA(cudaGetLastError());
    ctx->launches += 2;
}

// Row blocks of whole subtrees: block i = rows [r0, r0 + nrows) x width
// bytes, packed contiguously at buf_off (one warp per row).
struct BlockDesc {
    uint32_t r0, nrows, width, pad;
    uint64_t buf_off;
};
__global__ void pack_blocks_kernel(const BlockDesc* __restrict__ d, uint32_t nb, const uint32_t* __restrict__ rprefix,
                                   uint32_t total_rows, uint8_t* __restrict__ rows, uint64_t pitch,
                                   uint8_t* __restrict__ buf, int unpack) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < total_rows; t += nwarps) {
        uint32_t lo = 0, hi = nb;  // block holding packed row t
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (rprefix[mid] <= t) lo = mid;
            else hi = mid;
        }
        const BlockDesc b = d[lo];
        const uint32_t k = t - rprefix[lo];
        uint8_t* row = rows + (uint64_t)(b.r0 + k) * pitch;
        uint8_t* pk = buf + b.buf_off + (uint64_t)k * b.width;
        if (unpack)
            for (uint32_t c = lane; c < b.width; c += 32) row[c] = pk[c];
        else
            for (uint32_t c = lane; c < b.width; c += 32) pk[c] = row[c];
    }
}

void run_blocks(dm_ctx* ctx, const std::vector<BlockDesc>& blocks, uint8_t* rows, uint64_t pitch, uint8_t* buf,
                bool unpack) {
    if (blocks.empty()) return;
    std::vector<uint32_t> prefix(blocks.size() + 1, 0);
    for (size_t i = 0; i < blocks.size(); ++i) prefix[i + 1] = prefix[i] + blocks[i].nrows;
    BlockDesc* d_b = (BlockDesc*)ctx->aux.get(blocks.size() * sizeof(BlockDesc) + prefix.size() * 4 + 16);
    uint32_t* d_p = reinterpret_cast<uint32_t*>(d_b + blocks.size());
    DM_CUDA(cudaMemcpyAsync(d_b, blocks.data(), blocks.size() * sizeof(BlockDesc), cudaMemcpyHostToDevice,
                            ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_p, prefix.data(), prefix.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    const int grid = (int)std::max<uint32_t>(1, std::min<uint32_t>((prefix.back() + 7) / 8, ctx->sm_count * 16u));
    pack_blocks_kernel<<<grid, 256, 0, ctx->stream>>>(d_b, (uint32_t)blocks.size(), d_p, prefix.back(), rows, pitch,
                                                      buf, unpack ? 1 : 0);
    DM_CUDA(cudaGetLastError());
    DM_CUDA(cudaStreamSynchronize(ctx->stream));  // descriptors reused by the next call
    ++ctx->launches;
}

// After each rank merged its own cut subtrees: every rank gets every cut
// subtree's width (host all-gather) and row block (device all-gather of the
// packed blocks, padded to the largest rank's bytes).
void exchange_blocks(dm_ctx* ctx, const std::vector<dm_node>& nodes, const std::vector<uint32_t>& cut,
                     const std::vector<int>& region, std::vector<uint64_t>& W, DevBuf& rowsbuf, uint64_t& pitch,
                     uint32_t n) {
    const int w = ctx->world;
    std::vector<uint64_t> mine(cut.size(), 0), all(cut.size() * (size_t)w);
    for (size_t i = 0; i < cut.size(); ++i)
        if (region[cut[i]] == ctx->rank) mine[i] = W[cut[i]];
    comm_allgather_host(ctx, mine.data(), all.data(), mine.size() * sizeof(uint64_t));
    uint64_t wmax = 0;
    std::vector<uint64_t> bytes((size_t)w, 0);
    for (size_t i = 0; i < cut.size(); ++i) {
        const int r = region[cut[i]];
        W[cut[i]] = all[(size_t)r * cut.size() + i];
        wmax = std::max(wmax, W[cut[i]]);
        bytes[r] += (uint64_t)(nodes[cut[i]].end - nodes[cut[i]].begin) * W[cut[i]];
    }
    grow_rows(ctx, rowsbuf, pitch, n, wmax);
    uint64_t mx = 16;
    for (uint64_t b : bytes) mx = std::max(mx, b);
    uint8_t* buf = (uint8_t*)ctx->comm_dev.get(mx * (uint64_t)(w + 1) + 64);
    std::vector<std::vector<BlockDesc>> per((size_t)w);
    std::vector<uint64_t> at((size_t)w, 0);
    for (size_t i = 0; i < cut.size(); ++i) {
        const int r = region[cut[i]];
        const dm_node& nd = nodes[cut[i]];
        per[r].push_back(BlockDesc{nd.begin, nd.end - nd.begin, (uint32_t)W[cut[i]], 0, (uint64_t)r * mx + at[r]});
        at[r] += (uint64_t)(nd.end - nd.begin) * W[cut[i]];
    }
    run_blocks(ctx, per[ctx->rank], (uint8_t*)rowsbuf.p, pitch, buf, false);
    comm_allgather(ctx, buf + (uint64_t)ctx->rank * mx, buf, mx);
    std::vector<BlockDesc> others;
    for (int r = 0; r < w; ++r)
        if (r != ctx->rank) others.insert(others.end(), per[r].begin(), per[r].end());
    run_blocks(ctx, others, (uint8_t*)rowsbuf.p, pitch, buf, true);
}

}  // namespace

dm_msa_out* align_all(dm_ctx* ctx, const dm_seqset* s, const std::vector<dm_node>& nodes,
                      const std::vector<uint32_t>& order, const NwScheme& sc, dm_stats* st,
                      dm_progress_fn progress, void* progress_user, bool host_rows) {
    NvtxRange nvtx_align("dm align_all");
    const uint32_t n = s->n;
    if (order.size() != n) throw invalid_argument("tree order does not match the sequence set");
    if (nodes.empty()) throw invalid_argument("empty tree");
    for (int c = 0; c < 256; ++c)
        if (s->present[c] && (c >= 128 || !sc.has[c]))
            throw invalid_argument(std::string("sequence a contains symbol '") + (char)c +
                                   "' absent from the substitution table");
    auto* out = new dm_msa_out;
    try {
        cudaStream_t stream = ctx->stream;
        std::vector<uint32_t> pos(n);
        for (uint32_t r = 0; r < n; ++r) pos[order[r]] = r;
        // widths: leaves carry their sequence
        std::vector<uint64_t> W(nodes.size(), 0);
        uint32_t maxdepth = 0, maxlen = 1;
        for (uint32_t i = 0; i < n; ++i) maxlen = std::max(maxlen, s->len[i]);
        std::vector<std::vector<uint32_t>> by_depth;
        for (size_t v = 0; v < nodes.size(); ++v) {
            const dm_node& nd = nodes[v];
            if (nd.left < 0) {
                if (nd.end - nd.begin != 1) throw invalid_argument("align_leaf requires a singleton leaf node");
                W[v] = s->len[nd.center];
                continue;
            }
            if (by_depth.size() <= nd.depth) by_depth.resize(nd.depth + 1);
            by_depth[nd.depth].push_back((uint32_t)v);
            maxdepth = std::max(maxdepth, nd.depth);
        }
        // The NW trace of the largest level, estimated from the tree and mapped
        // once up front: growing the buffer level by level made the pool map
        // fresh memory several times on a context's first call (~60 GB for
        // cfg4). Widths are estimated as the subtree's longest sequence times
        // 1 + 2 % per merge above it (cfg4: 2,620 measured vs ~2,800
        // estimated at the root); an underestimate only means later growth.
        {
            std::vector<uint32_t> sub_len(nodes.size(), 0), height(nodes.size(), 0);
            for (size_t v = nodes.size(); v-- > 0;) {  // BFS numbering: children after parents
                const dm_node& nd = nodes[v];
                if (nd.left < 0) {
                    sub_len[v] = s->len[nd.center];
                    continue;
                }
                sub_len[v] = std::max(sub_len[nd.left], sub_len[nd.right]);
                height[v] = 1 + std::max(height[nd.left], height[nd.right]);
            }
            auto west = [&](size_t v) { return (double)sub_len[v] * (1.0 + 0.02 * height[v]) + 1.0; };
            std::vector<double> lvl((size_t)maxdepth + 1, 0.0);
            for (size_t v = 0; v < nodes.size(); ++v)
                if (nodes[v].left >= 0)
                    lvl[nodes[v].depth] += (west(nodes[v].left) + 32.0) * (west(nodes[v].right) + 32.0);
            double mx = 0;
            for (double x : lvl) mx = std::max(mx, x);
            const uint64_t cap = std::max<uint64_t>(6ull << 30, ctx->free_at_create / 100 * 45);
            const uint64_t want = std::min<uint64_t>((uint64_t)(mx * 1.05), cap);
            if (want > (64ull << 20)) ctx->nw_trace.reserve_exact(want);
        }
        uint64_t pitch = ((uint64_t)maxlen + maxlen / 2 + 64 + 63) & ~uint64_t(63);
        DevBuf& rowsbuf = ctx->rows_a;
        rowsbuf.get((uint64_t)n * pitch);
        uint32_t* d_order = ctx->rows_b.as<uint32_t>(n);
        DM_CUDA(cudaMemcpyAsync(d_order, order.data(), (size_t)n * 4, cudaMemcpyHostToDevice, stream));
        {
            const int grid = (int)std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16);
            init_rows_kernel<<<std::max(grid, 1), 256, 0, stream>>>(s->d_raw, s->d_raw_off, d_order, n,
                                                                   (uint8_t*)rowsbuf.p, pitch);
            DM_CUDA(cudaGetLastError());
            ctx->launches += 1;
        }
        // columns of a merge are a center row: the set's residues and '-'
        NwScheme scc = sc;
        {
            bool present[128] = {};
            for (int c = 0; c < 128; ++c) present[c] = s->present[c];
            present[(unsigned char)'-'] = true;
            set_columns(scc, present);
        }
        const bool trace = std::getenv("DM_TRACE") != nullptr;
        uint64_t done = 0;
        const uint64_t total = nodes.size();
        if (progress)
            for (const dm_node& nd : nodes)
                if (nd.left < 0) progress(++done, total, progress_user);
        float fwd_ms = 0, tb_ms = 0;
        uint64_t cells = 0, nw_calls = 0, launches = 0;
        // One tree level's merges (lvl): NW of the children's center rows,
        // then every child row rewritten through its column map. local: the
        // batch is this rank's own (subtree ownership), never sharded.
        auto run_level = [&](const std::vector<uint32_t>& lvl, int d, bool local) {
            if (lvl.empty()) return;
            NvtxRange nvtx_level("dm merge level");
            std::vector<NwJob> jobs(lvl.size());
            for (size_t k = 0; k < lvl.size(); ++k) {
                const dm_node& nd = nodes[lvl[k]];
                const dm_node& lc = nodes[nd.left];
                const dm_node& rc = nodes[nd.right];
                NwJob& jb = jobs[k];
                jb.a_off = (uint64_t)pos[lc.center] * pitch;
                jb.n = (uint32_t)W[nd.left];
                jb.b_off = (uint64_t)pos[rc.center] * pitch;
                jb.m = (uint32_t)W[nd.right];
            }
            NwOut no;
            const auto h0 = std::chrono::steady_clock::now();
            nw_run_sharded(ctx, (const uint8_t*)rowsbuf.p, jobs, scc, no, st != nullptr || trace, local);
            fwd_ms += no.fwd_ms;
            tb_ms += no.tb_ms;
            cells += no.cells;
            nw_calls += jobs.size();
            launches += no.launches;
            std::vector<NwRes> res(jobs.size());
            DM_CUDA(cudaMemcpyAsync(res.data(), no.d_res, res.size() * sizeof(NwRes), cudaMemcpyDeviceToHost, stream));
            DM_CUDA(cudaStreamSynchronize(stream));
            uint64_t wmax = 0, wold = 0;
            std::vector<SideDesc> sides;
            sides.reserve(2 * jobs.size());
            for (size_t k = 0; k < lvl.size(); ++k) {
                const dm_node& nd = nodes[lvl[k]];
                const dm_node& lc = nodes[nd.left];
                const dm_node& rc = nodes[nd.right];
                const uint64_t w = res[k].len;
                if (w != W[nd.left] + res[k].nga || w != W[nd.right] + res[k].ngb)
                    throw runtime_error("internal error: aligned width does not match the gap lists");
                W[lvl[k]] = w;
                wmax = std::max(wmax, w);
                wold = std::max<uint64_t>(wold, std::max(W[nd.left], W[nd.right]));
                if (res[k].nga)
                    sides.push_back(SideDesc{lc.begin, lc.end, (uint32_t)W[nd.left], (uint32_t)w, 0,
                                             jobs[k].ga_off, res[k].nga, 0});
                if (res[k].ngb)
                    sides.push_back(SideDesc{rc.begin, rc.end, (uint32_t)W[nd.right], (uint32_t)w, 0,
                                             jobs[k].gb_off, res[k].ngb, 0});
            }
            if (progress)
                for (size_t k = 0; k < lvl.size(); ++k) progress(++done, total, progress_user);
            if (trace) DM_CUDA(cudaEventRecord(ctx->ev0, stream));
            grow_rows(ctx, rowsbuf, pitch, n, wmax);
            apply_sides(ctx, sides, no.d_gaps, (uint8_t*)rowsbuf.p, pitch, wold);
            launches += 2;
            if (trace) {
                DM_CUDA(cudaEventRecord(ctx->ev1, stream));
                DM_CUDA(cudaStreamSynchronize(stream));
                float ins = 0;
                cudaEventElapsedTime(&ins, ctx->ev0, ctx->ev1);
                const double ms =
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
                std::fprintf(stderr,
                             "[dm align] depth %d merges %zu cells %.3e fwd %.3f ms tb %.3f ms insert %.3f ms level %.3f ms%s\n",
                             d, jobs.size(), (double)no.cells, no.fwd_ms, no.tb_ms, ins, ms, local ? " (own)" : "");
            }
        };
        // Subtree ownership (several attached ranks): subtrees of at most
        // n / (DM_OWN_SPLIT x world) rows are cut off and assigned to ranks by
        // their merge work (sum of the children's center lengths' products);
        // each rank merges its own (no collective), the finished row blocks
        // and widths are all-gathered once, and the levels above the cut run
        // on every rank with their NW batches sharded.
        std::vector<int> region(nodes.size(), -1);  // owner rank of the node's cut subtree; -1 above the cut
        std::vector<uint32_t> cut;
        if (comm_real(ctx) && n >= 4u * (uint32_t)ctx->world) {
            const uint64_t split = [] {
                const char* e = std::getenv("DM_OWN_SPLIT");
                return e ? (uint64_t)std::max(1, std::atoi(e)) : (uint64_t)8;
            }();
            const uint64_t lim = std::max<uint64_t>(2, n / (split * (uint64_t)ctx->world));
            // nodes are numbered parent before child (BFS): one pass finds the cut
            std::vector<uint8_t> below(nodes.size(), 0);
            for (size_t v = 0; v < nodes.size(); ++v) {
                const dm_node& nd = nodes[v];
                const bool above_parent = nd.parent < 0 || !below[nd.parent];
                if (above_parent && nd.end - nd.begin <= lim) {
                    cut.push_back((uint32_t)v);
                    below[v] = 1;
                } else if (!above_parent) {
                    below[v] = 1;
                }
            }
            if (cut.size() >= (size_t)ctx->world) {
                // merge work per node, children before parents (reverse BFS order)
                std::vector<uint64_t> work(nodes.size(), 0);
                for (size_t v = nodes.size(); v-- > 0;) {
                    const dm_node& nd = nodes[v];
                    if (nd.left < 0) continue;
                    work[v] = work[nd.left] + work[nd.right] +
                              (uint64_t)s->len[nodes[nd.left].center] * s->len[nodes[nd.right].center] + 1;
                }
                std::vector<uint64_t> cost(cut.size());
                for (size_t i = 0; i < cut.size(); ++i) cost[i] = work[cut[i]] + 1;
                std::vector<int> own;
                assign_lpt(cost.data(), cost.size(), ctx->world, own);
                for (size_t i = 0; i < cut.size(); ++i) {
                    region[cut[i]] = own[i];
                    ctx->own_msa += own[i] == ctx->rank;
                }
                for (size_t v = 0; v < nodes.size(); ++v)  // descendants inherit (parents come first)
                    if (region[v] < 0 && nodes[v].parent >= 0 && below[v] && region[nodes[v].parent] >= 0)
                        region[v] = region[nodes[v].parent];
            } else {
                cut.clear();
            }
        }
        if (cut.empty()) {
            for (int d = (int)by_depth.size() - 1; d >= 0; --d) run_level(by_depth[d], d, false);
        } else {
            // phase A: this rank's subtrees, deepest level first
            for (int d = (int)by_depth.size() - 1; d >= 0; --d) {
                std::vector<uint32_t> mine;
                for (uint32_t v : by_depth[d])
                    if (region[v] == ctx->rank) mine.push_back(v);
                run_level(mine, d, true);
            }
            // phase B: widths and row blocks of every cut subtree from its owner
            exchange_blocks(ctx, nodes, cut, region, W, rowsbuf, pitch, n);
            if (progress)
                for (size_t v = 0; v < nodes.size(); ++v)
                    if (nodes[v].left >= 0 && region[v] >= 0 && region[v] != ctx->rank)
                        progress(++done, total, progress_user);
            // phase C: the levels above the cut, on every rank
            for (int d = (int)by_depth.size() - 1; d >= 0; --d) {
                std::vector<uint32_t> up;
                for (uint32_t v : by_depth[d])
                    if (region[v] < 0) up.push_back(v);
                run_level(up, d, false);
            }
        }
        const uint64_t width = W[0];
        out->width = width;
        out->dev_pitch = pitch;
        if (host_rows) {  // (callers that read the device rows skip this copy)
            out->rows.resize((uint64_t)n * width);
            if (width) download_rows(ctx, out->rows.data(), rowsbuf.p, width, pitch, n, stream);
        }
        DM_CUDA(cudaStreamSynchronize(stream));
        out->row_seq = order;
        out->nodes = nodes;
        out->order = order;
        if (st) {
            st->cells += cells;
            st->nw_calls += nw_calls;
            st->launches += launches + 1;
            st->kernel_ms += fwd_ms + tb_ms;
        }
    } catch (...) {
        delete out;
        throw;
    }
    return out;
}

namespace {
// out[k] = src row sel[k] (warp per row, 16-byte loads from the pitched source)
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, uint64_t pitch, const uint32_t* __restrict__ sel,
                                   uint64_t n, uint64_t width, uint8_t* __restrict__ out) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp; k < n; k += nwarps) {
        const uint8_t* r = src + (uint64_t)sel[k] * pitch;  // pitch is a multiple of 64
        uint8_t* o = out + k * width;
        for (uint64_t c = (uint64_t)lane * 16; c < width; c += 32 * 16) {
            const uint4 v = *reinterpret_cast<const uint4*>(r + c);
            const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
            const uint64_t m = width - c < 16 ? width - c : 16;
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if ((uint64_t)t < m) o[c + t] = b[t];
        }
    }
}
}  // namespace

void gather_rows_to_host(dm_ctx* ctx, const uint8_t* src, uint64_t pitch, const uint32_t* sel, uint64_t n,
                         uint64_t width, char* out) {
    if (n == 0 || width == 0) return;
    uint32_t* d_sel = ctx->aux2.as<uint32_t>(n);
    DM_CUDA(cudaMemcpyAsync(d_sel, sel, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    uint8_t* d_out = (uint8_t*)ctx->rows_b.get(n * width);
    const uint64_t blocks = std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16);
    gather_rows_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(src, pitch, d_sel, n, width, d_out);
    DM_CUDA(cudaGetLastError());
    ctx->launches += 1;
    trace_bytes("gather_rows_kernel", n * width, n * width);
    download_host(ctx, out, d_out, n * width, ctx->stream);
}

void insert_gap_columns(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, const uint32_t* pos,
                        uint64_t npos, char* out) {
    // msa_merge.cpp:31-70 (validation messages :37-44)
    for (uint64_t i = 0; i < npos; ++i) {
        if (pos[i] > width)
            throw invalid_argument("gap position " + std::to_string(pos[i]) + " exceeds alignment width " +
                                   std::to_string(width));
        if (i > 0 && pos[i] < pos[i - 1]) throw invalid_argument("gap positions must be sorted ascending");
    }
    const uint64_t nw = width + npos;
    if (nrows == 0) return;
    if (npos == 0) {
        std::memcpy(out, rows, nrows * width);
        return;
    }
    const uint64_t pitch = (nw + 63) & ~uint64_t(63);
    uint8_t* d_rows = (uint8_t*)ctx->rows_a.get(nrows * pitch);
    DM_CUDA(cudaMemcpy2DAsync(d_rows, pitch, rows, width, width, nrows, cudaMemcpyHostToDevice, ctx->stream));
    std::vector<uint32_t> desc(npos);
    for (uint64_t i = 0; i < npos; ++i) desc[i] = pos[npos - 1 - i];
    uint32_t* d_g = ctx->rows_b.as<uint32_t>(npos);
    DM_CUDA(cudaMemcpyAsync(d_g, desc.data(), npos * 4, cudaMemcpyHostToDevice, ctx->stream));
    std::vector<SideDesc> sides{SideDesc{0, (uint32_t)nrows, (uint32_t)width, (uint32_t)nw, 0, 0, (uint32_t)npos, 0}};
    apply_sides(ctx, sides, d_g, d_rows, pitch, width);
    DM_CUDA(cudaMemcpy2DAsync(out, nw, d_rows, pitch, nw, nrows, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace dm
