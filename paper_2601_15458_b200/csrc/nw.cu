// Pairwise aligner: batched Gotoh Needleman-Wunsch
// with device-side traceback, bit-exact with nw_align (pairwise.cpp:301-415).
//
// Forward (K5, nw_fwd.cuh): one alignment per CTA of 1-4 or 8 warps. Lane g
// owns RR = 16 consecutive rows of its warp's 512-row band and sweeps the
// columns of b as a diagonal pipeline (lane g is on column s-g+1 at step s);
// the bottom row of lane g-1 arrives by __shfl_up each step, and each band
// streams its bottom row to the band below through a shared-memory ring, so
// all bands of an alignment run concurrently. Scores are kept in "tagged" form
//     V = 4 * score + tag,  tag(M) = 2, tag(GapB) = 1, tag(GapA) = 0,
// so ONE max over three tagged candidates returns both the best score and,
// on ties, the state pick_best prefers (M > GapB > GapA, pairwise.cpp:272-
// 286): the tag of the winner is the traceback code, with no compare/select.
// Penalties are pre-multiplied by 4 so tags survive the additions.
// Trace: one byte per cell, (tagM | tagGB<<2 | tagGA<<4), column-major
// [j-1][i-1] with the column padded to 16 bytes so every lane writes its 16
// rows with one 16-byte store. Row 0 / column 0 codes are analytic
// (pairwise.cpp:322-339) and never stored.
//
// Arithmetic: int32 while (n+m+2)*(max|s|+|open|+|extend|) stays far from
// 2^28 (always the case for the built-in schemes at realistic widths),
// otherwise the same kernel instantiated on int64 — never a CPU fallback.
// -inf is -2^30 (int32) / -2^60 (int64) in tagged units; every -inf-derived
// value stays below every finite one, so all decisions on finite states
// (the only ones a traceback visits) match the reference's int64 run.
//
// Traceback (K6): one warp per alignment; the warp stages a 32-column x
// 64-row trace tile into shared memory and lane 0 walks the path inside it
// (pairwise.cpp:384-409), emitting gaps_into_b (j at GapB) and gaps_into_a
// (i at GapA) in path (descending) order.
#include <algorithm>
#include <cstring>

#include "dm_internal.h"
#include "nvtx.h"
#include "nw.h"
#include "nw_fwd.cuh"
#include "nw_seq.cuh"
#include "nw_clu.cuh"
#include "comm.h"

namespace dm {
namespace {

using nwk::FULL;

struct TbArgs {
    const NwJob* jobs;
    uint32_t njobs;
    const uint8_t* trace;
    NwRes* res;
    uint32_t* gaps;
    uint32_t* counter;
    int diag;  // trace in the throughput kernel's step-major layout (nw_seq.cuh)
};

// 16 trace bytes: rows R .. R+15 (R 16-aligned, 0-based) of column j (1-based).
// Column-major (ring kernel): column j-1 of pa bytes. Step-major (throughput
// kernel, nw_seq.cuh): band b = R / 512 holds (m + 31) steps x 32 lanes x RR
// bytes, lane g owning rows [g RR, g RR + RR) of the band and writing column j
// at step j + g - 1; the last band has RR = 16, 8 or 4.
__device__ __forceinline__ uint4 trace_chunk16(const uint8_t* T, uint32_t n, uint32_t m, uint32_t pa, int diag,
                                               uint32_t R, uint32_t j) {
    if (!diag) return *reinterpret_cast<const uint4*>(T + (uint64_t)(j - 1) * pa + R);
    const uint32_t b = R / nwk::BAND, nb = (n + nwk::BAND - 1) / nwk::BAND;
    const uint32_t rr = b + 1 < nb ? 16u : nwk::seq_tail_rr(n - b * nwk::BAND);
    const uint8_t* base = T + (uint64_t)b * (m + 31) * nwk::BAND;
    const uint32_t l = R - b * nwk::BAND;
    if (rr == 16) {
        const uint32_t g = l / 16;
        return *reinterpret_cast<const uint4*>(base + (uint64_t)(j + g - 1) * 512 + g * 16);
    }
    // 12 / 8 / 4 rows per lane: each 4-row word lies inside one lane's rows
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t row = l + 4 * q, g = row / rr, r = row - g * rr;
        w[q] = *reinterpret_cast<const uint32_t*>(base + (uint64_t)(j + g - 1) * 32 * rr + g * rr + r);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

constexpr int TC = 32;  // tile columns (one per lane)
constexpr int TR = 64;  // tile rows (bytes per column)

// trace_chunk16 into shared memory with cp.async (the prefetched tile)
__device__ __forceinline__ void cp_async_n(void* smem, const void* gmem, int bytes) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    if (bytes == 16) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void trace_chunk16_async(uint8_t* dst, const uint8_t* T, uint32_t n, uint32_t m, uint32_t pa,
                                                    int diag, uint32_t R, uint32_t j) {
    if (!diag) {
        cp_async_n(dst, T + (uint64_t)(j - 1) * pa + R, 16);
        return;
    }
    const uint32_t b = R / nwk::BAND, nb = (n + nwk::BAND - 1) / nwk::BAND;
    const uint32_t rr = b + 1 < nb ? 16u : nwk::seq_tail_rr(n - b * nwk::BAND);
    const uint8_t* base = T + (uint64_t)b * (m + 31) * nwk::BAND;
    const uint32_t l = R - b * nwk::BAND;
    if (rr == 16) {
        const uint32_t g = l / 16;
        cp_async_n(dst, base + (uint64_t)(j + g - 1) * 512 + g * 16, 16);
        return;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t row = l + 4 * q, g = row / rr, r = row - g * rr;
        cp_async_n(dst + 4 * q, base + (uint64_t)(j + g - 1) * 32 * rr + g * rr + r, 4);
    }
}

// Warp per alignment. The path is walked by lane 0 inside a 32-column x
// 64-row tile of trace bytes staged in shared memory (lane g loads column
// jtop - g); while it walks, the tile the path most likely enters next (32
// columns to the left, rows following the diagonal) is prefetched with
// cp.async into the other buffer and used if the walk really ended there
// (else the tile is staged again at the walk's position, as for the first).
// The walk itself is branch-free: the state selects its 2-bit field of the
// trace byte by a shift, the gap lists are written under predicates.
__global__ void __launch_bounds__(128) nw_traceback_kernel(const TbArgs a) {
    __shared__ __align__(16) uint8_t tile[4][2][TC][TR];
    const int g = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    for (;;) {
        uint32_t jid = 0;
        if (g == 0) jid = atomicAdd(a.counter, 1u);
        jid = __shfl_sync(FULL, jid, 0);
        if (jid >= a.njobs) break;
        const NwJob job = a.jobs[jid];
        const uint32_t n = job.n;
        const uint32_t pa = (n + 15) & ~15u;
        const uint8_t* T = a.trace + job.t_off;
        uint32_t* ga = a.gaps + job.ga_off;
        uint32_t* gb = a.gaps + job.gb_off;
        NwRes& res = a.res[job.slot];
        uint32_t state = 2u - res.final_tag;  // 0 M, 1 GapB, 2 GapA
        uint32_t i = n, j = job.m, len = 0, nga = 0, ngb = 0;
        int buf = 0;
        bool have = false;   // tile[w][buf] already holds the tile (jtop = j, rows from r0)
        int r0 = 0;
        while (i > 0 && j > 0) {
            const uint32_t jtop = j;
            if (!have) {
                r0 = max(0, (int)((i - 1) & ~15u) - (TR - 16));
                const int jc = (int)jtop - g;
                if (jc >= 1) {
                    uint4* dst = reinterpret_cast<uint4*>(&tile[w][buf][g][0]);
#pragma unroll
                    for (int q = 0; q < TR / 16; ++q)
                        if ((uint32_t)(r0 + q * 16) < pa)
                            dst[q] = trace_chunk16(T, n, job.m, pa, a.diag, (uint32_t)(r0 + q * 16), (uint32_t)jc);
                }
            }
            // the likely next tile: columns jtop-32 .. jtop-63, rows for a path near the diagonal
            const bool pf = jtop > (uint32_t)TC && i > 24;
            const uint32_t jtop_n = jtop - TC;
            const int r0n = pf ? max(0, (int)((i - 25) & ~15u) - (TR - 16)) : 0;
            if (pf) {
                const int jc = (int)jtop_n - g;
                if (jc >= 1) {
#pragma unroll
                    for (int q = 0; q < TR / 16; ++q)
                        if ((uint32_t)(r0n + q * 16) < pa)
                            trace_chunk16_async(&tile[w][buf ^ 1][g][q * 16], T, n, job.m, pa, a.diag,
                                                (uint32_t)(r0n + q * 16), (uint32_t)jc);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            __syncwarp();
            if (g == 0) {
                // pairwise.cpp:384-409 inside the staged tile, in tile coordinates:
                // column c = jtop - j (j > 0 <=> c < jtop), row r = (i - 1) - r0
                // (r >= 0 implies i > 0). One dependent chain per step: trace byte ->
                // the state's 2-bit field -> next state -> r / c; the gap lists
                // (GapB records j, GapA records i) are written under predicates.
                const uint8_t* tb = &tile[w][buf][0][0];
                int c = 0, r = (int)(i - 1) - r0;
                const int cmax = (int)min((uint32_t)TC, jtop);
                uint32_t st = state;
                while (r >= 0 && c < cmax) {
                    const uint32_t code = tb[c * TR + r];
                    const uint32_t nxt = 2u - ((code >> (st + st)) & 3u);
                    asm volatile(
                        "{ .reg .pred p, q;\n"
                        "  setp.eq.u32 p, %4, 1;\n"
                        "  setp.eq.u32 q, %4, 2;\n"
                        "  @p st.global.u32 [%0], %1;\n"
                        "  @q st.global.u32 [%2], %3; }" ::"l"(gb + ngb),
                        "r"(jtop - (uint32_t)c), "l"(ga + nga), "r"((uint32_t)(r + r0 + 1)), "r"(st)
                        : "memory");
                    ngb += st == 1u;
                    nga += st == 2u;
                    r -= st != 2u;
                    c += st != 1u;
                    st = nxt;
                    ++len;
                }
                i = (uint32_t)(r + r0 + 1);
                j = jtop - (uint32_t)c;
                state = st;
            }
            i = __shfl_sync(FULL, i, 0);
            j = __shfl_sync(FULL, j, 0);
            state = __shfl_sync(FULL, state, 0);
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
            have = pf && j == jtop_n && i > 0 && (int)(i - 1) >= r0n && (int)(i - 1) < r0n + TR;
            if (have) {
                buf ^= 1;
                r0 = r0n;
            }
        }
        if (g == 0) {
            // row 0 is all GapA, column 0 all GapB (pairwise.cpp:322-339)
            while (j > 0) {
                ga[nga++] = 0;
                --j;
                ++len;
            }
            while (i > 0) {
                gb[ngb++] = 0;
                --i;
                ++len;
            }
            res.len = len;
            res.nga = nga;
            res.ngb = ngb;
        }
    }
}

// wrap_m: largest width of an alignment with more bands than NWW (0: none);
// such launches get a per-CTA global row for the round-to-round hand-off.
template <class V, int NWW>
void launch_fwd(dm_ctx* ctx, const nwk::FwdArgs& fa, size_t smem, uint32_t wrap_m, cudaStream_t st) {
    const int occ = occupancy((const void*)nwk::nw_fwd_kernel<V, NWW>, NWW * 32, smem);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(fa.njobs, (uint64_t)occ * ctx->sm_count));
    nwk::FwdArgs f = fa;
    if (NWW > 1 && wrap_m) {
        f.wrap_stride = ((uint64_t)wrap_m + 1) * 3;
        f.wrap = ctx->nw_wrap.get((uint64_t)grid * f.wrap_stride * sizeof(V));
    }
    nwk::nw_fwd_kernel<V, NWW><<<grid, NWW * 32, smem, st>>>(f);
}

template <class V>
void launch_group(dm_ctx* ctx, int nww, const nwk::FwdArgs& fa, size_t smem, uint32_t wrap_m, cudaStream_t st) {
    if (nww == 1) launch_fwd<V, 1>(ctx, fa, smem, 0, st);
    else if (nww == 2) launch_fwd<V, 2>(ctx, fa, smem, wrap_m, st);
    else if (nww == 3) launch_fwd<V, 3>(ctx, fa, smem, wrap_m, st);
    else if (nww == 4) launch_fwd<V, 4>(ctx, fa, smem, wrap_m, st);
    else if (nww == 5) launch_fwd<V, 5>(ctx, fa, smem, wrap_m, st);
    else if (nww == 6) launch_fwd<V, 6>(ctx, fa, smem, wrap_m, st);
    else if (nww == 7) launch_fwd<V, 7>(ctx, fa, smem, wrap_m, st);
    else launch_fwd<V, 8>(ctx, fa, smem, wrap_m, st);
}

// warps per alignment: one band per warp up to 8 bands (a CTA's warps wait
// for each other between alignments, so no idle warps there), then 8 with
// rounds (5-7 bands on 8 warps left 1-3 warps idle: 2,500-row merges ran at
// half the throughput kernel's rate)
constexpr int kGroups = 8;
int group_of(uint32_t n) {
    const uint32_t nb = (n + nwk::BAND - 1) / nwk::BAND;
    return (int)std::min<uint32_t>(std::max<uint32_t>(nb, 1), 8);
}

// Throughput form (nw_seq.cuh): one warp per alignment, bands in sequence.
// Used when a batch holds at least ~4 alignments per SM: every warp then has
// its own work and the multi-warp form's ring hand-off (there to cut one
// alignment's latency) only costs.
bool use_seq(const dm_ctx* ctx, size_t cnt) {
    const char* e = std::getenv("DM_NW_SEQ");  // tests / tuning: 1 always, 0 never
    const int force = e ? std::atoi(e) : -1;
    if (force >= 0) return force > 0;
    // measured on 2,300^2 alignments (tools/nw_many.py): equal at 600, 1.37 vs
    // 1.00 TCUPS at 1,000 (the ring kernel's per-alignment latency is shorter,
    // its throughput lower)
    return cnt >= (size_t)ctx->sm_count * 4;
}

// Latency form across a cluster (nw_clu.cuh) for batches too small to fill
// the GPU one alignment per CTA (the top merge levels): cluster size so that
// cnt x CL <= SM count. 0 = not used. DM_NW_CLU=0 disables, =k forces k.
constexpr uint32_t kCluMaxM = 4000;  // b and CL_NWW full-width rows in shared memory (52 B per column)
int clu_size(const dm_ctx* ctx, size_t cnt, bool wide, uint32_t mmax, const NwScheme& sc) {
    const char* e = std::getenv("DM_NW_CLU");
    const int force = e ? std::atoi(e) : -1;
    if (force == 0 || wide || cnt == 0 || mmax > kCluMaxM) return 0;
    if (nwk::clu_smem_bytes(sc.K, sc.Kp, mmax) > 220 * 1024) return 0;
    if (force == 2 || force == 4 || force == 8) return force;
    // clusters of 8 need 8 free SMs of one GPC: beyond ~8 of them at once they
    // queue (measured: 16 x 2,600^2 take 1.48 ms at 8, 0.95 ms at 4)
    // (2,400^2 alignments, tools/nw_many.py: 32 of them 0.86 ms at 4 vs 1.26 ms
    // on the ring kernel; 64 at 2: 1.31 vs 1.26 -- the ring kernel from there)
    if (cnt <= 8) return 8;
    if (cnt * 4 <= (size_t)ctx->sm_count - 20) return 4;
    return 0;
}

template <int CL>
void launch_clu(dm_ctx* ctx, const nwk::FwdArgs& fa, const NwScheme& sc, uint32_t mmax) {  // mmax <= kCluMaxM
    constexpr int RRT = 4;
    auto kern = nwk::nw_clu_kernel<RRT, CL>;
    const size_t smem = nwk::clu_smem_bytes(sc.K, sc.Kp, mmax);
    if (smem > 48 * 1024)
        DM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(fa.njobs * CL);
    cfg.blockDim = dim3(nwk::CL_NWW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DM_CUDA(cudaLaunchKernelEx(&cfg, kern, fa));
}

struct SeqDev {
    const int32_t* table = nullptr;
    const int32_t* ptab = nullptr;
    const uint8_t* plut = nullptr;
};

template <class V, bool PROF>
void launch_seq(dm_ctx* ctx, const nwk::SeqArgs& base, uint32_t mmax) {
    const size_t smem = PROF ? (size_t)nwk::SEQ_WARPS * base.KE * 2048 : (size_t)base.K * base.Kp * 4;
    const int occ = occupancy((const void*)nwk::nw_seq_kernel<V, PROF>, nwk::SEQ_WARPS * 32, smem);
    const uint64_t want = (base.njobs + nwk::SEQ_WARPS - 1) / nwk::SEQ_WARPS;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)occ * ctx->sm_count));
    nwk::SeqArgs a = base;
    a.hstride = ((uint64_t)mmax + 2) * nwk::Cell4<V>::words;
    a.hrow = (int4*)ctx->nw_wrap.get((uint64_t)grid * nwk::SEQ_WARPS * a.hstride * sizeof(int4));
    nwk::nw_seq_kernel<V, PROF><<<grid, nwk::SEQ_WARPS * 32, smem, ctx->stream>>>(a);
}

// rows the throughput kernel computes for n rows: whole 512-row bands, the
// last one at 16 / 8 / 4 rows per lane
uint64_t seq_rows(uint32_t n) {
    const uint32_t nb = (n + nwk::BAND - 1) / nwk::BAND;
    return (uint64_t)(nb - 1) * nwk::BAND + 32ull * nwk::seq_tail_rr(n - (nb - 1) * nwk::BAND);
}
// trace bytes of one alignment: column-major (ring kernel) or step-major
uint64_t trace_bytes(const NwJob& jb, bool seq) {
    return seq ? seq_rows(jb.n) * (jb.m + 31ull) : (uint64_t)jb.m * ((jb.n + 15) & ~15u);
}

}  // namespace

void nw_warm() {
    cudaFuncAttributes fa;
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 1>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 2>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 3>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 4>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 5>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 6>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 7>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int32_t, 8>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int64_t, 1>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int64_t, 2>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int64_t, 3>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int64_t, 4>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_fwd_kernel<int64_t, 8>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nw_traceback_kernel));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_clu_kernel<4, 2>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_clu_kernel<4, 4>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_clu_kernel<4, 8>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_seq_kernel<int32_t, true>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_seq_kernel<int32_t, false>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_seq_kernel<int64_t, true>));
    DM_CUDA(cudaFuncGetAttributes(&fa, nwk::nw_seq_kernel<int64_t, false>));
}

NwScheme make_scheme(const int16_t* table, const uint8_t* has_symbol, int open_surcharge, int gap_extend) {
    NwScheme s;
    for (int c = 0; c < 128; ++c) {
        s.has[c] = has_symbol[c] != 0;
        if (s.has[c]) s.lut[c] = (uint8_t)s.K++;
    }
    if (s.K == 0) throw invalid_argument("scoring scheme has no symbols");
    s.Kp = s.K | 1;
    s.table4.assign((size_t)s.K * s.Kp, 0);
    s.score.assign((size_t)s.K * s.K, 0);
    for (int x = 0; x < 128; ++x) {
        if (!s.has[x]) continue;
        for (int y = 0; y < 128; ++y) {
            if (!s.has[y]) continue;
            const int v = table[x * 128 + y];
            s.table4[(size_t)s.lut[x] * s.Kp + s.lut[y]] = 4 * v;
            s.score[(size_t)s.lut[x] * s.K + s.lut[y]] = (int16_t)v;
            s.maxabs = std::max(s.maxabs, std::abs(v));
        }
    }
    s.open = open_surcharge;
    s.extend = gap_extend;
    return s;
}

void set_columns(NwScheme& sc, const bool* present) {
    sc.KE = 0;
    std::memset(sc.plut, 0, sizeof(sc.plut));
    for (int c = 0; c < 128; ++c)
        if (present[c] && sc.has[c]) {
            sc.plut[c] = (uint8_t)sc.KE;
            sc.pdense[sc.KE] = sc.lut[c];
            ++sc.KE;
        }
}

namespace {
// Result slots and gap-list offsets of a batch (one layout for all shards).
uint64_t assign_layout(std::vector<NwJob>& jobs) {
    uint64_t gtot = 0;
    for (size_t k = 0; k < jobs.size(); ++k) {
        NwJob& jb = jobs[k];
        if (jb.n == 0 || jb.m == 0) throw invalid_argument("nw_align requires non-empty inputs");
        jb.slot = (uint32_t)k;
        jb.ga_off = gtot;
        gtot += jb.m;
        jb.gb_off = gtot;
        gtot += jb.n;
    }
    return gtot;
}
}  // namespace

void nw_run(dm_ctx* ctx, const uint8_t* d_chars, std::vector<NwJob>& jobs, const NwScheme& sc, NwOut& out,
            bool time_kernels, bool layout_given) {
    out.fwd_ms = out.tb_ms = 0.f;
    out.cells = 0;
    out.cells_exec = 0;
    out.launches = 0;
    const size_t nj = jobs.size();
    if (!layout_given) {
        const uint64_t gtot = assign_layout(jobs);
        out.d_res = ctx->nw_res.as<NwRes>(std::max<size_t>(nj, 1));
        out.d_gaps = ctx->nw_gaps.as<uint32_t>(std::max<uint64_t>(gtot, 1));
        out.gaps_total = gtot;
    }
    uint64_t ttot = 0;
    uint32_t nmmax = 0;
    const bool seq = use_seq(ctx, nj);
    for (const auto& jb : jobs) {
        nmmax = std::max(nmmax, jb.n + jb.m);
        out.cells += (uint64_t)jb.n * jb.m;
        out.cells_exec += (seq ? seq_rows(jb.n) : (uint64_t)((jb.n + nwk::BAND - 1) / nwk::BAND) * nwk::BAND) * jb.m;
        ttot += trace_bytes(jb, seq);
    }
    if (nj == 0) return;
    // tagged units: 4 * score (ring kernel), 256 * score (throughput kernel)
    // (the shifted domain of the forward kernels, nw_seq.cuh, moves values by
    // up to (n+m)|extend| and the scores by 2|extend|)
    const int64_t bound = ((int64_t)nmmax + 2) * (sc.maxabs + std::llabs(sc.open) + 4 * std::llabs(sc.extend)) *
                          (seq ? 256 : 4);
    const bool wide = bound >= (1ll << 28);
    SeqDev sd;
    const bool prof = seq && sc.KE > 0 && sc.KE <= 8;
    if (seq) {  // 256-scaled table (TAB) or profile table K x KE (PROF), and the column map
        std::vector<int32_t> t256((size_t)sc.K * sc.Kp, 0);
        for (int x = 0; x < sc.K; ++x)
            for (int y = 0; y < sc.K; ++y)
                t256[(size_t)x * sc.Kp + y] = 256 * (sc.score[(size_t)x * sc.K + y] - 2 * sc.extend);  // shifted domain
        std::vector<int32_t> pt((size_t)sc.K * std::max(sc.KE, 1), 0);
        for (int x = 0; x < sc.K; ++x)
            for (int c = 0; c < sc.KE; ++c)
                pt[(size_t)x * sc.KE + c] = 256 * (sc.score[(size_t)x * sc.K + sc.pdense[c]] - 2 * sc.extend);
        char* buf = (char*)ctx->nw_seqtab.get(t256.size() * 4 + pt.size() * 4 + 128 + 64);
        int32_t* d_t = (int32_t*)buf;
        int32_t* d_p = d_t + t256.size();
        uint8_t* d_pl = (uint8_t*)(d_p + pt.size());
        DM_CUDA(cudaMemcpyAsync(d_t, t256.data(), t256.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        DM_CUDA(cudaMemcpyAsync(d_p, pt.data(), pt.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        DM_CUDA(cudaMemcpyAsync(d_pl, sc.plut, 128, cudaMemcpyHostToDevice, ctx->stream));
        sd = SeqDev{d_t, d_p, d_pl};
    }
    const size_t smem = (size_t)sc.K * sc.Kp * 4;
    // ring / cluster kernels: 4 * (s - 2 * extend), the shifted domain (nw_fwd.cuh)
    std::vector<int32_t> t4s(sc.table4);
    for (int x = 0; x < sc.K; ++x)
        for (int y = 0; y < sc.K; ++y) t4s[(size_t)x * sc.Kp + y] -= (int32_t)(8 * sc.extend);
    const int32_t* d_table = ctx->nw_table.as<int32_t>(t4s.size());
    uint8_t* d_lut = (uint8_t*)ctx->aux2.get(128);
    DM_CUDA(cudaMemcpyAsync((void*)d_table, t4s.data(), t4s.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_lut, sc.lut, 128, cudaMemcpyHostToDevice, ctx->stream));

    // Larger alignments first (better tail balance), grouped by warps per
    // alignment; chunked by a trace-memory budget.
    std::vector<NwJob> sj(jobs);
    std::stable_sort(sj.begin(), sj.end(), [seq](const NwJob& x, const NwJob& y) {
        const int gx = seq ? 0 : group_of(x.n), gy = seq ? 0 : group_of(y.n);
        if (gx != gy) return gx > gy;
        return (uint64_t)x.n * x.m > (uint64_t)y.n * y.m;
    });
    // Trace budget: up to ~45 % of the device's free memory (every chunk ends
    // with a host sync and a half-empty last wave, so one chunk per batch is
    // best: a cfg4 merge level holds up to 2.4e10 cells = 24 GB of trace),
    // at least 6 GB; DM_NW_TRACE_GB caps it (tests).
    uint64_t cap = std::max<uint64_t>(6ull << 30, ctx->free_at_create / 100 * 45);
    if (const char* e = std::getenv("DM_NW_TRACE_GB")) cap = std::max<uint64_t>(1, (uint64_t)(std::atof(e) * (1ull << 30)));
    const uint64_t budget = std::max<uint64_t>(std::min<uint64_t>(ttot, cap), 1);
    size_t c0 = 0;
    while (c0 < nj) {
        size_t c1 = c0;
        uint64_t tb = 0;
        while (c1 < nj) {
            const uint64_t t = trace_bytes(sj[c1], seq);
            if (c1 > c0 && tb + t > budget) break;
            sj[c1].t_off = tb;
            tb += t;
            ++c1;
        }
        const uint32_t cnt = (uint32_t)(c1 - c0);
        uint8_t* d_trace = (uint8_t*)ctx->nw_trace.get(tb + 64);
        NwJob* d_jobs = ctx->nw_jobs.as<NwJob>(cnt);
        DM_CUDA(cudaMemcpyAsync(d_jobs, sj.data() + c0, cnt * sizeof(NwJob), cudaMemcpyHostToDevice, ctx->stream));
        uint32_t* d_cnt = ctx->counter.as<uint32_t>(kGroups + 1);  // one per group launch + the traceback
        DM_CUDA(cudaMemsetAsync(d_cnt, 0, (kGroups + 1) * sizeof(uint32_t), ctx->stream));
        if (time_kernels) DM_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        size_t g0 = c0;
        int gi = 0;
        if (seq) {  // one launch for the whole chunk
            uint32_t mmax = 1;
            for (size_t q = c0; q < c1; ++q) mmax = std::max(mmax, sj[q].m);
            nwk::SeqArgs sa{};
            sa.chars = d_chars;
            sa.jobs = d_jobs;
            sa.njobs = cnt;
            sa.lut = d_lut;
            sa.plut = sd.plut;
            sa.table = sd.table;
            sa.ptab = sd.ptab;
            sa.K = sc.K;
            sa.Kp = sc.Kp;
            sa.KE = sc.KE;
            sa.O = 256 * sc.open;
            sa.E = 256 * sc.extend;
            sa.trace = d_trace;
            sa.res = out.d_res;
            sa.counter = d_cnt;
            sa.one = 1;
            if (wide) {
                if (prof) launch_seq<int64_t, true>(ctx, sa, mmax);
                else launch_seq<int64_t, false>(ctx, sa, mmax);
            } else {
                if (prof) launch_seq<int32_t, true>(ctx, sa, mmax);
                else launch_seq<int32_t, false>(ctx, sa, mmax);
            }
            DM_CUDA(cudaGetLastError());
            out.launches += 1;
            ctx->launches += 1;
            g0 = c1;
        }
        if (!seq) {
            uint32_t mmax = 1;
            for (size_t q = c0; q < c1; ++q) mmax = std::max(mmax, sj[q].m);
            const int cl = clu_size(ctx, cnt, wide, mmax, sc);
            if (cl) {  // one cluster per alignment, one launch for the chunk
                nwk::FwdArgs fa{d_chars, d_jobs, cnt, d_lut, d_table, sc.K, sc.Kp, 4 * sc.open, 4 * sc.extend,
                                d_trace, out.d_res, d_cnt, 1};
                if (cl == 8) launch_clu<8>(ctx, fa, sc, mmax);
                else if (cl == 4) launch_clu<4>(ctx, fa, sc, mmax);
                else launch_clu<2>(ctx, fa, sc, mmax);
                DM_CUDA(cudaGetLastError());
                out.launches += 1;
                ctx->launches += 1;
                g0 = c1;
            }
        }
        // one launch per warps-per-alignment group, the groups side by side on
        // the side streams (one after another, each small launch ran alone)
        int ngroups = 0;
        for (size_t q = g0; q < c1; ++q)
            if (q == g0 || group_of(sj[q].n) != group_of(sj[q - 1].n)) ++ngroups;
        const bool fork = ngroups > 1;
        if (fork) {
            // the wrap rows (group 8 only) are allocated before the fork: a
            // stream-ordered allocation on ctx->stream after it would not be
            // ordered before the side stream's kernel
            uint64_t nwrap = 0, wm = 0;
            for (size_t q = g0; q < c1; ++q)
                if ((sj[q].n + nwk::BAND - 1) / nwk::BAND > 8) {
                    ++nwrap;
                    wm = std::max<uint64_t>(wm, sj[q].m);
                }
            if (nwrap) ctx->nw_wrap.get(nwrap * (wm + 1) * 3 * (wide ? 8 : 4));
            ensure_side_streams(ctx);
            DM_CUDA(cudaEventRecord(ctx->lev_fork, ctx->stream));
            for (int k = 0; k < std::min(ngroups, dm_ctx::kLevSide); ++k)
                DM_CUDA(cudaStreamWaitEvent(ctx->lev_side[k], ctx->lev_fork, 0));
        }
        while (g0 < c1) {
            const int grp = group_of(sj[g0].n);
            size_t g1 = g0;
            while (g1 < c1 && group_of(sj[g1].n) == grp) ++g1;
            nwk::FwdArgs fa{d_chars, d_jobs + (g0 - c0), (uint32_t)(g1 - g0), d_lut, d_table, sc.K, sc.Kp,
                            4 * sc.open, 4 * sc.extend, d_trace, out.d_res, d_cnt + gi, 1};
            uint32_t wrap_m = 0;  // widest alignment with more bands than warps
            for (size_t q = g0; q < g1; ++q)
                if ((sj[q].n + nwk::BAND - 1) / nwk::BAND > (uint32_t)grp) wrap_m = std::max(wrap_m, sj[q].m);
            cudaStream_t gst = fork ? ctx->lev_side[gi % dm_ctx::kLevSide] : ctx->stream;
            if (wide) launch_group<int64_t>(ctx, grp, fa, smem, wrap_m, gst);
            else launch_group<int32_t>(ctx, grp, fa, smem, wrap_m, gst);
            DM_CUDA(cudaGetLastError());
            out.launches += 1;
            ctx->launches += 1;
            g0 = g1;
            ++gi;
        }
        if (fork)
            for (int k = 0; k < std::min(ngroups, dm_ctx::kLevSide); ++k) {
                DM_CUDA(cudaEventRecord(ctx->lev_join[k], ctx->lev_side[k]));
                DM_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->lev_join[k], 0));
            }
        cudaEvent_t ev_fwd = nullptr, ev_tb = nullptr;
        if (time_kernels) {  // read after the chunk (no host sync between forward and traceback)
            DM_CUDA(cudaEventCreate(&ev_fwd));
            DM_CUDA(cudaEventCreate(&ev_tb));
            DM_CUDA(cudaEventRecord(ev_fwd, ctx->stream));
        }
        nvtxRangePushA("dm nw traceback");
        TbArgs ta{d_jobs, cnt, d_trace, out.d_res, out.d_gaps, d_cnt + kGroups, seq ? 1 : 0};
        const int tgrid = (int)std::max<uint64_t>(1, std::min<uint64_t>((cnt + 3) / 4, (uint64_t)ctx->sm_count * 8));
        nw_traceback_kernel<<<tgrid, 128, 0, ctx->stream>>>(ta);
        DM_CUDA(cudaGetLastError());
        if (time_kernels) {
            DM_CUDA(cudaEventRecord(ev_tb, ctx->stream));
            DM_CUDA(cudaEventSynchronize(ev_tb));
            float f = 0, t = 0;
            DM_CUDA(cudaEventElapsedTime(&f, ctx->ev0, ev_fwd));
            DM_CUDA(cudaEventElapsedTime(&t, ev_fwd, ev_tb));
            out.fwd_ms += f;
            out.tb_ms += t;
            cudaEventDestroy(ev_fwd);
            cudaEventDestroy(ev_tb);
        }
        out.launches += 1;
        ctx->launches += 1;
        nvtxRangePop();
        if (c1 < nj) DM_CUDA(cudaStreamSynchronize(ctx->stream));  // trace buffer reused by the next chunk
        c0 = c1;
    }
}

namespace {
struct CompactDesc {
    uint64_t src_a, src_b, dst;
    uint32_t na, nb;
};
__global__ void compact_gaps_kernel(const uint32_t* __restrict__ gaps, const CompactDesc* __restrict__ d, uint64_t n,
                                    uint32_t* __restrict__ out) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp; k < n; k += nwarps) {
        const CompactDesc c = d[k];
        for (uint32_t t = lane; t < c.na; t += 32) out[c.dst + t] = gaps[c.src_a + t];
        for (uint32_t t = lane; t < c.nb; t += 32) out[c.dst + c.na + t] = gaps[c.src_b + t];
    }
}
// inverse of compact_gaps_kernel: compacted entries back to the job's slots
__global__ void expand_gaps_kernel(const uint32_t* __restrict__ in, const CompactDesc* __restrict__ d, uint64_t n,
                                   uint32_t* __restrict__ gaps) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp; k < n; k += nwarps) {
        const CompactDesc c = d[k];
        for (uint32_t t = lane; t < c.na; t += 32) gaps[c.src_a + t] = in[c.dst + t];
        for (uint32_t t = lane; t < c.nb; t += 32) gaps[c.src_b + t] = in[c.dst + c.na + t];
    }
}
}  // namespace

namespace {
__global__ void bad_symbol_kernel(const uint8_t* __restrict__ b, uint64_t n, uint32_t hasmask0, uint32_t hasmask1,
                                  uint32_t hasmask2, uint32_t hasmask3, unsigned long long* __restrict__ first,
                                  uint32_t* __restrict__ seen) {
    const uint32_t m[4] = {hasmask0, hasmask1, hasmask2, hasmask3};
    uint32_t sm[4] = {0u, 0u, 0u, 0u};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t c = b[i];
        if (c < 128) sm[c >> 5] |= 1u << (c & 31);
        if (c >= 128 || !((m[c >> 5] >> (c & 31)) & 1u)) {
            atomicMin(first, (unsigned long long)i);
            break;  // later bytes of this thread are larger indices
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t v = __reduce_or_sync(0xffffffffu, sm[k]);
        if ((threadIdx.x & 31) == 0 && v) atomicOr(&seen[k], v);
    }
}
}  // namespace

uint64_t nw_first_bad_symbol(dm_ctx* ctx, const uint8_t* d_bytes, uint64_t n, const bool* has, bool* present) {
    if (n == 0) return UINT64_MAX;
    uint32_t m[4] = {0, 0, 0, 0};
    for (int c = 0; c < 128; ++c)
        if (has[c]) m[c >> 5] |= 1u << (c & 31);
    unsigned long long* d_first = ctx->aux.as<unsigned long long>(3);
    uint32_t* d_seen = reinterpret_cast<uint32_t*>(d_first + 1);
    DM_CUDA(cudaMemsetAsync(d_first, 0xff, 8, ctx->stream));
    DM_CUDA(cudaMemsetAsync(d_seen, 0, 16, ctx->stream));
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 8);
    bad_symbol_kernel<<<std::max(grid, 1), 256, 0, ctx->stream>>>(d_bytes, n, m[0], m[1], m[2], m[3], d_first,
                                                                 d_seen);
    DM_CUDA(cudaGetLastError());
    ctx->launches += 1;
    unsigned long long h[3] = {0, 0, 0};
    DM_CUDA(cudaMemcpyAsync(h, d_first, 24, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    if (present) {
        const uint32_t* sv = reinterpret_cast<const uint32_t*>(h + 1);
        for (int c = 0; c < 128; ++c) present[c] = (sv[c >> 5] >> (c & 31)) & 1u;
    }
    return h[0];
}

void nw_compact_gaps(dm_ctx* ctx, const uint32_t* d_gaps, const std::vector<NwJob>& jobs,
                     const std::vector<NwRes>& res, std::vector<uint32_t>& out, std::vector<uint64_t>& off) {
    const uint64_t n = jobs.size();
    off.assign(n + 1, 0);
    std::vector<CompactDesc> desc(n);
    for (uint64_t k = 0; k < n; ++k) {
        desc[k] = CompactDesc{jobs[k].ga_off, jobs[k].gb_off, off[k], res[k].nga, res[k].ngb};
        off[k + 1] = off[k] + res[k].nga + res[k].ngb;
    }
    out.resize(off[n]);
    if (off[n] == 0) return;
    CompactDesc* d_desc = (CompactDesc*)ctx->aux.get(n * sizeof(CompactDesc));
    uint32_t* d_out = ctx->aux2.as<uint32_t>(off[n]);
    DM_CUDA(cudaMemcpyAsync(d_desc, desc.data(), n * sizeof(CompactDesc), cudaMemcpyHostToDevice, ctx->stream));
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16));
    compact_gaps_kernel<<<grid, 256, 0, ctx->stream>>>(d_gaps, d_desc, n, d_out);
    DM_CUDA(cudaGetLastError());
    ++ctx->launches;
    DM_CUDA(cudaMemcpyAsync(out.data(), d_out, off[n] * 4, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Sharded batch: rank r aligns the cost-balanced range [bounds[r],
// bounds[r+1]) (cost n * m) into the batch's result layout; the ranks then
// all-gather the NwRes records and the COMPACTED gap lists (nga + ngb
// entries per job, not the m + n capacity), and every rank expands them into
// the layout, so all hold every result. Simulated worlds run the ranges in
// turn into the shared buffers (no exchange needed).
void nw_run_sharded(dm_ctx* ctx, const uint8_t* d_chars, std::vector<NwJob>& jobs, const NwScheme& sc,
                    NwOut& out, bool time_kernels, bool local) {
    const int w = local ? 1 : shard_world(ctx);
    if (w == 1 || jobs.size() < 2) {
        nw_run(ctx, d_chars, jobs, sc, out, time_kernels);
        return;
    }
    const size_t nj = jobs.size();
    const uint64_t gtot = assign_layout(jobs);
    out = NwOut{};
    out.d_res = ctx->nw_res.as<NwRes>(nj);
    out.d_gaps = ctx->nw_gaps.as<uint32_t>(std::max<uint64_t>(gtot, 1));
    out.gaps_total = gtot;
    std::vector<uint64_t> cost(nj), bounds;
    for (size_t k = 0; k < nj; ++k) cost[k] = (uint64_t)jobs[k].n * jobs[k].m;
    shard_bounds(cost.data(), nj, w, bounds);
    const bool real = comm_real(ctx);
    for (int r = 0; r < w; ++r) {
        if (real && r != ctx->rank) continue;
        const uint64_t lo = bounds[r], hi = bounds[r + 1];
        if (hi == lo) continue;
        std::vector<NwJob> sub(jobs.begin() + lo, jobs.begin() + hi);
        NwOut part;
        part.d_res = out.d_res;
        part.d_gaps = out.d_gaps;
        part.gaps_total = gtot;
        nw_run(ctx, d_chars, sub, sc, part, time_kernels, /*layout_given=*/true);
        out.fwd_ms += part.fwd_ms;
        out.tb_ms += part.tb_ms;
        out.cells += part.cells;
        out.cells_exec += part.cells_exec;
        out.launches += part.launches;
    }
    if (!real) return;
    // 1. results: all-gather each rank's NwRes range (padded to the largest)
    uint64_t maxc = 1;
    for (int r = 0; r < w; ++r) maxc = std::max<uint64_t>(maxc, bounds[r + 1] - bounds[r]);
    const uint64_t lo = bounds[ctx->rank], hi = bounds[ctx->rank + 1];
    NwRes* d_all = (NwRes*)ctx->nw_shard.get((uint64_t)(w + 1) * maxc * sizeof(NwRes));
    if (hi > lo)
        DM_CUDA(cudaMemcpyAsync(d_all + (uint64_t)ctx->rank * maxc, out.d_res + lo, (hi - lo) * sizeof(NwRes),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    comm_allgather(ctx, d_all + (uint64_t)ctx->rank * maxc, d_all, maxc * sizeof(NwRes));
    for (int r = 0; r < w; ++r)
        if (r != ctx->rank && bounds[r + 1] > bounds[r])
            DM_CUDA(cudaMemcpyAsync(out.d_res + bounds[r], d_all + (uint64_t)r * maxc,
                                    (bounds[r + 1] - bounds[r]) * sizeof(NwRes), cudaMemcpyDeviceToDevice,
                                    ctx->stream));
    std::vector<NwRes> res(nj);
    DM_CUDA(cudaMemcpyAsync(res.data(), out.d_res, nj * sizeof(NwRes), cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    // 2. gap lists: each rank compacts its own jobs', the compacted lists are
    // all-gathered (padded to the largest) and expanded into the layout
    std::vector<uint64_t> coff(nj + 1, 0), rank_g((size_t)w, 0);
    std::vector<CompactDesc> desc(nj);
    for (int r = 0; r < w; ++r) {
        uint64_t acc = 0;
        for (uint64_t k = bounds[r]; k < bounds[r + 1]; ++k) {
            coff[k] = acc;
            acc += res[k].nga + res[k].ngb;
        }
        rank_g[r] = acc;
    }
    uint64_t maxg = 1;
    for (int r = 0; r < w; ++r) maxg = std::max(maxg, rank_g[r]);
    uint32_t* d_cg = ctx->nw_shard_gaps.as<uint32_t>((uint64_t)(w + 1) * maxg);
    uint32_t* mine = d_cg + (uint64_t)ctx->rank * maxg;
    CompactDesc* d_desc = (CompactDesc*)ctx->aux.get(std::max<size_t>(nj, 1) * sizeof(CompactDesc));
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((nj + 7) / 8, (uint64_t)ctx->sm_count * 16));
    if (hi > lo) {
        for (uint64_t k = lo; k < hi; ++k)
            desc[k - lo] = CompactDesc{jobs[k].ga_off, jobs[k].gb_off, coff[k], res[k].nga, res[k].ngb};
        DM_CUDA(cudaMemcpyAsync(d_desc, desc.data(), (hi - lo) * sizeof(CompactDesc), cudaMemcpyHostToDevice,
                                ctx->stream));
        compact_gaps_kernel<<<grid, 256, 0, ctx->stream>>>(out.d_gaps, d_desc, hi - lo, mine);
        DM_CUDA(cudaGetLastError());
    }
    comm_allgather(ctx, mine, d_cg, maxg * sizeof(uint32_t));
    uint64_t nd = 0;
    for (int r = 0; r < w; ++r) {
        if (r == ctx->rank) continue;
        for (uint64_t k = bounds[r]; k < bounds[r + 1]; ++k)
            desc[nd++] = CompactDesc{jobs[k].ga_off, jobs[k].gb_off, (uint64_t)r * maxg + coff[k], res[k].nga,
                                     res[k].ngb};
    }
    if (nd) {
        DM_CUDA(cudaMemcpyAsync(d_desc, desc.data(), nd * sizeof(CompactDesc), cudaMemcpyHostToDevice, ctx->stream));
        expand_gaps_kernel<<<grid, 256, 0, ctx->stream>>>(d_cg, d_desc, nd, out.d_gaps);
        DM_CUDA(cudaGetLastError());
    }
    ctx->launches += 2;
}

}  // namespace dm
