// Pairwise aligner: batched Gotoh Needleman-Wunsch
// with device-side traceback, bit-exact with nw_align (pairwise.cpp:301-415).
//
// Forward (K5): one warp per alignment. Lane g owns RR consecutive rows of
// a 32*RR-row pass and sweeps the columns of b as a diagonal pipeline (lane
// g is on column s-g+1 at step s); the bottom row of lane g-1 arrives by
// __shfl_up each step, the bottom row of a pass is parked in a per-warp
// buffer for the next pass. Scores are kept in "tagged" form
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
#include "nw.h"

namespace dm {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int RR = 16;  // rows per lane
constexpr int PASS = 32 * RR;

template <class V>
__device__ __forceinline__ V neg_inf();
template <>
__device__ __forceinline__ int32_t neg_inf<int32_t>() { return -(1 << 30); }
template <>
__device__ __forceinline__ int64_t neg_inf<int64_t>() { return -(1ll << 60); }

__device__ __forceinline__ int32_t vmax3(int32_t a, int32_t b, int32_t c) { return __vimax3_s32(a, b, c); }
__device__ __forceinline__ int64_t vmax3(int64_t a, int64_t b, int64_t c) { return max(max(a, b), c); }
__device__ __forceinline__ int32_t addmax(int32_t a, int32_t b, int32_t c) { return __viaddmax_s32(a, b, c); }
__device__ __forceinline__ int64_t addmax(int64_t a, int64_t b, int64_t c) { return max(a + b, c); }

template <class V>
__device__ __forceinline__ V shfl_up(V v) {
    if constexpr (sizeof(V) == 4) {
        return __shfl_up_sync(FULL, v, 1);
    } else {
        return (V)__shfl_up_sync(FULL, (long long)v, 1);
    }
}

struct FwdArgs {
    const uint8_t* chars;
    const NwJob* jobs;
    uint32_t njobs;
    const uint8_t* lut;
    const int32_t* table;  // 4*score, K x Kp
    int K, Kp;
    int64_t O4, E4;
    uint8_t* trace;
    void* passbuf;  // per warp: 3 x (mmax+1) values
    uint32_t mmax;
    NwRes* res;
    uint32_t* counter;
};

template <class V>
__global__ void __launch_bounds__(128) nw_fwd_kernel(const FwdArgs a) {
    extern __shared__ int32_t s_table[];
    __shared__ uint8_t s_lut[128];
    for (int x = threadIdx.x; x < a.K * a.Kp; x += blockDim.x) s_table[x] = a.table[x];
    for (int x = threadIdx.x; x < 128; x += blockDim.x) s_lut[x] = a.lut[x];
    __syncthreads();
    const int g = threadIdx.x & 31;
    const uint32_t wglob = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    V* pbuf = reinterpret_cast<V*>(a.passbuf) + (uint64_t)wglob * 3 * (a.mmax + 1);
    const V NEG = neg_inf<V>();
    const V O4 = (V)a.O4, E4 = (V)a.E4;
    for (;;) {
        uint32_t jid = 0;
        if (g == 0) jid = atomicAdd(a.counter, 1u);
        jid = __shfl_sync(FULL, jid, 0);
        if (jid >= a.njobs) break;
        const NwJob job = a.jobs[jid];
        const uint32_t n = job.n, m = job.m;
        const uint8_t* A = a.chars + job.a_off;
        const uint8_t* B = a.chars + job.b_off;
        const uint32_t pa = (n + 15) & ~15u;
        uint8_t* T = a.trace + job.t_off;
        for (uint32_t p0 = 0; p0 < n; p0 += PASS) {
            const uint32_t i0 = p0 + (uint32_t)g * RR + 1;
            int ca[RR];
            V LM[RR], LGB[RR], LGA[RR];
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const uint32_t i = i0 + r;
                ca[r] = i <= n ? (int)s_lut[A[i - 1] & 127] * a.Kp : 0;
                LM[r] = (V)(NEG | 2);
                LGA[r] = NEG;
                LGB[r] = (V)((a.O4 + (int64_t)i * a.E4) | 1);  // column 0: GB = open + i*extend
            }
            // values of row i0-1 at column 0 (the first row's diagonal at column 1)
            V pM, pGB, pGA;
            if (i0 == 1) {
                pM = 2;  // M[0][0] = 0
                pGB = (V)(NEG | 1);
                pGA = NEG;
            } else {
                pM = (V)(NEG | 2);
                pGB = (V)((a.O4 + (int64_t)(i0 - 1) * a.E4) | 1);
                pGA = NEG;
            }
            V sM = 0, sGB = 0, sGA = 0;
            const bool store_pass = (g == 31) && (p0 + PASS < n);
            const uint32_t steps = m + 31;
            for (uint32_t s = 0; s < steps; ++s) {
                const V rM = shfl_up(sM), rGB = shfl_up(sGB), rGA = shfl_up(sGA);
                const uint32_t j = s - (uint32_t)g + 1;  // 1..m when active
                if (j - 1 < m) {
                    V uM, uGB, uGA;
                    if (g == 0) {
                        if (p0 == 0) {  // row 0 (pairwise.cpp:322-330)
                            uM = (V)(NEG | 2);
                            uGB = (V)(NEG | 1);
                            uGA = (V)(a.O4 + (int64_t)j * a.E4);
                        } else {
                            uM = pbuf[j];
                            uGB = pbuf[(a.mmax + 1) + j];
                            uGA = pbuf[2 * (a.mmax + 1) + j];
                        }
                    } else {
                        uM = rM;
                        uGB = rGB;
                        uGA = rGA;
                    }
                    V dM = pM, dGB = pGB, dGA = pGA;
                    pM = uM;
                    pGB = uGB;
                    pGA = uGA;
                    const int cb = s_lut[B[j - 1] & 127];
                    uint32_t tw[RR / 4];
#pragma unroll
                    for (int q = 0; q < RR / 4; ++q) tw[q] = 0;
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        const V mraw = vmax3(dM, dGB, dGA) + (V)s_table[ca[r] + cb];
                        const V gbraw = addmax(uGA, O4, addmax(uM, O4, uGB)) + E4;
                        const V garaw = addmax(LGB[r], O4, addmax(LM[r], O4, LGA[r])) + E4;
                        const V nM = (mraw & ~(V)3) | 2;
                        const V nGB = (gbraw & ~(V)3) | 1;
                        const V nGA = garaw & ~(V)3;
                        const uint32_t code = ((uint32_t)mraw & 3u) | (((uint32_t)gbraw & 3u) << 2) |
                                              (((uint32_t)garaw & 3u) << 4);
                        tw[r >> 2] |= code << ((r & 3) * 8);
                        if (j == m && i0 + r == n) {  // pairwise.cpp:374-375
                            const V fin = vmax3(nM, nGB, nGA);
                            a.res[jid].score = (int64_t)(fin >> 2);
                            a.res[jid].final_tag = (uint32_t)(fin & 3);
                        }
                        dM = LM[r];
                        dGB = LGB[r];
                        dGA = LGA[r];
                        LM[r] = nM;
                        LGB[r] = nGB;
                        LGA[r] = nGA;
                        uM = nM;
                        uGB = nGB;
                        uGA = nGA;
                    }
                    sM = uM;
                    sGB = uGB;
                    sGA = uGA;
                    if (store_pass) {
                        pbuf[j] = uM;
                        pbuf[(a.mmax + 1) + j] = uGB;
                        pbuf[2 * (a.mmax + 1) + j] = uGA;
                    }
                    if (i0 <= n)
                        *reinterpret_cast<uint4*>(T + (uint64_t)(j - 1) * pa + (i0 - 1)) =
                            make_uint4(tw[0], tw[1], tw[2], tw[3]);
                }
            }
            __syncwarp();
        }
    }
}

struct TbArgs {
    const NwJob* jobs;
    uint32_t njobs;
    const uint8_t* trace;
    NwRes* res;
    uint32_t* gaps;
    uint32_t* counter;
};

constexpr int TC = 32;  // tile columns (one per lane)
constexpr int TR = 64;  // tile rows (bytes per column)

__global__ void __launch_bounds__(128) nw_traceback_kernel(const TbArgs a) {
    __shared__ __align__(16) uint8_t tile[4][TC][TR];
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
        uint32_t state = 2u - a.res[jid].final_tag;  // 0 M, 1 GapB, 2 GapA
        uint32_t i = n, j = job.m, len = 0, nga = 0, ngb = 0;
        while (i > 0 && j > 0) {
            const uint32_t jtop = j;
            const int r0 = max(0, (int)((i - 1) & ~15u) - (TR - 16));
            const int jc = (int)jtop - g;
            if (jc >= 1) {
                const uint4* src = reinterpret_cast<const uint4*>(T + (uint64_t)(jc - 1) * pa + r0);
                uint4* dst = reinterpret_cast<uint4*>(&tile[w][g][0]);
#pragma unroll
                for (int q = 0; q < TR / 16; ++q)
                    if ((uint32_t)(r0 + q * 16) < pa) dst[q] = src[q];
            }
            __syncwarp();
            if (g == 0) {
                // pairwise.cpp:384-409, inside the staged tile
                while (i > 0 && j > 0 && jtop - j < (uint32_t)TC && (int)(i - 1) >= r0) {
                    const uint32_t code = tile[w][jtop - j][(i - 1) - r0];
                    ++len;
                    if (state == 0) {
                        state = 2u - (code & 3u);
                        --i;
                        --j;
                    } else if (state == 1) {
                        gb[ngb++] = j;
                        state = 2u - ((code >> 2) & 3u);
                        --i;
                    } else {
                        ga[nga++] = i;
                        state = 2u - ((code >> 4) & 3u);
                        --j;
                    }
                }
            }
            i = __shfl_sync(FULL, i, 0);
            j = __shfl_sync(FULL, j, 0);
            state = __shfl_sync(FULL, state, 0);
            __syncwarp();
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
            a.res[jid].len = len;
            a.res[jid].nga = nga;
            a.res[jid].ngb = ngb;
        }
    }
}

template <class V>
void launch_fwd(dm_ctx* ctx, const FwdArgs& fa, int grid, size_t smem) {
    DM_CUDA(cudaFuncSetAttribute(nw_fwd_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nw_fwd_kernel<V><<<grid, 128, smem, ctx->stream>>>(fa);
}

template <class V>
int fwd_occupancy(size_t smem) {
    int occ = 0;
    DM_CUDA(cudaFuncSetAttribute(nw_fwd_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nw_fwd_kernel<V>, 128, smem));
    return std::max(occ, 1);
}

}  // namespace

NwScheme make_scheme(const int16_t* table, const uint8_t* has_symbol, int open_surcharge, int gap_extend) {
    NwScheme s;
    for (int c = 0; c < 128; ++c) {
        s.has[c] = has_symbol[c] != 0;
        if (s.has[c]) s.lut[c] = (uint8_t)s.K++;
    }
    if (s.K == 0) throw invalid_argument("scoring scheme has no symbols");
    s.Kp = s.K | 1;
    s.table4.assign((size_t)s.K * s.Kp, 0);
    for (int x = 0; x < 128; ++x) {
        if (!s.has[x]) continue;
        for (int y = 0; y < 128; ++y) {
            if (!s.has[y]) continue;
            const int v = table[x * 128 + y];
            s.table4[(size_t)s.lut[x] * s.Kp + s.lut[y]] = 4 * v;
            s.maxabs = std::max(s.maxabs, std::abs(v));
        }
    }
    s.open = open_surcharge;
    s.extend = gap_extend;
    return s;
}

void nw_run(dm_ctx* ctx, const uint8_t* d_chars, std::vector<NwJob>& jobs, const NwScheme& sc, NwOut& out,
            bool time_kernels) {
    out.fwd_ms = out.tb_ms = 0.f;
    out.cells = 0;
    out.launches = 0;
    const size_t nj = jobs.size();
    // outputs: results + gap lists
    uint64_t gtot = 0, ttot = 0;
    uint32_t mmax = 0, nmmax = 0;
    for (auto& jb : jobs) {
        if (jb.n == 0 || jb.m == 0) throw invalid_argument("nw_align requires non-empty inputs");
        jb.ga_off = gtot;
        gtot += jb.m;
        jb.gb_off = gtot;
        gtot += jb.n;
        mmax = std::max(mmax, jb.m);
        nmmax = std::max(nmmax, jb.n + jb.m);
        out.cells += (uint64_t)jb.n * jb.m;
        ttot += (uint64_t)jb.m * ((jb.n + 15) & ~15u);
    }
    out.d_res = ctx->nw_res.as<NwRes>(std::max<size_t>(nj, 1));
    out.d_gaps = ctx->nw_gaps.as<uint32_t>(std::max<uint64_t>(gtot, 1));
    out.gaps_total = gtot;
    if (nj == 0) return;
    const int64_t bound = ((int64_t)nmmax + 2) * (sc.maxabs + std::llabs(sc.open) + std::llabs(sc.extend)) * 4;
    const bool wide = bound >= (1ll << 28);
    const size_t smem = (size_t)sc.K * sc.Kp * 4;
    const int32_t* d_table = ctx->nw_table.as<int32_t>(sc.table4.size());
    uint8_t* d_lut = (uint8_t*)ctx->aux2.get(128);
    DM_CUDA(cudaMemcpyAsync((void*)d_table, sc.table4.data(), sc.table4.size() * 4, cudaMemcpyHostToDevice,
                            ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_lut, sc.lut, 128, cudaMemcpyHostToDevice, ctx->stream));

    // chunk by trace budget
    const uint64_t budget = std::max<uint64_t>(ttot < (6ull << 30) ? ttot : (6ull << 30), 1);
    const int occ = wide ? fwd_occupancy<int64_t>(smem) : fwd_occupancy<int32_t>(smem);
    size_t c0 = 0;
    while (c0 < nj) {
        size_t c1 = c0;
        uint64_t tb = 0;
        while (c1 < nj) {
            const uint64_t t = (uint64_t)jobs[c1].m * ((jobs[c1].n + 15) & ~15u);
            if (c1 > c0 && tb + t > budget) break;
            jobs[c1].t_off = tb;
            tb += t;
            ++c1;
        }
        const uint32_t cnt = (uint32_t)(c1 - c0);
        uint8_t* d_trace = (uint8_t*)ctx->nw_trace.get(tb + 64);
        NwJob* d_jobs = ctx->nw_jobs.as<NwJob>(cnt);
        DM_CUDA(cudaMemcpyAsync(d_jobs, jobs.data() + c0, cnt * sizeof(NwJob), cudaMemcpyHostToDevice, ctx->stream));
        uint32_t* d_cnt = ctx->counter.as<uint32_t>(2);
        DM_CUDA(cudaMemsetAsync(d_cnt, 0, 8, ctx->stream));
        const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((cnt + 3) / 4, (uint64_t)occ * ctx->sm_count));
        const uint64_t warps = (uint64_t)grid * 4;
        void* d_pass = ctx->nw_in.get(warps * 3 * (mmax + 1) * (wide ? 8 : 4));
        FwdArgs fa{d_chars, d_jobs, cnt, d_lut, d_table, sc.K, sc.Kp, 4 * sc.open, 4 * sc.extend, d_trace, d_pass,
                   mmax, out.d_res + c0, d_cnt};
        if (time_kernels) DM_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        if (wide) launch_fwd<int64_t>(ctx, fa, grid, smem);
        else launch_fwd<int32_t>(ctx, fa, grid, smem);
        DM_CUDA(cudaGetLastError());
        if (time_kernels) {
            DM_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
            DM_CUDA(cudaEventSynchronize(ctx->ev1));
            float ms = 0;
            DM_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            out.fwd_ms += ms;
            DM_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        }
        TbArgs ta{d_jobs, cnt, d_trace, out.d_res + c0, out.d_gaps, d_cnt + 1};
        const int tgrid = (int)std::max<uint64_t>(1, std::min<uint64_t>((cnt + 3) / 4, (uint64_t)ctx->sm_count * 8));
        nw_traceback_kernel<<<tgrid, 128, 0, ctx->stream>>>(ta);
        DM_CUDA(cudaGetLastError());
        if (time_kernels) {
            DM_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
            DM_CUDA(cudaEventSynchronize(ctx->ev1));
            float ms = 0;
            DM_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            out.tb_ms += ms;
        }
        out.launches += 2;
        ctx->launches += 2;
        if (c1 < nj) DM_CUDA(cudaStreamSynchronize(ctx->stream));  // trace buffer reused by the next chunk
        c0 = c1;
    }
}

}  // namespace dm
