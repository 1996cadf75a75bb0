// Gotoh NW forward pass, latency form across a thread-block CLUSTER (K5c),
// included by nw.cu after nw_fwd.cuh.
//
// The top merge levels hold a handful of long alignments (cfg4 depth 0: one
// 2,620 x 2,620 merge); one CTA per alignment leaves 147 SMs idle and runs
// each 512-row band's 16-row lane chain at the latency of one SM. Here one
// alignment runs on a cluster of CL CTAs (CL x NWW warps) with short bands of
// 32 x RRT rows (RRT = 4: 21 bands for 2,620 rows), band b on warp
// b mod (CL x NWW) of the cluster.
//
// Hand-off: every warp owns a FULL-WIDTH row in its CTA's shared memory (the
// (PM, GB, PGA) of columns 0..m of the row above its band). The band above --
// on another CTA of the cluster for the first warp of a CTA -- writes it
// through distributed shared memory and publishes the column count with a
// release store at cluster scope every CHUNK columns; the consumer acquires.
// No back-pressure is needed: a producer can only compute column j after
// the chain of bands between it and the consumer of the previous round has
// passed column j, i.e. after that consumer read it, so rows are rewritten
// in place round after round (more bands than warps) with no wrap buffer.
// Every spin is bounded (a trap instead of a hang).
//
// The column string b is staged in shared memory as score-table offsets (a
// cluster-scope acquire invalidates the L1, so a per-step global load of b
// would go to L2 every time). Per cell the arithmetic, tie-breaks and trace
// byte are the ring kernel's (nw_fwd.cuh: V = 4 score + tag, offset states,
// one vimax3 per state); the trace is written in the same column-major layout
// ([j-1][i-1], columns padded to 16 bytes), so the traceback kernel is shared.
#pragma once

#include <cooperative_groups.h>

namespace dm {
namespace nwk {

constexpr int CL_NWW = 4;      // warps per CTA
constexpr int CL_CHUNK = 16;   // publication granularity (columns)

__device__ __forceinline__ void st_release_cluster(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cluster.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cluster(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// spin until *p >= target (acquire); bounded: a lost hand-off traps instead of hanging the GPU
__device__ __forceinline__ void wait_at_least(const uint32_t* p, uint32_t target) {
    for (uint32_t it = 0; ld_acquire_cluster(p) < target; ++it)
        if (it > (1u << 28)) __trap();
}

// dynamic shared memory: table (K x Kp int32, padded to 16 B) | b's columns
// (m int32 table offsets, padded) | CL_NWW rows of (m + 1) x 3 int32
__host__ __device__ inline size_t clu_smem_bytes(int K, int Kp, uint32_t m) {
    return (((size_t)K * Kp + 3) & ~(size_t)3) * 4 + (((size_t)m + 4) & ~(size_t)3) * 4 +
           (size_t)CL_NWW * ((size_t)m + 1) * 12;
}

template <int RRT, int CL>
__global__ void __launch_bounds__(CL_NWW * 32, 1) nw_clu_kernel(const FwdArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) int32_t s_dyn[];
    __shared__ uint32_t s_pub[CL_NWW];  // columns published into row w (sequence: round * (m + 1) + column)
    __shared__ uint8_t s_lut[128];
    using V = int32_t;
    constexpr int BANDC = 32 * RRT;
    constexpr uint32_t W = CL * CL_NWW;  // warps of the cluster
    const uint32_t jid = blockIdx.x / CL;
    const NwJob job = a.jobs[jid < a.njobs ? jid : 0];
    const uint32_t n = job.n, m = job.m;
    int32_t* s_table = s_dyn;
    int32_t* s_bcol = s_dyn + ((a.K * a.Kp + 3) & ~3);
    int32_t* s_rows = s_bcol + ((m + 4) & ~3u);
    for (int x = threadIdx.x; x < a.K * a.Kp; x += blockDim.x) s_table[x] = a.table[x];
    for (int x = threadIdx.x; x < 128; x += blockDim.x) s_lut[x] = a.lut[x];
    if (threadIdx.x < CL_NWW) s_pub[threadIdx.x] = 0;
    __syncthreads();
    {
        const uint8_t* Bg = a.chars + job.b_off;
        for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) s_bcol[j] = (int)s_lut[Bg[j] & 127] * 4;
    }
    cluster.sync();  // every CTA's counters are zero before any remote access; b staged

    const uint32_t crank = cluster.block_rank();
    const int g = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const uint32_t gw = crank * CL_NWW + (uint32_t)w;  // warp index in the cluster
    const V NEG = neg_inf<V>();
    const V O4 = (V)a.O4;
    const char* tbytes = reinterpret_cast<const char*>(s_table);
    const uint32_t tag1 = (uint32_t)a.one, tag2 = tag1 + tag1, keep = ~(tag2 + tag1);
    const uint32_t four = tag2 + tag2, sixteen = four * four;
    const V NO4 = -O4;
    const int32_t* my_row = s_rows + (size_t)w * (m + 1) * 3;  // the row above this warp's bands

    if (jid < a.njobs) {
        const uint8_t* A = a.chars + job.a_off;
        const uint32_t pa = (n + 15) & ~15u;
        uint8_t* T = a.trace + job.t_off;
        const uint32_t nbands = (n + BANDC - 1) / BANDC;
        // the next band's warp and its row (local or another CTA's)
        const uint32_t ow = (gw + 1) % W;
        int32_t* out_row = cluster.map_shared_rank(s_rows + (size_t)(ow % CL_NWW) * (m + 1) * 3, ow / CL_NWW);
        uint32_t* out_pub = cluster.map_shared_rank(&s_pub[ow % CL_NWW], ow / CL_NWW);
        for (uint32_t band = gw; band < nbands; band += W) {
            const uint32_t i0 = band * BANDC + (uint32_t)g * RRT + 1;
            int rowoff[RRT];
            V LM[RRT], LGB[RRT], LGA[RRT];
#pragma unroll
            for (int r = 0; r < RRT; ++r) {
                const uint32_t i = i0 + r;
                rowoff[r] = (i <= n ? (int)s_lut[A[i - 1] & 127] : 0) * a.Kp * 4;
                LM[r] = (V)(NEG | 2) + O4;
                LGA[r] = NEG + O4;
                LGB[r] = (V)(a.O4 | 1) + O4;
            }
            V pmax = (i0 == 1 ? (V)2 : (V)(a.O4 | 1)) + O4;
            const uint32_t seq_in = (band / W) * (m + 1);
            const bool has_out = band + 1 < nbands;
            const uint32_t seq_out = ((band + 1) / W) * (m + 1);
            V sM = 0, sGB = 0, sGA = 0;
            // FIRST: band 0 (row 0 analytic); otherwise the row above from my_row
            auto run = [&](auto first_t) {
                constexpr bool FIRST = decltype(first_t)::value;
                auto step = [&](uint32_t s, auto chk) {
                    constexpr bool CHK = decltype(chk)::value;
                    const V rM = shfl_up1(sM), rGB = shfl_up1(sGB), rGA = shfl_up1(sGA);
                    if constexpr (CHK && !FIRST) {
                        if ((s % CL_CHUNK) == 0 && s < m) {  // columns s+1 .. s+CHUNK published
                            if (g == 0) wait_at_least(&s_pub[w], seq_in + min(s + CL_CHUNK, m));
                            __syncwarp();
                        }
                    }
                    const uint32_t j = s - (uint32_t)g + 1;
                    if (!CHK || j - 1 < m) {
                        V iM, iGB, iGA;
                        if constexpr (FIRST) {
                            iM = (V)(NEG | 2) + O4;
                            iGB = (V)(NEG | 1);
                            iGA = (V)a.O4 + O4;  // row 0 in the shifted domain (nw_seq.cuh)
                        } else {
                            const int32_t* e = my_row + (size_t)(s + 1) * 3;
                            iM = e[0];
                            iGB = e[1];
                            iGA = e[2];
                        }
                        V uM = g == 0 ? iM : rM;
                        V uGB = g == 0 ? iGB : rGB;
                        V uGA = g == 0 ? iGA : rGA;
                        V dmax = pmax;
                        pmax = vmax3(uM, add_fma(uGB, O4, a.one), uGA);
                        const int cb4 = s_bcol[j - 1];
                        uint32_t tw[RRT / 4];
                        uint32_t tm[4], tgb[4], tga[4];
#pragma unroll
                        for (int r = 0; r < RRT; ++r) {
                            const int32_t sc =
                                *reinterpret_cast<const int32_t*>(tbytes + add_fma(rowoff[r], cb4, a.one));
                            const V mo = add_fma(dmax, (V)sc, a.one);
                            dmax = vmax3(LM[r], LGB[r], LGA[r]);
                            const V gao = add_fma(vmax3(LM[r], LGB[r], add_fma(LGA[r], NO4, a.one)), O4, a.one);
                            const V gbraw = vmax3(uM, uGB, uGA);  // shifted domain: no extend
                            tm[r & 3] = (uint32_t)mo;
                            tgb[r & 3] = (uint32_t)gbraw;
                            tga[r & 3] = (uint32_t)gao;
                            if ((r & 3) == 3) {
                                const uint32_t wm = gather_lo(tm[0], tm[1], tm[2], tm[3]);
                                const uint32_t wb = gather_lo(tgb[0], tgb[1], tgb[2], tgb[3]);
                                const uint32_t wa = gather_lo(tga[0], tga[1], tga[2], tga[3]);
                                tw[r >> 2] =
                                    bitsel(bitsel(wm, umul(wb, four), 0x03030303u), umul(wa, sixteen), 0x0F0F0F0Fu);
                            }
                            LM[r] = retag(mo, keep, tag2);
                            const V lgb = retag(gbraw, keep, tag1);
                            LGB[r] = add_fma(lgb, O4, a.one);
                            LGA[r] = retag(gao, keep, 0u);
                            uM = LM[r];
                            uGB = lgb;
                            uGA = LGA[r];
                        }
                        sM = uM;
                        sGB = uGB;
                        sGA = uGA;
                        if (i0 <= n) {
                            uint8_t* dst = T + (uint64_t)(j - 1) * pa + (i0 - 1);
                            if constexpr (RRT == 4) *reinterpret_cast<uint32_t*>(dst) = tw[0];
                            else if constexpr (RRT == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(tw[0], tw[1]);
                            else *reinterpret_cast<uint4*>(dst) = make_uint4(tw[0], tw[1], tw[2], tw[3]);
                        }
                        if (has_out && g == 31) {
                            int32_t* e = out_row + (size_t)j * 3;
                            e[0] = uM;
                            e[1] = uGB;
                            e[2] = uGA;
                            if (CHK && ((j % CL_CHUNK) == 0 || j == m)) st_release_cluster(out_pub, seq_out + j);
                        }
                    }
                };
                const uint32_t steps = m + 31;
                uint32_t s = 0;
                for (; s < min(32u, steps); ++s) step(s, std::true_type{});
                if (m > 32) {
                    const uint32_t s_end = 32 + ((m - 32) & ~(uint32_t)(CL_CHUNK - 1));
#pragma unroll 1
                    for (; s < s_end; s += CL_CHUNK) {
                        if constexpr (!FIRST) {
                            if (g == 0) wait_at_least(&s_pub[w], seq_in + min(s + CL_CHUNK, m));
                            __syncwarp();
                        }
#pragma unroll 1
                        for (uint32_t q = 0; q < CL_CHUNK; ++q) step(s + q, std::false_type{});
                        // lane 31 wrote columns through s + CHUNK - 31 (the release orders them)
                        if (has_out && g == 31) st_release_cluster(out_pub, seq_out + (s + CL_CHUNK - 1 - 30));
                    }
                }
                for (; s < steps; ++s) step(s, std::true_type{});
            };
            if (band == 0) run(std::true_type{});
            else run(std::false_type{});
            if (n >= i0 && n < i0 + RRT) {
                V fM = LM[0], fGB = LGB[0], fGA = LGA[0];
#pragma unroll
                for (int r = 1; r < RRT; ++r)
                    if (i0 + r == n) {
                        fM = LM[r];
                        fGB = LGB[r];
                        fGA = LGA[r];
                    }
                const V fin = vmax3(fM, fGB, fGA) - O4;
                a.res[job.slot].score = (int64_t)(fin >> 2) + (int64_t)(n + m) * (a.E4 / 4);
                a.res[job.slot].final_tag = (uint32_t)(fin & 3);
            }
            __syncwarp();
        }
    }
    cluster.sync();  // no CTA leaves while another may still write into its shared memory
}

}  // namespace nwk
}  // namespace dm
