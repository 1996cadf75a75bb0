// Gotoh NW forward pass, throughput form (K5b), included by nw.cu.
//
// One warp per alignment, its 512-row bands swept one after another by the
// same warp: no CTA-wide rings, barriers or spin-waits, so warps of a batch
// with many alignments (the NW micro-benchmark, the lower merge levels) run
// independently. The row leaving band b goes to band b+1 through a per-warp
// row in global memory (L2; lane 31 writes column j 30 steps after lane 0
// read it, so the row is rewritten in place), which lane 0 streams into a
// shared-memory FIFO with cp.async.cg FIFO - 1 columns ahead.
//
// Per cell, relative to the ring kernel (nw_fwd.cuh), which keeps serving
// small batches where one alignment's latency matters:
//  * tagged values are 256 * score + tag (not 4 * score + tag): the low byte
//    of every state is its tag alone, so the three trace codes combine with
//    two IMADs (mo + 4 gb + 16 ga, FMA pipe) and four cells' bytes gather
//    with three PRMTs -- 0.75 ALU + 2 FMA per cell instead of 2.75 ALU +
//    0.5 FMA (the kernel is ALU-bound: 3 max3 + 3 retags per cell remain);
//  * PROF (<= 8 distinct column symbols, nucleotide merges): each lane keeps
//    a query profile in shared memory -- for every column symbol the scores
//    of its rows, laid out [symbol][row quad][lane][4] -- so a step reads its
//    rows' scores with RR/4 conflict-free LDS.128 from one base address
//    instead of RR address IMADs + RR LDS.32 (which conflicted on 61 % of
//    their wavefronts); TAB (protein, custom schemes) reads the K x Kp table;
//  * the last band of an alignment uses 12, 8 or 4 rows per lane when it has
//    at most 384 / 256 / 128 rows, so the padded rows per alignment drop from
//    up to 511 to at most 127 (cells_executed).
//  * shifted domain: every state is kept as X''(i,j) = X(i,j) - (i+j)*extend
//    (one constant per cell, so every max compares the same candidates with
//    the same ties). Both gap chains then lose their "+ extend" (the row
//    chain's add is gone, the column's open+extend becomes open), and the
//    diagonal's -2*extend is folded into the score table / profiles (host,
//    nw.cu); row 0 / column 0 become constants and the final score adds
//    (n+m)*extend back. One IMAD per cell fewer.
// Same recurrence, tie-breaks and trace byte (tagM | tagGB << 2 | tagGA << 4)
// as nw_fwd.cuh / pairwise.cpp:332-372; the traceback kernel is shared.
#pragma once

#include <type_traits>

namespace dm {
namespace nwk {

#ifndef DM_NW_SEQ_WARPS
#define DM_NW_SEQ_WARPS 4
#endif
constexpr int SEQ_WARPS = DM_NW_SEQ_WARPS;  // warps per CTA (independent alignments)
#ifndef DM_NW_SEQ_MINB
#define DM_NW_SEQ_MINB 3  // resident CTAs per SM the int32 kernels are built for (<= 170 registers: measured
                          // faster than 4 CTAs at 128 registers, 1100 vs 1036 GCUPS at L = 1000)
#endif

// a * b + c on the FMA pipe (b opaque)
__device__ __forceinline__ uint32_t imad_u(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// rows per lane of an alignment's last band holding `left` rows (1..512)
__host__ __device__ __forceinline__ uint32_t seq_tail_rr(uint32_t left) {
#ifdef DM_NW_SEQ_NO12
    return left > 256 ? 16u : left > 128 ? 8u : 4u;
#else
    return left > 384 ? 16u : left > 256 ? 12u : left > 128 ? 8u : 4u;
#endif
}

struct SeqArgs {
    const uint8_t* chars;
    const NwJob* jobs;
    uint32_t njobs;
    const uint8_t* lut;    // char -> dense code (TAB rows and columns; PROF rows)
    const uint8_t* plut;   // char -> profile symbol (PROF columns)
    const int32_t* table;  // 256 * score, K x Kp (dense codes)
    const int32_t* ptab;   // PROF: 256 * score, K x KE (row dense code, column profile symbol)
    int K, Kp, KE;
    int64_t O, E;          // 256 * open surcharge, 256 * extend
    uint8_t* trace;
    NwRes* res;
    uint32_t* counter;
    int32_t one;           // == 1 (opaque to ptxas)
    int4* hrow;            // per-warp hand-off rows (V = int32: 1 int4 per column; int64: 2)
    uint64_t hstride;      // int4 per warp
};

// One column of the hand-off row: the bottom row's (PM, GB, PGA) and the
// column's symbol code (profile symbol with PROF, dense code with TAB), so
// no lane loads b: lane 0 takes the code from the row, the others from the
// lane above with the states.
template <class V>
struct Cell4;
template <>
struct Cell4<int32_t> {
    static __device__ __forceinline__ void store(int4* p, int32_t m, int32_t gb, int32_t ga, uint32_t code) {
        *p = make_int4(m, gb, ga, (int)code);
    }
    static __device__ __forceinline__ void read(const int4* p, int32_t& m, int32_t& gb, int32_t& ga,
                                                uint32_t& code) {
        const int4 v = *p;
        m = v.x;
        gb = v.y;
        ga = v.z;
        code = (uint32_t)v.w;
    }
    static constexpr int words = 1;
};
template <>
struct Cell4<int64_t> {
    static __device__ __forceinline__ void store(int4* p, int64_t m, int64_t gb, int64_t ga, uint32_t code) {
        reinterpret_cast<longlong2*>(p)[0] = make_longlong2(m, gb);
        reinterpret_cast<longlong2*>(p)[1] = make_longlong2(ga, (long long)code);
    }
    static __device__ __forceinline__ void read(const int4* p, int64_t& m, int64_t& gb, int64_t& ga,
                                                uint32_t& code) {
        const longlong2 v0 = reinterpret_cast<const longlong2*>(p)[0];
        const longlong2 v1 = reinterpret_cast<const longlong2*>(p)[1];
        m = v0.x;
        gb = v0.y;
        ga = v1.x;
        code = (uint32_t)v1.y;
    }
    static constexpr int words = 2;
};

// Lane 0's input row goes through a per-warp FIFO in shared memory, filled
// FIFO columns ahead by cp.async.cg (L2 -> smem, no L1: the row is rewritten
// in place by the same warp), so the L2 latency is off the step's path.
constexpr int FIFO = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile(
        "{ .reg .pred p; setp.ne.u32 p, %2, 0;\n"
        "  @p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(sa),
        "l"(gmem), "r"((uint32_t)pred)
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <class V>
__device__ __forceinline__ void fifo_fetch(int4* slot, const int4* src, bool pred) {  // one column
#pragma unroll
    for (int k = 0; k < Cell4<V>::words; ++k) cp_async16(slot + k, src + k, pred);
}

template <class V>
__device__ __forceinline__ V neg_inf256();
template <>
__device__ __forceinline__ int32_t neg_inf256<int32_t>() { return -(1 << 29); }
template <>
__device__ __forceinline__ int64_t neg_inf256<int64_t>() { return -(1ll << 60); }

// (x & ~255) | tag as ONE LOP3 (keep = ~255 held in a register)
__device__ __forceinline__ int32_t retag256(int32_t x, uint32_t keep, uint32_t tag) {
    return (int32_t)lop3<0xEA>((uint32_t)x, keep, tag);
}
__device__ __forceinline__ int64_t retag256(int64_t x, uint32_t, uint32_t tag) {
    return (x & ~(int64_t)255) | (int64_t)tag;
}
// low 32 bits (the trace code sits in the low byte)
__device__ __forceinline__ uint32_t lo32(int32_t x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t lo32(int64_t x) { return (uint32_t)(uint64_t)x; }

// One band of RR rows per lane (32 * RR rows), swept over all m columns.
template <class V, bool PROF, int RR>
__device__ __forceinline__ void seq_band(const SeqArgs& a, const NwJob& job, uint32_t band, int4* hin,
                                         const int32_t* s_table, int4* s_prof, const uint8_t* s_plut,
                                         const uint8_t* s_lut, int4* s_fifo, uint32_t keep, uint32_t four,
                                         uint32_t sixteen) {
    const int g = threadIdx.x & 31;
    const uint32_t n = job.n, m = job.m;
    const uint8_t* A = a.chars + job.a_off;
    uint8_t* T = a.trace + job.t_off;
    const V NEG = neg_inf256<V>();
    const V O = (V)a.O, NO = -O;
    const uint32_t i0 = band * BAND + (uint32_t)g * RR + 1;
    const uint32_t tag1 = (uint32_t)a.one, tag2 = tag1 + tag1;

    [[maybe_unused]] int rowoff[RR];
    V LM[RR], LGB[RR], LGA[RR];  // PM, PGB, PGA of the lane's rows at the previous column
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        const uint32_t i = i0 + r;
        const int rc = i <= n ? (int)s_lut[A[i - 1] & 127] : 0;
        if constexpr (!PROF) rowoff[r] = rc * a.Kp * 4;
        LM[r] = (V)(NEG | 2) + O;
        LGA[r] = NEG + O;
        LGB[r] = (V)(a.O | 1) + O;  // column 0: GB = open + i*extend, i.e. open in the shifted domain
    }
    if constexpr (PROF) {
        // this lane's rows against every column symbol: [sym][quad][lane][4]
        int32_t* p = reinterpret_cast<int32_t*>(s_prof);
        for (int c = 0; c < a.KE; ++c) {
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const uint32_t i = i0 + r;
                const int rc = i <= n ? (int)s_lut[A[i - 1] & 127] : 0;
                p[((c * (RR / 4) + r / 4) * 32 + g) * 4 + (r & 3)] = __ldg(a.ptab + rc * a.KE + c);
            }
        }
        __syncwarp();
    }
    V pmax = (i0 == 1 ? (V)2 : (V)(a.O | 1)) + O;
    V sM = 0, sGB = 0, sGA = 0;
    // lane 0's input row (the band above, or row 0): columns 1..FIFO in flight
    constexpr int W4 = Cell4<V>::words;
#pragma unroll
    for (int k = 0; k < FIFO; ++k) {
        fifo_fetch<V>(s_fifo + k * W4, hin + (uint64_t)(k + 1) * W4, g == 0 && (uint32_t)k + 1 <= m);
        cp_async_commit();
    }
    // lane 0's input for step 0 (column 1); cc = symbol code of this lane's
    // column in the coming step (known one step ahead, so the step's score
    // loads do not wait on its shuffles)
    V iM, iGB, iGA;
    uint32_t cc;
    cp_async_wait<FIFO - 1>();
    Cell4<V>::read(s_fifo, iM, iGB, iGA, cc);
    const int32_t* tab = s_table;
    const char* tbytes = reinterpret_cast<const char*>(tab);
    [[maybe_unused]] const uint32_t kemax = (uint32_t)a.KE - 1u;
    // step-major trace (see nw.cu trace_chunk16): this band's (m + 31) steps
    // x 32 lanes x RR bytes; the lane's bytes of step s at + s * 32 RR + g RR
    uint8_t* tptr = T + (uint64_t)band * (m + 31) * BAND + (uint32_t)g * RR;
    int4* hout = hin + W4;           // lane 31: hand-off column j (from 1)

    auto step = [&](uint32_t s, auto chk) {
        constexpr bool CHK = decltype(chk)::value;
        const uint32_t j = s - (uint32_t)g + 1;  // 1..m when active
        [[maybe_unused]] int4 pq[PROF ? RR / 4 : 1];
        [[maybe_unused]] int cb4 = 0;
        if constexpr (PROF) {  // this step's scores, first: the address is known
            // (clamped: lanes outside their columns carry stale codes)
            const int4* pp = s_prof + (int)min(cc, kemax) * (RR / 4) * 32 + g;
#pragma unroll
            for (int q = 0; q < RR / 4; ++q) pq[q] = pp[q * 32];
        } else {
            cb4 = (int)cc * 4;
        }
        const V rM = shfl_up1(sM), rGB = shfl_up1(sGB), rGA = shfl_up1(sGA);
        const uint32_t nc = __shfl_up_sync(FULL, cc, 1);  // next step's code (lanes 1..31)
        // lane 0's input for the next step: column s+2 from the FIFO (every
        // lane reads the slot); then lane 0 refills the slot column s+1 came
        // from with column s+1+FIFO
        V xM, xGB, xGA;
        uint32_t xC;
        {
            cp_async_wait<FIFO - 2>();
            Cell4<V>::read(s_fifo + ((s + 1) % FIFO) * W4, xM, xGB, xGA, xC);
            fifo_fetch<V>(s_fifo + (s % FIFO) * W4, hin + (uint64_t)(s + 1 + FIFO) * W4,
                          g == 0 && s + 1 + FIFO <= m);
            cp_async_commit();
        }
        const uint32_t ccur = cc;
        cc = g == 0 ? xC : nc;
        uint32_t tw[RR / 4];
        if (!CHK || j - 1 < m) {
            V uM = g == 0 ? iM : rM;
            V uGB = g == 0 ? iGB : rGB;
            V uGA = g == 0 ? iGA : rGA;
            V dmax = pmax;
            pmax = vmax3(uM, add_fma(uGB, O, a.one), uGA);
            uint32_t tv[4];
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                int32_t sc;
                if constexpr (PROF) {
                    const int4& w4 = pq[r >> 2];
                    sc = (r & 3) == 0 ? w4.x : (r & 3) == 1 ? w4.y : (r & 3) == 2 ? w4.z : w4.w;
                } else {
                    sc = *reinterpret_cast<const int32_t*>(tbytes + add_fma(rowoff[r], cb4, a.one));
                }
                const V mo = add_fma(dmax, (V)sc, a.one);                            // M + O
                dmax = vmax3(LM[r], LGB[r], LGA[r]);                                 // old row r, + O
                const V gao = add_fma(vmax3(LM[r], LGB[r], add_fma(LGA[r], NO, a.one)), O, a.one);
                const V gbraw = vmax3(uM, uGB, uGA);  // the row chain (no extend: shifted domain)
                // trace byte: low bytes are the tags alone (256 scale)
                tv[r & 3] = (uint32_t)imad_u(lo32(gao), sixteen, imad_u(lo32(gbraw), four, lo32(mo)));
                if ((r & 3) == 3) tw[r >> 2] = gather_lo(tv[0], tv[1], tv[2], tv[3]);
                LM[r] = retag256(mo, keep, tag2);
                const V lgb = retag256(gbraw, keep, tag1);
                LGB[r] = add_fma(lgb, O, a.one);
                LGA[r] = retag256(gao, keep, 0u);
                uM = LM[r];
                uGB = lgb;
                uGA = LGA[r];
            }
            sM = uM;
            sGB = uGB;
            sGA = uGA;
            if (g == 31) Cell4<V>::store(hout, uM, uGB, uGA, ccur);
            hout += W4;
        }
        // the step's trace bytes, coalesced (32 x RR contiguous bytes; lanes
        // outside their columns store don't-care bytes no traceback reads)
        if constexpr (RR == 16) *reinterpret_cast<uint4*>(tptr) = make_uint4(tw[0], tw[1], tw[2], tw[3]);
        else if constexpr (RR == 8) *reinterpret_cast<uint2*>(tptr) = make_uint2(tw[0], tw[1]);
        else if constexpr (RR == 12) {
            reinterpret_cast<uint32_t*>(tptr)[0] = tw[0];
            reinterpret_cast<uint32_t*>(tptr)[1] = tw[1];
            reinterpret_cast<uint32_t*>(tptr)[2] = tw[2];
        }
        else *reinterpret_cast<uint32_t*>(tptr) = tw[0];
        tptr += 32 * RR;
        iM = xM;
        iGB = xGB;
        iGA = xGA;
    };
    const uint32_t steps = m + 31;
    uint32_t s = 0;
    for (; s < min(31u, steps); ++s) step(s, std::true_type{});
    const uint32_t s_end = m >= 1 ? m : 0;  // steps 31 .. m-1: every lane inside 1..m
#pragma unroll 1
    for (; s < s_end; ++s) step(s, std::false_type{});
    for (; s < steps; ++s) step(s, std::true_type{});
    // final state at (n, m) (pairwise.cpp:374-375): the lane owning row n
    if (n >= i0 && n < i0 + RR) {
        V fM = LM[0], fGB = LGB[0], fGA = LGA[0];
#pragma unroll
        for (int r = 1; r < RR; ++r)
            if (i0 + r == n) {
                fM = LM[r];
                fGB = LGB[r];
                fGA = LGA[r];
            }
        const V fin = vmax3(fM, fGB, fGA) - O;
        a.res[job.slot].score = (int64_t)(fin >> 8) + (int64_t)(n + m) * (a.E / 256);  // back from the shifted domain
        a.res[job.slot].final_tag = (uint32_t)(fin & 3);
    }
}

template <class V, bool PROF>
__global__ void __launch_bounds__(SEQ_WARPS * 32, sizeof(V) == 4 ? DM_NW_SEQ_MINB : 1) nw_seq_kernel(const SeqArgs a) {
    extern __shared__ __align__(16) int32_t s_dyn[];  // PROF: per-warp profiles; TAB: the table
    __shared__ uint8_t s_lut[128], s_plut[128];
    __shared__ int4 s_fifo_all[SEQ_WARPS][FIFO * 2];
    const int g = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    if constexpr (!PROF)
        for (int x = threadIdx.x; x < a.K * a.Kp; x += blockDim.x) s_dyn[x] = a.table[x];
    for (int x = threadIdx.x; x < 128; x += blockDim.x) {
        s_lut[x] = a.lut[x];
        if (PROF) s_plut[x] = a.plut[x];
    }
    __syncthreads();
    int4* s_prof = PROF ? reinterpret_cast<int4*>(s_dyn) + (size_t)w * a.KE * 4 * 32 : nullptr;
    const uint32_t keep = ~(uint32_t)(a.one * 255);
    const uint32_t four = (uint32_t)a.one * 4u, sixteen = four * four;
    int4* hin = a.hrow + (uint64_t)(blockIdx.x * SEQ_WARPS + w) * a.hstride;
    const V NEG = neg_inf256<V>();
    const V O = (V)a.O;
    for (;;) {
        uint32_t jid = 0;
        if (g == 0) jid = atomicAdd(a.counter, 1u);
        jid = __shfl_sync(FULL, jid, 0);
        if (jid >= a.njobs) break;
        const NwJob job = a.jobs[jid];
        // row 0 (pairwise.cpp:322-330) as the input of band 0: PM = -inf|2 + O,
        // GB = -inf|1, PGA = open + j*extend + O, and b's symbol codes
        const uint8_t* B = a.chars + job.b_off;
        for (uint32_t j = g; j <= job.m; j += 32) {
            const uint32_t ch = j ? (uint32_t)B[j - 1] & 127u : 0u;
            Cell4<V>::store(hin + (uint64_t)j * Cell4<V>::words, (V)(NEG | 2) + O, (V)(NEG | 1), (V)a.O + O,
                            PROF ? s_plut[ch] : s_lut[ch]);
        }
        __syncwarp();
        const uint32_t nb = (job.n + BAND - 1) / BAND;
        for (uint32_t band = 0; band < nb; ++band) {
            const uint32_t left = job.n - band * BAND;
            const uint32_t rr = seq_tail_rr(left > BAND ? BAND : left);
            if (rr == 16)
                seq_band<V, PROF, 16>(a, job, band, hin, s_dyn, s_prof, s_plut, s_lut, s_fifo_all[w], keep,
                                      four, sixteen);
#ifndef DM_NW_SEQ_NO12
            else if (rr == 12)
                seq_band<V, PROF, 12>(a, job, band, hin, s_dyn, s_prof, s_plut, s_lut, s_fifo_all[w], keep,
                                      four, sixteen);
#endif
            else if (rr == 8)
                seq_band<V, PROF, 8>(a, job, band, hin, s_dyn, s_prof, s_plut, s_lut, s_fifo_all[w], keep,
                                      four, sixteen);
            else
                seq_band<V, PROF, 4>(a, job, band, hin, s_dyn, s_prof, s_plut, s_lut, s_fifo_all[w], keep,
                                      four, sixteen);
            __syncwarp();  // the band's row (lane 31's stores) before the next band reads it
        }
    }
}

}  // namespace nwk
}  // namespace dm
