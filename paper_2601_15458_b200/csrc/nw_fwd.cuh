// Gotoh NW forward pass (K5), included by nw.cu. See nw.cu for the tagged
// score encoding and the trace layout.
//
// Work decomposition: one alignment per CTA of NWW warps. The rows of a are
// cut into bands of 32*RR rows; warp w sweeps bands w, w+NWW, ... Inside a
// band the 32 lanes form a diagonal pipeline over the columns of b (lane g
// is on column s-g+1 at step s; the bottom row of lane g-1 arrives by three
// __shfl_up). Between bands, lane 31 of the band above streams its bottom
// row (M, GapB, GapA per column) through a shared-memory ring to lane 0 of
// the band below, so all bands of one alignment run concurrently, a few
// columns apart, instead of one after another: the latency of a 2400 x 2400
// merge drops from 5 sequential passes to ~1. Flow control is two monotonic
// sequence counters per ring (published / consumed), checked once per
// CHUNK columns. NWW = 1 is the plain warp-per-alignment kernel for
// single-band alignments. With more bands than warps, warp w sweeps bands
// w, w+NWW, ...; the row from the last band of a round to the first band of
// the next (ring 0) cannot be a bounded ring (band NWW starts only when band
// 0 has finished the whole width, which a 128-column ring would stall
// through back-pressure), so it goes through a full-width row in global
// memory: the producer never waits, the consumer waits on the same
// publication counter and reads L2 (ld.cg: the row is rewritten in place
// by the next round, never read from a stale L1 line).
//
// State convention (fewer ALU ops per cell, the kernel is ALU-bound): a row
// keeps PM = M + O4, PGB = GapB + O4, PGA = GapA + O4 (tags survive: O4 is a
// multiple of 4), all in the (i+j)*extend-shifted domain of nw_seq.cuh
// (X'' = X - (i+j)*E4: the gap chains lose their extend adds, the score table
// holds s - 2*E4, the final score adds (n+m)*E4 back). Then per cell
//   diag   = max3(PM, PGB, PGA) of the row above, previous column  (= max + O4)
//   M + O4 = diag + s - 2 E4                             -> retag 2 = new PM
//   GA + O4 = max3(PM, PGB, PGA - O4) (own row, prev col) + O4 -> & ~3 = new PGA
//   GB     = max3(PM, GB, PGA) (row above, this column)  -> retag 1; +O4 = new PGB
// i.e. 6 ALU (3 max3, 3 retags) + 5 FMA (adds incl. the score-table address),
// where the max3-of-sums form needed 4 ALU VIADDMNMX + 3 retags + 1 max3 +
// an ALU address add. The vertical-gap chain down the 16 rows of a lane is
// max3 -> retag (9 cycles a row; 13 with the extend add of the unshifted
// form, 30 with two dependent VIADDMNMX). Lanes and the band ring pass (PM,
// GB, PGA) of their bottom row.
#pragma once

#include <type_traits>

namespace dm {
namespace nwk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int RR = 16;           // rows per lane
constexpr int BAND = 32 * RR;    // rows per band (one warp)
constexpr int RING = 128;        // columns buffered between two bands
constexpr int CHUNK = 16;        // flow-control granularity (columns)

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
__device__ __forceinline__ V shfl_up1(V v) {
    if constexpr (sizeof(V) == 4) {
        return __shfl_up_sync(FULL, v, 1);
    } else {
        return (V)__shfl_up_sync(FULL, (long long)v, 1);
    }
}

// x + y on the FMA pipe (the forward pass is ALU-bound): `one` is an opaque 1
__device__ __forceinline__ int32_t add_fma(int32_t x, int32_t y, int32_t one) {
    int32_t d;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(one), "r"(y));
    return d;
}
__device__ __forceinline__ int64_t add_fma(int64_t x, int64_t y, int32_t) { return x + y; }

__device__ __forceinline__ int32_t ldcg(const int32_t* p) { return __ldcg(p); }
__device__ __forceinline__ int64_t ldcg(const int64_t* p) { return (int64_t)__ldcg(reinterpret_cast<const long long*>(p)); }

// x * y on the FMA pipe (y opaque: no strength reduction to a shift)
__device__ __forceinline__ uint32_t umul(uint32_t x, uint32_t y) {
    uint32_t d;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    return d;
}

// low bytes of four values -> one word (byte k = low byte of value k)
__device__ __forceinline__ uint32_t gather_lo(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    const uint32_t ab = __byte_perm(a, b, 0x0040);
    const uint32_t cd = __byte_perm(c, d, 0x0040);
    return __byte_perm(ab, cd, 0x5410);
}

template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t x, uint32_t y, uint32_t z) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(x), "r"(y), "r"(z), "n"(LUT));
    return d;
}

// (x & ~3) | tag as ONE LOP3: `keep` (= ~3) and `tag` live in registers
// (opaque to ptxas, which would otherwise split the immediates over two ops)
__device__ __forceinline__ int32_t retag(int32_t x, uint32_t keep, uint32_t tag) {
    return (int32_t)lop3<0xEA>((uint32_t)x, keep, tag);
}
__device__ __forceinline__ int64_t retag(int64_t x, uint32_t, uint32_t tag) { return (x & ~(int64_t)3) | (int64_t)tag; }

// bits of x where mask is set, bits of y elsewhere (one LOP3)
__device__ __forceinline__ uint32_t bitsel(uint32_t x, uint32_t y, uint32_t mask) { return lop3<0xE4>(x, y, mask); }

struct FwdArgs {
    const uint8_t* chars;
    const NwJob* jobs;
    uint32_t njobs;
    const uint8_t* lut;
    const int32_t* table;  // 4*score, K x Kp
    int K, Kp;
    int64_t O4, E4;
    uint8_t* trace;
    NwRes* res;
    uint32_t* counter;
    int32_t one;  // == 1 (opaque to ptxas)
    // alignments with more bands than warps: the row passed from band NWW-1
    // of one round to band NWW of the next (ring 0) goes through this
    // per-CTA global row (wrap_stride V per CTA, columns 0..m) instead
    void* wrap;
    uint64_t wrap_stride;
};

template <class V, int NWW>
struct FwdSmem {
    V ring[NWW > 1 ? NWW : 1][RING][3];
    volatile uint32_t pub[NWW], con[NWW];
    uint32_t jid;
    uint8_t lut[128];
};

template <class V, int NWW>
__global__ void __launch_bounds__(NWW * 32) nw_fwd_kernel(const FwdArgs a) {
    extern __shared__ int32_t s_table[];
    __shared__ FwdSmem<V, NWW> sm;
    for (int x = threadIdx.x; x < a.K * a.Kp; x += blockDim.x) s_table[x] = a.table[x];
    for (int x = threadIdx.x; x < 128; x += blockDim.x) sm.lut[x] = a.lut[x];
    const int g = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const V NEG = neg_inf<V>();
    const V O4 = (V)a.O4;
    const char* tbytes = reinterpret_cast<const char*>(s_table);
    // opaque ~3 / tag constants (from the runtime 1) for the one-LOP3 retags
    const uint32_t tag1 = (uint32_t)a.one, tag2 = tag1 + tag1, keep = ~(tag2 + tag1);
    const uint32_t four = tag2 + tag2, sixteen = four * four;
    const V NO4 = -O4;
    for (;;) {
        __syncthreads();  // previous job fully done; table/lut loaded
        if (threadIdx.x == 0) sm.jid = atomicAdd(a.counter, 1u);
        if (threadIdx.x < NWW) {
            sm.pub[threadIdx.x] = 0;
            sm.con[threadIdx.x] = 0;
        }
        __syncthreads();
        const uint32_t jid = sm.jid;
        if (jid >= a.njobs) break;
        const NwJob job = a.jobs[jid];
        const uint32_t n = job.n, m = job.m;

        const uint8_t* A = a.chars + job.a_off;
        const uint8_t* B = a.chars + job.b_off;
        const uint32_t pa = (n + 15) & ~15u;
        uint8_t* T = a.trace + job.t_off;
        const uint32_t nbands = (n + BAND - 1) / BAND;
        for (uint32_t band = w; band < nbands; band += NWW) {
            const uint32_t i0 = band * BAND + (uint32_t)g * RR + 1;
            int rowoff[RR];  // byte offset of the score-table row of a[i]
            V LM[RR], LGB[RR], LGA[RR];  // PM, PGB, PGA (offset by O4, see above)
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const uint32_t i = i0 + r;
                rowoff[r] = (i <= n ? (int)sm.lut[A[i - 1] & 127] : 0) * a.Kp * 4;
                LM[r] = (V)(NEG | 2) + O4;
                LGA[r] = NEG + O4;
                LGB[r] = (V)(a.O4 | 1) + O4;  // column 0: GB = open + i*extend
            }
            // row i0-1 at column 0: the first row's diagonal at column 1
            // (as the max over its three states: all the M recurrence needs), + O4
            V pmax = (i0 == 1 ? (V)2 /* M[0][0] = 0 */ : (V)(a.O4 | 1)) + O4;
            // ring in (from band-1) and out (to band+1); sequence = gen*(m+1)+j
            const int rin = (int)(band % NWW), rout = (int)((band + 1) % NWW);
            const uint32_t seq_in = (band / NWW) * (m + 1), seq_out = ((band + 1) / NWW) * (m + 1);
            const bool has_in = NWW > 1 && band > 0;
            const bool has_out = NWW > 1 && band + 1 < nbands;
            V* wrapbuf = NWW > 1 ? reinterpret_cast<V*>(a.wrap) + (uint64_t)blockIdx.x * a.wrap_stride : nullptr;
            V sM = 0, sGB = 0, sGA = 0;
            // b's residue for the lane's next column, loaded one step ahead
            // (the global load's latency was the top stall of the step)
            uint32_t bnext = (g == 0 && m > 0) ? (uint32_t)B[0] : 0u;
            // One column step of the band's lane pipeline. CHK: generic step
            // (pipeline fill/drain: lanes may be outside 1..m; ring flow
            // control decided from s, per step). Steady steps (every lane
            // inside, s in whole 16-column chunks) drop the range checks and
            // all flow control: the steady loop does it once per chunk.
            auto step = [&](uint32_t s, auto chk) {
                constexpr bool CHK = decltype(chk)::value;
                const V rM = shfl_up1(sM), rGB = shfl_up1(sGB), rGA = shfl_up1(sGA);
                if constexpr (NWW > 1 && CHK) {
                    // consumer side (lane 0 reads column s+1 this step)
                    if (has_in && (s % CHUNK) == 0 && s < m) {
                        if (g == 0) {
                            const uint32_t need = seq_in + min(s + CHUNK, m);
                            while (sm.pub[rin] < need) {
                            }
                        }
                        __syncwarp();
                    }
                    // producer side (lane 31 writes column s-30 this step)
                    if (has_out && rout != 0 && s >= 31 && ((s - 31) % CHUNK) == 0 && s - 31 < m) {
                        if (g == 31) {
                            const uint32_t jj = s - 30;  // first column of the chunk
                            const uint32_t last = seq_out + min(jj + CHUNK - 1, m);
                            while (sm.con[rout] + RING < last + 1) {
                            }
                        }
                        __syncwarp();
                    }
                }
                const uint32_t j = s - (uint32_t)g + 1;  // 1..m when active
                const uint32_t bcur = bnext;
                bnext = j < m ? (uint32_t)B[j] : 0u;  // column j + 1 next step
                if (!CHK || j - 1 < m) {
                    // lane 0's input row (band 0: row 0, pairwise.cpp:322-330;
                    // else the band above via the ring), read at lane 0's
                    // column s+1 by every lane (one broadcast, no divergence)
                    V iM, iGB, iGA;  // (PM, GB, PGA) of the row above lane 0
                    if (band == 0) {
                        iM = (V)(NEG | 2) + O4;
                        iGB = (V)(NEG | 1);
                        iGA = (V)a.O4 + O4;  // row 0 in the shifted domain (nw_seq.cuh)
                    } else if (NWW > 1 && rin == 0) {
                        const V* e = wrapbuf + (uint64_t)(s + 1) * 3;
                        iM = ldcg(e);
                        iGB = ldcg(e + 1);
                        iGA = ldcg(e + 2);
                    } else {
                        const V* e = sm.ring[rin][(seq_in + s + 1) % RING];
                        iM = e[0];
                        iGB = e[1];
                        iGA = e[2];
                    }
                    V uM = g == 0 ? iM : rM;
                    V uGB = g == 0 ? iGB : rGB;
                    V uGA = g == 0 ? iGA : rGA;
                    // diagonal of row r = old (previous column) values of row r-1,
                    // pre-reduced to their max before row r-1 is overwritten, so
                    // every state updates in place (no register rotation)
                    V dmax = pmax;
                    pmax = vmax3(uM, add_fma(uGB, O4, a.one), uGA);
                    const int cb4 = (int)sm.lut[bcur & 127] * 4;
                    uint32_t tw[RR / 4];
                    uint32_t tm[4], tgb[4], tga[4];
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        const int32_t sc = *reinterpret_cast<const int32_t*>(tbytes + add_fma(rowoff[r], cb4, a.one));
                        const V mo = add_fma(dmax, (V)sc, a.one);                  // M + O4
                        dmax = vmax3(LM[r], LGB[r], LGA[r]);                       // old row r, + O4
                        const V gao = add_fma(vmax3(LM[r], LGB[r], add_fma(LGA[r], NO4, a.one)), O4, a.one);
                        const V gbraw = vmax3(uM, uGB, uGA);   // the row chain (shifted domain: no extend)
                        tm[r & 3] = (uint32_t)mo;
                        tgb[r & 3] = (uint32_t)gbraw;
                        tga[r & 3] = (uint32_t)gao;
                        if ((r & 3) == 3) {  // four rows of codes -> one trace word
                            const uint32_t wm = gather_lo(tm[0], tm[1], tm[2], tm[3]);
                            const uint32_t wb = gather_lo(tgb[0], tgb[1], tgb[2], tgb[3]);
                            const uint32_t wa = gather_lo(tga[0], tga[1], tga[2], tga[3]);
                            // byte = tagM | tagGB << 2 | tagGA << 4 (bits 6-7 are
                            // don't-care: the traceback masks every field); the
                            // shifts as multiplies by opaque 4 / 16 (FMA pipe)
                            tw[r >> 2] = bitsel(bitsel(wm, umul(wb, four), 0x03030303u), umul(wa, sixteen), 0x0F0F0F0Fu);
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
                    if (i0 <= n)
                        *reinterpret_cast<uint4*>(T + (uint64_t)(j - 1) * pa + (i0 - 1)) =
                            make_uint4(tw[0], tw[1], tw[2], tw[3]);
                    if constexpr (NWW > 1) {
                        if (has_out && g == 31) {
                            V* e = rout == 0 ? wrapbuf + (uint64_t)j * 3 : sm.ring[rout][(seq_out + j) % RING];
                            e[0] = uM;
                            e[1] = uGB;
                            e[2] = uGA;
                            if (CHK && ((j % CHUNK) == 0 || j == m)) {
                                __threadfence_block();
                                sm.pub[rout] = seq_out + j;
                            }
                        }
                        if (CHK && has_in && g == 0 && ((j % CHUNK) == 0 || j == m)) {
                            __threadfence_block();  // ring reads complete before the slot is released
                            sm.con[rin] = seq_in + j;
                        }
                    }
                }
            };
            const uint32_t steps = m + 31;
            uint32_t s = 0;
            for (; s < min(32u, steps); ++s) step(s, std::true_type{});
            // steady state: s in [32, s_end), whole chunks of CHUNK columns;
            // flow control once per chunk, around the chunk:
            //  - consumer (lane 0 reads columns s+1 .. s+16): wait until the
            //    band above published them; release them after the chunk;
            //  - producer (lane 31 writes columns s-30 .. s-15): wait for ring
            //    space through column s (this chunk plus the next 15 writes,
            //    which the drain steps' own checks do not cover); publish
            //    through s-15 after the chunk.
            // The producer then runs 31..143 columns ahead of its consumer.
            if (m > 32) {
                const uint32_t s_end = 32 + ((m - 32) & ~(uint32_t)(CHUNK - 1));
#pragma unroll 1
                for (; s < s_end; s += CHUNK) {
                    if constexpr (NWW > 1) {
                        if (has_in) {
                            if (g == 0) {
                                const uint32_t need = seq_in + min(s + CHUNK, m);
                                while (sm.pub[rin] < need) {
                                }
                            }
                            __syncwarp();
                        }
                        if (has_out && rout != 0) {
                            if (g == 31) {
                                const uint32_t last = seq_out + min(s, m);
                                while (sm.con[rout] + RING < last + 1) {
                                }
                            }
                            __syncwarp();
                        }
                    }
                    // not unrolled: one step is ~300 instructions, a chunk of
                    // them would not fit the instruction cache
#pragma unroll 1
                    for (uint32_t q = 0; q < CHUNK; ++q) step(s + q, std::false_type{});
                    if constexpr (NWW > 1) {
                        if (has_out && g == 31) {
                            __threadfence_block();
                            sm.pub[rout] = seq_out + (s + CHUNK - 1 - 30);
                        }
                        if (has_in && g == 0) {
                            __threadfence_block();  // ring reads complete before the slots are released
                            sm.con[rin] = seq_in + s + CHUNK;
                        }
                    }
                }
            }
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
                const V fin = vmax3(fM, fGB, fGA) - O4;
                a.res[job.slot].score = (int64_t)(fin >> 2) + (int64_t)(n + m) * (a.E4 / 4);
                a.res[job.slot].final_tag = (uint32_t)(fin & 3);
            }
            __syncwarp();
        }
    }
}

}  // namespace nwk
}  // namespace dm
