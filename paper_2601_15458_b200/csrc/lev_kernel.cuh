// Distance-engine kernel K1 (see lev.cu for the design): the bit-parallel
// Myers/Hyyro lane pipeline, its launch and bucket dispatch. Shared by lev.cu
// (bit-plane pattern source: resident sequence sets) and lev_src.cu (2-bit
// code and raw A/C/G/T byte sources: host-planned streamed chunks).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "dm_internal.h"
#include "lev_chains.h"

namespace dm {

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
    uint32_t one;        // == 1; opaque to ptxas so the carry chains stay on the FMA pipe
    uint32_t max_pulls;  // task pulls per warp before its block retires (see launch_one)
    uint32_t waves;      // host only: grid in waves of resident blocks (0: DM_LEV_WAVES, default 4)
    // multi-pass mode (LONG kernels, patterns longer than one warp's rows):
    // pass `pass` covers pattern rows [pass * 1024 W, (pass + 1) * 1024 W);
    // hbuf + hoff[item] holds, per text column, the horizontal delta leaving
    // the previous pass's bottom row (2 bits: h_minus << 1 | h_plus), and is
    // overwritten in place with the one leaving this pass.
    uint8_t* hbuf;
    const uint64_t* hoff;
    uint32_t pass;
};

namespace {

constexpr unsigned FULL = 0xffffffffu;

// Words (32 rows each) per lane: the register budget is ~(NP + 6) * W.
template <int NP>
struct WMax;
template <>
struct WMax<2> { static constexpr int value = 24; };
template <>
struct WMax<5> { static constexpr int value = 10; };
template <>
struct WMax<8> { static constexpr int value = 6; };

inline int wmax_for(int np) { return np == 2 ? WMax<2>::value : (np == 5 ? WMax<5>::value : WMax<8>::value); }



// One lane = W consecutive 32-bit words of the pattern, handled as ONE
// multi-precision bit-vector (Myers' recurrence needs its addition and
// shifts to carry across the whole vector; inside a lane the carry flag does
// it, between lanes the horizontal delta h_in/h_out does, as in Myers'
// block formulation). Per word and column: NP IMAD (match mask from the
// bit-planes: P ^ ~m == P * (1 + 2t) + t with t = ~m in {0,-1}), 8 LOP3 and
// 3 carry-chained adds (add + two 1-bit shifts).
// FMA-pipe integer helper: with an opaque multiplier (`two`, `one` derive
// from a runtime 1) ptxas keeps IMAD instead of strength-reducing to ALU ops.
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

// v = (v << 1) | cin over W words; returns the bit shifted out. The shift
// is v + v as ONE carry-chained add over the words (one IADD3.X per word);
// the carry-in lands in the free bit 0 of word 0. Measured on the bare
// per-word mix (tools/ubench/mix.cu): 61 TCUPS with both shifts as add
// chains vs 54 with IMAD.WIDE + IMAD per word on the FMA pipe — fewer
// instructions issued beats moving work off the ALU pipe here.
// Two of its ops go to the FMA pipe (the kernel is ALU-bound, the FMA pipe
// has room): word 0 = t0 * 2 + cin as an IMAD (the chain's own word 0 only
// feeds the carry), the bit shifted out = hi(t * 2) as an IMAD.HI, and the
// top word's add (carry in, none out) as an IMAD.X (Chain::addm).
template <int W>
__device__ __forceinline__ uint32_t shl1(uint32_t (&v)[W], uint32_t cin, uint32_t two, uint32_t one) {
    uint32_t t[W];
#pragma unroll
    for (int w = 0; w < W; ++w) t[w] = v[w];
    Chain<W>::addm(v, t, t, one);
    v[0] = imad(t[0], two, cin);
    return __umulhi(t[W - 1], two);
}

// LONG: the multi-pass form for patterns longer than 32 lanes x W words
// (Myers' block formulation across passes: the same recurrence, with the
// horizontal delta between row blocks carried through global memory instead
// of a shuffle). One warp (G = 32) per job, checked columns only.
// Where a job's residues come from. kSrcPlanes: the sequence set's bit-plane
// profiles (patterns) and dense codes (texts) -- resident sets, any alphabet.
// NP == 2 only: kSrcCodes, the 2-bit code layout alone (the pattern's match
// masks are split out of the codes at job start); kSrcRaw, the caller's
// A/C/G/T bytes as uploaded (code = ((c >> 1) ^ (c >> 2)) & 3, the same
// A0 C1 G2 T3 map as host_pack.cpp). The last two need no device-side
// preparation of a streamed chunk: its kernels start when its bytes land.
enum : int { kSrcPlanes = 0, kSrcCodes = kLevSrcCodes, kSrcRaw = kLevSrcRaw };

// Inverse perfect shuffle: even bits -> low half, odd bits -> high half.
__device__ __forceinline__ uint32_t unshuffle32(uint32_t x) {
    uint32_t t;
    t = (x ^ (x >> 1)) & 0x22222222u;
    x = x ^ t ^ (t << 1);
    t = (x ^ (x >> 2)) & 0x0C0C0C0Cu;
    x = x ^ t ^ (t << 2);
    t = (x ^ (x >> 4)) & 0x00F000F0u;
    x = x ^ t ^ (t << 4);
    t = (x ^ (x >> 8)) & 0x0000FF00u;
    x = x ^ t ^ (t << 8);
    return x;
}

// 2-bit codes of 16 residues (code k in bits 2k, 2k+1) from 16 A/C/G/T bytes at
// any alignment (the buffer is padded: the 5th aligned word may be read).
__device__ __forceinline__ uint32_t raw16_codes(const uint8_t* p) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(p) & 3u) * 8u;
    uint32_t w[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) w[k] = __ldg(q + k);
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t g = __funnelshift_r(w[k], w[k + 1], sh);
        const uint32_t y = ((g >> 1) ^ (g >> 2)) & 0x03030303u;  // code per byte
        uint32_t z = y | (y >> 6);
        z = (z | (z >> 12)) & 0xffu;  // 4 codes in 8 bits
        r |= z << (8 * k);
    }
    return r;
}

// bit-planes of 32 rows from their 2-bit codes (x0: rows 0-15, x1: rows 16-31)
__device__ __forceinline__ void planes_of_codes(uint32_t x0, uint32_t x1, uint32_t& p0, uint32_t& p1) {
    const uint32_t u0 = unshuffle32(x0), u1 = unshuffle32(x1);
    p0 = __byte_perm(u0, u1, 0x5410);
    p1 = __byte_perm(u0, u1, 0x7632);
}

template <int NP, int W, bool LONG = false, int SRC = kSrcPlanes>
__global__ void __launch_bounds__(256, NP == 2 ? (W <= 16 ? 3 : 2) : 1) lev_kernel(const LevArgs a) {
    constexpr bool TAB = NP == 2;
    static_assert(SRC == kSrcPlanes || (TAB && !LONG), "code / raw sources: <= 4 symbols, one pass");
    constexpr bool RAW = SRC == kSrcRaw;
    extern __shared__ uint32_t s_tab[];  // TAB: 4 codes x W words x 256 threads
    // opaque constants (derived from the runtime 1) keep the bit arithmetic on IMAD
    const uint32_t two = a.one + a.one, four = two + two;
    const int lane = threadIdx.x & 31;
    const int lgG = a.lgG;
    const int G = 1 << lgG;
    const int g = lane & (G - 1);
    const int grp = lane >> lgG;
    const uint32_t gpw = 32u >> lgG;

    for (uint32_t pull = 0; pull < a.max_pulls; ++pull) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(a.counter, gpw);
        base = __shfl_sync(FULL, base, 0);
        if (base >= a.nitems) break;
        const uint32_t it = base + grp;
        const bool valid = it < a.nitems;
        LevItem item{0, 0, 0};
        if (valid) item = a.items[it];
        constexpr uint32_t kPassRows = 32u * W * 32u;
        uint32_t m = valid ? a.len[item.pat] : 0;
        const uint32_t n = valid ? a.len[item.txt] : 0;
        uint64_t blk0 = SRC == kSrcPlanes ? a.blk[item.pat] : 0;
        if constexpr (LONG) {
            const uint32_t done = a.pass * kPassRows;  // rows handled by earlier passes
            if (m <= done) continue;                   // whole warp: one job per warp
            m = min(m - done, kPassRows);
            blk0 += done / 64u;
        }
        const uint32_t nwords = (m + 31) >> 5;

        // NP == 2 (<= 4 residue codes, DNA): the lane's match masks for all
        // four codes live in shared memory, [code][word][thread] so a warp's
        // 32 lanes always hit 32 distinct banks whatever codes they look up.
        // Otherwise the bit-planes stay in registers and Eq is rebuilt per
        // column with one IMAD per plane.
        constexpr int NPR = TAB ? 1 : NP;
        uint32_t P[NPR][W];
        uint32_t Pv[W], Mv[W];
        const uint32_t* pp = reinterpret_cast<const uint32_t*>(a.planes + blk0 * NP);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t gw = (uint32_t)g * W + w;  // global word index in the pattern
            if constexpr (TAB) {
                const bool in = valid && gw < nwords;
                uint32_t p0 = 0u, p1 = 0u;
                if constexpr (SRC == kSrcPlanes) {
                    p0 = in ? __ldg(pp + (uint64_t)(gw >> 1) * 4 + (gw & 1)) : 0u;
                    p1 = in ? __ldg(pp + (uint64_t)(gw >> 1) * 4 + 2 + (gw & 1)) : 0u;
                } else if (in) {
                    // rows past m in the last word are junk: rows only feed rows below
                    // them and the result masks them out
                    const uint8_t* pc = a.codes + a.off[item.pat];
                    uint32_t x0, x1;
                    if constexpr (RAW) {
                        x0 = raw16_codes(pc + 32u * gw);
                        x1 = raw16_codes(pc + 32u * gw + 16u);
                    } else {
                        const uint2 v = __ldg(reinterpret_cast<const uint2*>(pc) + gw);
                        x0 = v.x;
                        x1 = v.y;
                    }
                    planes_of_codes(x0, x1, p0, p1);
                }
                s_tab[(0 * W + w) * 256 + threadIdx.x] = ~p0 & ~p1;
                s_tab[(1 * W + w) * 256 + threadIdx.x] = p0 & ~p1;
                s_tab[(2 * W + w) * 256 + threadIdx.x] = ~p0 & p1;
                s_tab[(3 * W + w) * 256 + threadIdx.x] = p0 & p1;
            } else {
#pragma unroll
                for (int k = 0; k < NP; ++k)
                    P[k][w] = (valid && gw < nwords) ? __ldg(pp + (uint64_t)(gw >> 1) * (2 * NP) + 2 * k + (gw & 1)) : 0u;
            }
            Pv[w] = ~0u;
            Mv[w] = 0u;
        }
        const int first_row = g * W * 32;
        int partial = max(0, min((int)m - first_row, W * 32));

        uint32_t steps = valid ? n + (uint32_t)G - 1u : 0u;
        steps = __reduce_max_sync(FULL, steps);
        const uint8_t* tp = a.codes + a.off[item.txt];
        const bool lead = g == 0 && valid;  // lane reading the text
        [[maybe_unused]] uint8_t* hb = nullptr;
        if constexpr (LONG) hb = a.hbuf + a.hoff[it];
        const uint32_t leadmask = g == 0 ? 0xffffffffu : 0u;
        uint32_t word = 0;
        // One text column through the lane pipeline. CHK: some lane of the
        // warp may be outside its text (pipeline fill/drain, shorter texts of
        // other groups, the final column); the steady state skips the checks.
        // ownw: lane 0's own word for this column, code << 2 | 1 (h_in = +1)
        auto column = [&](uint32_t s, auto chk, uint32_t ownw) {
            constexpr bool CHK = decltype(chk)::value;
            // word = code << 2 | h_minus << 1 | h_plus; lane 0 synthesises its
            // own (text code, h_in = +1). Branch-free select on a mask.
            const uint32_t recv = __shfl_up_sync(FULL, word, 1, G);
            const uint32_t r = lop3<0xCA>(leadmask, ownw, recv);  // lead ? own word : recv
            const uint32_t c = r >> 2;
            uint32_t hm = (r >> 1) & 1u;
            uint32_t hp = r & 1u;
            const uint32_t j = s - (uint32_t)g;
            if (!CHK || j < n) {
                // t_k = bit_k(c) - 1 (0 or all-ones), s_k = 2 t_k + 1 (+1 / -1)
                [[maybe_unused]] uint32_t ts[NP], ss[NP];
                if constexpr (!TAB) {
#pragma unroll
                    for (int k = 0; k < NP; ++k) {
                        ts[k] = ((c >> k) & 1u) - 1u;
                        ss[k] = imad(ts[k], two, a.one);
                    }
                }
                // Myers step, rewritten so Xh is never materialised (7 LOP3 per
                // word): with E = Eq (| h_minus on row 0), X = E & Pv, S = X + Pv,
                //   Mh = Pv & Xh         = (Pv & ~S) | X
                //   Ph = Mv | ~(Xh | Pv) = Mv | ~(S | Pv | Xv (| h_minus))
                // (on Pv bits S^Pv = ~S; off Pv bits Xh = S | E; Mv bits force Ph).
                // LUT constants: lop3(a, b, c) truth table over (0xF0, 0xCC, 0xAA).
                uint32_t X[W], S[W], Ph[W], Mh[W], Xv[W], T0 = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    uint32_t e;
                    if constexpr (TAB) {
                        e = s_tab[(c * W + w) * 256 + threadIdx.x];
                    } else {
                        e = imad(P[0][w], ss[0], ts[0]);
#pragma unroll
                        for (int k = 1; k < NP; ++k) e &= imad(P[k][w], ss[k], ts[k]);
                    }
                    Xv[w] = e | Mv[w];
                    // row 0 of the lane: h_in = -1 enters as a carry
                    X[w] = w == 0 ? lop3<0xA8>(e, hm, Pv[w]) : (e & Pv[w]);  // (e | hm) & Pv
                    if (w == 0) T0 = lop3<0xFE>(Pv[w], Xv[w], hm);
                }
                Chain<W>::addm(S, X, Pv, a.one);  // top word on the FMA pipe (IMAD.X)
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    Mh[w] = lop3<0xBA>(Pv[w], S[w], X[w]);  // (Pv & ~S) | X
                    // Ph = Mv | ~(S | Pv | Xv): Mv is a subset of Xv, so the two
                    // terms are disjoint and the OR is an add -> FMA pipe
                    Ph[w] = w == 0 ? lop3<0xF1>(Mv[w], S[w], T0) : imad(lop3<0x01>(S[w], Pv[w], Xv[w]), a.one, Mv[w]);
                }
                const uint32_t hpo = shl1<W>(Ph, hp, two, a.one);
                const uint32_t hmo = shl1<W>(Mh, hm, two, a.one);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    Pv[w] = lop3<0xF1>(Mh[w], Xv[w], Ph[w]);  // Mh | ~(Xv | Ph)
                    Mv[w] = Ph[w] & Xv[w];
                }
                hp = hpo;
                hm = hmo;
                if (CHK && j == n - 1) {
                    int acc = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        const int lo = first_row + w * 32;
                        const int cnt = max(0, min((int)m - lo, 32));
                        const uint32_t rm = cnt >= 32 ? ~0u : ((1u << cnt) - 1u);
                        acc += __popc(Pv[w] & rm) - __popc(Mv[w] & rm);
                    }
                    partial = acc;
                }
            }
            word = imad(c, four, imad(hm, two, hp));
            if constexpr (LONG) {  // bottom lane: the delta leaving this pass, in place
                if (g == G - 1 && j < n) hb[j] = (uint8_t)(word & 3u);
            }
        };
        // steady state [s0, s1): every valid lane has 0 <= j < n - 1
        uint32_t nmin = __reduce_min_sync(FULL, valid ? n : 0xffffffffu);
        const uint32_t s1 = nmin == 0xffffffffu || nmin == 0 ? 0u : nmin - 1u;
        const uint32_t s0 = min((uint32_t)G - 1u, s1);
        // text codes: 2 bits per residue (16 per word) when TAB, else bytes (code_bytes())
        const uint32_t* tw = reinterpret_cast<const uint32_t*>(tp);
        auto code_at = [&](uint32_t s) -> uint32_t {  // as a lane-0 word (code << 2 | 1)
            uint32_t c = 0u;
            if (lead && s < n) {
                if constexpr (RAW) {
                    const uint32_t b = __ldg(tp + s);
                    c = ((b >> 1) ^ (b >> 2)) & 3u;
                } else if constexpr (TAB) {
                    c = (__ldg(tw + (s >> 4)) >> ((s & 15u) * 2u)) & 3u;
                } else {
                    c = (uint32_t)__ldg(tp + s);
                }
            }
            return imad(c, four, a.one);
        };
        uint32_t s = 0;
        if constexpr (LONG) {
            // lane 0's word: text code, h_in from the previous pass (+1 on the first)
            for (; s < steps; ++s) {
                uint32_t w0 = code_at(s);
                if (a.pass > 0 && lead && s < n) w0 = (w0 & ~3u) | hb[s];
                column(s, std::true_type{}, w0);
            }
        } else {
            for (; s < s0; ++s) column(s, std::true_type{}, code_at(s));
            if constexpr (TAB && !RAW) {
                // steady state, 16 columns per text word (2-bit codes), taken 4 at a
                // time from a register (the 4-column body is not unrolled further:
                // instruction cache)
                for (; s < s1 && (s & 15u); ++s) column(s, std::false_type{}, code_at(s));
                for (; s + 16 <= s1; s += 16) {
                    uint32_t w16 = lead ? __ldg(tw + (s >> 4)) : 0u;
    #pragma unroll 1
                    for (uint32_t q = 0; q < 16; q += 4) {
                        // word k = (code_k << 2) | 1, one or two ops each
                        column(s + q, std::false_type{}, lop3<0xEA>(w16 << 2, 0xcu, 1u));
                        column(s + q + 1, std::false_type{}, lop3<0xEA>(w16, 0xcu, 1u));
                        column(s + q + 2, std::false_type{}, lop3<0xEA>(w16 >> 2, 0xcu, 1u));
                        column(s + q + 3, std::false_type{}, lop3<0xEA>(w16 >> 4, 0xcu, 1u));
                        w16 >>= 8;
                    }
                }
            }
            // steady state, four columns per text load (4-aligned code runs)
            for (; s < s1 && (s & 3u); ++s) column(s, std::false_type{}, code_at(s));
            for (; s + 4 <= s1; s += 4) {
                if constexpr (RAW) {
                    // 4 A/C/G/T bytes (any alignment); code << 2 = ((b << 1) ^ b) & 0xc per byte
                    uint32_t u = 0u;
                    if (lead) {
                        const uintptr_t ad = reinterpret_cast<uintptr_t>(tp + s);
                        const uint32_t* q = reinterpret_cast<const uint32_t*>(ad & ~uintptr_t(3));
                        const uint32_t t4 = __funnelshift_r(__ldg(q), __ldg(q + 1), (uint32_t)(ad & 3u) * 8u);
                        u = t4 ^ (t4 << 1);
                    }
                    column(s, std::false_type{}, lop3<0xEA>(u, 0xcu, 1u));
                    column(s + 1, std::false_type{}, lop3<0xEA>(u >> 8, 0xcu, 1u));
                    column(s + 2, std::false_type{}, lop3<0xEA>(u >> 16, 0xcu, 1u));
                    column(s + 3, std::false_type{}, lop3<0xEA>(u >> 24, 0xcu, 1u));
                } else if constexpr (TAB) {
                    // 4 codes in bits 0..7 of t4; word k = (code_k << 2) | 1, one or two ops each
                    const uint32_t t4 = lead ? __ldg(tw + (s >> 4)) >> ((s & 12u) * 2u) : 0u;
                    column(s, std::false_type{}, lop3<0xEA>(t4 << 2, 0xcu, 1u));
                    column(s + 1, std::false_type{}, lop3<0xEA>(t4, 0xcu, 1u));
                    column(s + 2, std::false_type{}, lop3<0xEA>(t4 >> 2, 0xcu, 1u));
                    column(s + 3, std::false_type{}, lop3<0xEA>(t4 >> 4, 0xcu, 1u));
                } else {
                    const uint32_t t4 = lead ? __ldg(reinterpret_cast<const uint32_t*>(tp + s)) : 0u;
                    column(s, std::false_type{}, imad(t4 & 0xffu, four, a.one));
                    column(s + 1, std::false_type{}, imad(__byte_perm(t4, 0u, 0x4441u), four, a.one));
                    column(s + 2, std::false_type{}, imad(__byte_perm(t4, 0u, 0x4442u), four, a.one));
                    column(s + 3, std::false_type{}, imad(t4 >> 24, four, a.one));
                }
            }
            for (; s < s1; ++s) column(s, std::false_type{}, code_at(s));
            for (; s < steps; ++s) column(s, std::true_type{}, code_at(s));
        }
        for (int o = G >> 1; o > 0; o >>= 1) partial += __shfl_down_sync(FULL, partial, o, G);
        // D[m][n] = n + sum of the vertical deltas of every row block at column n
        if (valid && g == 0) {
            if (LONG && a.pass > 0) a.out[item.slot] += (uint32_t)partial;
            else a.out[item.slot] = n + (uint32_t)partial;
        }
    }
}

template <int NP, int W, bool LONG = false, int SRC = kSrcPlanes>
void launch_one(const LevArgs& a, int sm_count, cudaStream_t st) {
    const size_t smem = NP == 2 ? (size_t)4 * W * 256 * sizeof(uint32_t) : 0;
    const int occ = occupancy((const void*)lev_kernel<NP, W, LONG, SRC>, 256, smem);
    // Warps pull tasks (32/G jobs) from the counter; each retires after
    // max_pulls tasks, and the grid is sized for ~kWaves waves of resident
    // blocks, so blocks turn over during a launch: kernels on other streams
    // (the planners of streamed batches) get SM slots within a fraction of
    // a bucket instead of after it. grid * 8 warps * max_pulls >= tasks.
    static const uint64_t kWaves = [] {
        const char* e = std::getenv("DM_LEV_WAVES");
        return e ? (uint64_t)std::max(1, std::atoi(e)) : (uint64_t)4;
    }();
    const uint64_t tasks = ((uint64_t)a.nitems + (32u >> a.lgG) - 1) / (32u >> a.lgG);
    const uint64_t resident = (uint64_t)occ * sm_count;
    const uint64_t want = (tasks + 7) / 8;  // blocks if every warp pulled once
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(want, resident * (a.waves ? a.waves : kWaves)));
    LevArgs b = a;
    b.max_pulls = (uint32_t)((tasks + grid * 8 - 1) / (grid * 8));
    lev_kernel<NP, W, LONG, SRC><<<(unsigned)grid, 256, smem, st>>>(b);
}

template <int NP, int W, int SRC = kSrcPlanes>
void dispatch_w(int w, const LevArgs& a, int sm, cudaStream_t st) {
    if constexpr (W <= WMax<NP>::value) {
        if (w == W) {
            launch_one<NP, W, false, SRC>(a, sm, st);
            return;
        }
        dispatch_w<NP, W + 1, SRC>(w, a, sm, st);
    } else {
        throw runtime_error("distance engine: unsupported word count");
    }
}

template <int NP, int W, int SRC = kSrcPlanes>
void warm_np() {
    if constexpr (W <= WMax<NP>::value) {
        cudaFuncAttributes fa;
        DM_CUDA(cudaFuncGetAttributes(&fa, lev_kernel<NP, W, false, SRC>));
        warm_np<NP, W + 1, SRC>();
    }
}
}  // namespace
}  // namespace dm
