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
#include "lev_chains.h"

namespace dm {
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

int wmax_for(int np) { return np == 2 ? WMax<2>::value : (np == 5 ? WMax<5>::value : WMax<8>::value); }

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
    // multi-pass mode (LONG kernels, patterns longer than one warp's rows):
    // pass `pass` covers pattern rows [pass * 1024 W, (pass + 1) * 1024 W);
    // hbuf + hoff[item] holds, per text column, the horizontal delta leaving
    // the previous pass's bottom row (2 bits: h_minus << 1 | h_plus), and is
    // overwritten in place with the one leaving this pass.
    uint8_t* hbuf;
    const uint64_t* hoff;
    uint32_t pass;
};

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
// feeds the carry), and the bit shifted out = hi(t * 2) as an IMAD.HI.
template <int W>
__device__ __forceinline__ uint32_t shl1(uint32_t (&v)[W], uint32_t cin, uint32_t two) {
    uint32_t t[W];
#pragma unroll
    for (int w = 0; w < W; ++w) t[w] = v[w];
    Chain<W>::add(v, t, t);
    v[0] = imad(t[0], two, cin);
    return __umulhi(t[W - 1], two);
}

// LONG: the multi-pass form for patterns longer than 32 lanes x W words
// (Myers' block formulation across passes: the same recurrence, with the
// horizontal delta between row blocks carried through global memory instead
// of a shuffle). One warp (G = 32) per job, checked columns only.
template <int NP, int W, bool LONG = false>
__global__ void __launch_bounds__(256, NP == 2 ? (W <= 16 ? 3 : 2) : 1) lev_kernel(const LevArgs a) {
    constexpr bool TAB = NP == 2;
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
        uint64_t blk0 = a.blk[item.pat];
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
                const uint32_t p0 = in ? __ldg(pp + (uint64_t)(gw >> 1) * 4 + (gw & 1)) : 0u;
                const uint32_t p1 = in ? __ldg(pp + (uint64_t)(gw >> 1) * 4 + 2 + (gw & 1)) : 0u;
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
                Chain<W>::add(S, X, Pv);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    Mh[w] = lop3<0xBA>(Pv[w], S[w], X[w]);  // (Pv & ~S) | X
                    // Ph = Mv | ~(S | Pv | Xv): Mv is a subset of Xv, so the two
                    // terms are disjoint and the OR is an add -> FMA pipe
                    Ph[w] = w == 0 ? lop3<0xF1>(Mv[w], S[w], T0) : imad(lop3<0x01>(S[w], Pv[w], Xv[w]), a.one, Mv[w]);
                }
                const uint32_t hpo = shl1<W>(Ph, hp, two);
                const uint32_t hmo = shl1<W>(Mh, hm, two);
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
                if constexpr (TAB) c = (__ldg(tw + (s >> 4)) >> ((s & 15u) * 2u)) & 3u;
                else c = (uint32_t)__ldg(tp + s);
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
            if constexpr (TAB) {
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
                if constexpr (TAB) {
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

template <int NP, int W, bool LONG = false>
void launch_one(const LevArgs& a, int sm_count, cudaStream_t st) {
    const size_t smem = NP == 2 ? (size_t)4 * W * 256 * sizeof(uint32_t) : 0;
    const int occ = occupancy((const void*)lev_kernel<NP, W, LONG>, 256, smem);
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
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(want, resident * kWaves));
    LevArgs b = a;
    b.max_pulls = (uint32_t)((tasks + grid * 8 - 1) / (grid * 8));
    lev_kernel<NP, W, LONG><<<(unsigned)grid, 256, smem, st>>>(b);
}

template <int NP, int W>
void dispatch_w(int w, const LevArgs& a, int sm, cudaStream_t st) {
    if constexpr (W <= WMax<NP>::value) {
        if (w == W) {
            launch_one<NP, W>(a, sm, st);
            return;
        }
        dispatch_w<NP, W + 1>(w, a, sm, st);
    } else {
        throw runtime_error("distance engine: unsupported word count");
    }
}

template <int NP, int W>
void warm_np() {
    if constexpr (W <= WMax<NP>::value) {
        cudaFuncAttributes fa;
        DM_CUDA(cudaFuncGetAttributes(&fa, lev_kernel<NP, W>));
        warm_np<NP, W + 1>();
    }
}

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

// Orient each job (shorter string = pattern), pick (G, R) and build the
// radix key (bucket << 32 | ~n) so one sort groups buckets and balances warps.
__global__ void plan_kernel(const uint32_t* __restrict__ ia, const uint32_t* __restrict__ ib,
                            const LevItem* __restrict__ in_items, uint64_t n,
                            const uint32_t* __restrict__ len, int lg_gpar, int wsel, int wmax,
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

// A planned batch: bucket-sorted items plus the host copy of the histogram.
struct LevPlan {
    LevItem* items = nullptr;
    uint32_t* counters = nullptr;
    unsigned int h[kBuckets];
    unsigned long long hc[2];
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
}

// Planner phase on `ctx`'s stream (scratch from ctx): orient, bucket, sort,
// read the histogram back (the one host sync of a batch) -- or, given the
// host offsets of identity pairs (2i, 2i+1), count it on the host and stay
// asynchronous.
void plan_batch(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia, const uint32_t* d_ib,
                const LevItem* d_in_items, uint64_t n, LevPlan& P, const uint64_t* pair_offs = nullptr) {
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
    plan_kernel<<<grid, 256, 0, st>>>(d_ia, d_ib, d_in_items, n, s->d_len, lg_gpar, wsel, wmax, it0, k0, i0,
                                      hist, cells);
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
int launch_plan(dm_ctx* ctx, const LevPlan& P, const dm_seqset* s, uint32_t* d_out, cudaStream_t st,
                cudaEvent_t after = nullptr) {
    uint64_t starts[kBuckets];
    int order[kBuckets], nb = 0;
    uint64_t start = 0;
    for (int b = 0; b < kBuckets; ++b) {
        starts[b] = start;
        start += P.h[b];
        if (P.h[b]) order[nb++] = b;
    }
    // the multi-pass bucket (largest work per job) is first in `order`:
    // it goes to the first side stream and syncs that stream once to size
    // its buffers (run_long)
    // largest per-task work first: lanes per pair x words per lane
    std::stable_sort(order, order + nb, [](int x, int y) { return ((x % 32) << (x / 32)) > ((y % 32) << (y / 32)); });
    const bool fork = nb > 1 || after != nullptr;
    int used[kLevSide], nused = 0;
    if (fork) {
        if (!ctx->lev_fork) {
            DM_CUDA(cudaEventCreateWithFlags(&ctx->lev_fork, cudaEventDisableTiming));
            for (int k = 0; k < kLevSide; ++k) {
                DM_CUDA(cudaStreamCreateWithFlags(&ctx->lev_side[k], cudaStreamNonBlocking));
                DM_CUDA(cudaEventCreateWithFlags(&ctx->lev_join[k], cudaEventDisableTiming));
            }
        }
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
            run_long(ctx, P.items + starts[b], P.h[b], s, d_out, fork ? ctx->lev_side[used[i % nused]] : st);
            continue;
        }
        LevArgs a{};
        a.items = P.items + starts[b];
        a.nitems = P.h[b];
        a.lgG = b / 32;
        a.codes = s->d_codes;
        a.off = s->d_off;
        a.len = s->d_len;
        a.blk = s->d_blk;
        a.planes = s->d_planes;
        a.out = d_out;
        a.counter = P.counters + b;
        a.one = 1u;
        launch_bucket(s->planes, b % 32, a, ctx->sm_count, fork ? ctx->lev_side[used[i % nused]] : st);
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
                 bool time_kernels) {
    if (n == 0) return;
    LevPlan P;
    plan_batch(ctx, s, d_ia, d_ib, d_in_items, n, P);
    cudaStream_t st = ctx->stream;
    if (time_kernels) DM_CUDA(cudaEventRecord(ctx->ev0, st));
    const int launches = launch_plan(ctx, P, s, d_out, st);
    if (time_kernels) DM_CUDA(cudaEventRecord(ctx->ev1, st));
    ctx->launches += launches;
    if (tot) {
        tot->cells += P.hc[0];
        tot->cells_exec += P.hc[1];
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

// Loads every kernel instance up front (lazy module loading would otherwise
// charge the first batch that hits a new bucket).
void lev_warm() {
    warm_np<2, 1>();
    warm_np<5, 1>();
    warm_np<8, 1>();
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
    const int launches = launch_plan(ctx, P, s, d_out, ctx->stream, planned);
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

}  // namespace dm
