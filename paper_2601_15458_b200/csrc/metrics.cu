// Alignment quality metrics: divmsa::evaluate
// (metrics.cpp:84-169) with its helpers gap_percent (:16-27), p_score
// (:29-45), hamming_aligned (distance.cpp:50-57) and distortion_pair (:47-56).
//
// The seeded sampling stays on the host and is bit-identical to the
// reference (rows: sample_distinct(mt19937_64(combine_seed(seed, 1)), ...);
// pairs: sample_distinct(mt19937_64(combine_seed(seed, 2)), k(k-1)/2, ...),
// decoded by pair_from_index). The data-parallel work runs on the device:
//   * gap census over the whole N x W block (gap_count_kernel, HBM-bound);
//   * one warp per sampled row pair streams both rows 16 bytes per lane and
//     counts shared-residue columns, mismatches among them and differing
//     columns (SIMD byte compares; rows padded with '-' to 16 B, which is
//     neutral for all three counts) -> p_score and hamming;
//   * the Levenshtein distance of the pair's raw sequences through the
//     distance engine (K1).
// The doubles are then formed and summed on the host in pair order, exactly
// as metrics.cpp:146-166 does, so every field is bit-identical.
#include <algorithm>
#include <chrono>
#include <cstring>

#include "capi_guard.h"
#include "rng.h"

namespace dm {
namespace {

constexpr uint32_t GAP4 = 0x2d2d2d2du;  // kGapSymbol '-' in every byte (alphabet.hpp)

__device__ __forceinline__ uint32_t popc_bytes(uint32_t mask) { return __popc(mask) >> 3; }

__global__ void gap_count_kernel(const uint4* __restrict__ rows, uint64_t nvec,
                                 unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
        const uint4 v = rows[i];
        c += popc_bytes(__vcmpeq4(v.x, GAP4)) + popc_bytes(__vcmpeq4(v.y, GAP4)) +
             popc_bytes(__vcmpeq4(v.z, GAP4)) + popc_bytes(__vcmpeq4(v.w, GAP4));
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

struct PairCounts {
    uint32_t considered, mismatched, hamming, pad;
};

// One warp per pair of rows (pitch bytes, multiple of 16, '-' padded).
__global__ void row_pair_kernel(const uint8_t* __restrict__ rows, uint64_t pitch, const uint32_t* __restrict__ ra,
                                const uint32_t* __restrict__ rb, uint64_t npairs, PairCounts* __restrict__ out) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nvec = pitch / 16;
    for (uint64_t p = warp; p < npairs; p += nwarps) {
        const uint4* a = reinterpret_cast<const uint4*>(rows + (uint64_t)ra[p] * pitch);
        const uint4* b = reinterpret_cast<const uint4*>(rows + (uint64_t)rb[p] * pitch);
        uint32_t cons = 0, mism = 0, ham = 0;
        for (uint64_t v = lane; v < nvec; v += 32) {
            const uint4 x = a[v], y = b[v];
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t eq = __vcmpeq4(xs[k], ys[k]);
                const uint32_t res = ~(__vcmpeq4(xs[k], GAP4) | __vcmpeq4(ys[k], GAP4));  // both residues
                cons += popc_bytes(res);
                mism += popc_bytes(res & ~eq);
                ham += popc_bytes(~eq);
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            cons += __shfl_xor_sync(0xffffffffu, cons, o);
            mism += __shfl_xor_sync(0xffffffffu, mism, o);
            ham += __shfl_xor_sync(0xffffffffu, ham, o);
        }
        if (lane == 0) out[p] = PairCounts{cons, mism, ham, 0};
    }
}

// metrics.cpp:62-80: the t'th pair (i < j) of k rows in lexicographic order.
std::pair<uint32_t, uint32_t> pair_from_index(uint64_t t, uint64_t k) {
    const auto before = [k](uint64_t i) { return i * k - i * (i + 1) / 2; };
    uint64_t lo = 0, hi = k - 1;
    while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) / 2;
        if (before(mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    return {(uint32_t)lo, (uint32_t)(lo + 1 + (t - before(lo)))};
}

// Rows -> device, pitch rounded to 16 B and padded with '-'.
uint8_t* upload_rows(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, uint64_t* pitch_out) {
    const uint64_t pitch = std::max<uint64_t>(16, (width + 15) & ~uint64_t(15));
    uint8_t* d = (uint8_t*)ctx->rows_a.get(nrows * pitch);
    if (pitch != width) DM_CUDA(cudaMemsetAsync(d, '-', nrows * pitch, ctx->stream));
    if (width)
        DM_CUDA(cudaMemcpy2DAsync(d, pitch, rows, width, width, nrows, cudaMemcpyHostToDevice, ctx->stream));
    *pitch_out = pitch;
    return d;
}

uint64_t gap_count(dm_ctx* ctx, const uint8_t* d_rows, uint64_t nrows, uint64_t pitch, uint64_t width) {
    unsigned long long* d_c = ctx->counter.as<unsigned long long>(1);
    DM_CUDA(cudaMemsetAsync(d_c, 0, 8, ctx->stream));
    const uint64_t nvec = nrows * pitch / 16;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((nvec + 255) / 256, (uint64_t)ctx->sm_count * 8));
    gap_count_kernel<<<grid, 256, 0, ctx->stream>>>(reinterpret_cast<const uint4*>(d_rows), nvec, d_c);
    DM_CUDA(cudaGetLastError());
    ++ctx->launches;
    unsigned long long c = 0;
    DM_CUDA(cudaMemcpyAsync(&c, d_c, 8, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    return (uint64_t)c - nrows * (pitch - width);  // the '-' padding is not part of the block
}

// Counts of row pairs (ra[p], rb[p]) of a device row block.
std::vector<PairCounts> row_pairs(dm_ctx* ctx, const uint8_t* d_rows, uint64_t pitch, const std::vector<uint32_t>& ra,
                                  const std::vector<uint32_t>& rb) {
    const uint64_t n = ra.size();
    std::vector<PairCounts> out(n);
    if (!n) return out;
    uint32_t* d_idx = ctx->aux.as<uint32_t>(2 * n);
    PairCounts* d_out = (PairCounts*)ctx->out.get(n * sizeof(PairCounts));
    DM_CUDA(cudaMemcpyAsync(d_idx, ra.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_idx + n, rb.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16));
    row_pair_kernel<<<grid, 256, 0, ctx->stream>>>(d_rows, pitch, d_idx, d_idx + n, n, d_out);
    DM_CUDA(cudaGetLastError());
    ++ctx->launches;
    DM_CUDA(cudaMemcpyAsync(out.data(), d_out, n * sizeof(PairCounts), cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
}

}  // namespace

void evaluate(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, const uint32_t* row_to_sequence,
              const char* raw, const uint64_t* raw_offsets, uint32_t nraw, uint64_t sample_size, uint64_t pair_budget,
              uint64_t seed, dm_metrics* rep) {
    if (nrows == 0) throw invalid_argument("cannot evaluate an empty alignment");  // metrics.cpp:87-89
    const auto t0 = std::chrono::steady_clock::now();
    std::memset(rep, 0, sizeof(*rep));
    rep->width = width;
    rep->seed = seed;
    for (uint64_t r = 0; r < nrows; ++r)
        if (row_to_sequence[r] >= nraw) throw invalid_argument("row_to_sequence index out of range");
    if (width == 0) throw invalid_argument("gap_percent of an empty alignment");  // metrics.cpp:17-19
    uint64_t pitch = 0;
    const uint8_t* d_rows = upload_rows(ctx, rows, nrows, width, &pitch);
    const uint64_t gaps = gap_count(ctx, d_rows, nrows, pitch, width);
    rep->gap_percent = 100.0 * (double)gaps / ((double)nrows * (double)width);  // metrics.cpp:24-26

    uint64_t max_len = 0;  // metrics.cpp:94-98
    for (uint64_t r = 0; r < nrows; ++r) {
        const uint32_t s = row_to_sequence[r];
        max_len = std::max<uint64_t>(max_len, raw_offsets[s + 1] - raw_offsets[s]);
    }
    rep->stretch = (double)width / (double)max_len;

    // metrics.cpp:103-120: seeded row sample, then a pair sample over it
    std::mt19937_64 row_rng(rng::combine_seed(seed, 1));
    const std::vector<uint64_t> row_pick = rng::sample_distinct(row_rng, nrows, sample_size);
    const uint64_t k = row_pick.size();
    rep->sample_size = k;
    if (k >= 2) {
        const uint64_t all_pairs = k * (k - 1) / 2;
        std::mt19937_64 pair_rng(rng::combine_seed(seed, 2));
        const std::vector<uint64_t> pair_pick = rng::sample_distinct(pair_rng, all_pairs, pair_budget);
        const uint64_t np = pair_pick.size();
        rep->pair_count = np;
        if (np) {
            std::vector<uint32_t> ra(np), rb(np);
            std::vector<LevItem> items(np);
            for (uint64_t t = 0; t < np; ++t) {
                const auto [pi, pj] = pair_from_index(pair_pick[t], k);
                ra[t] = (uint32_t)row_pick[pi];
                rb[t] = (uint32_t)row_pick[pj];
                items[t] = LevItem{row_to_sequence[ra[t]], row_to_sequence[rb[t]], (uint32_t)t};
            }
            const std::vector<PairCounts> pc = row_pairs(ctx, d_rows, pitch, ra, rb);
            // Levenshtein of the raw sequences (metrics.cpp:134-138) on the distance engine
            dm_seqset* s = seqset_create(ctx, raw, raw_offsets, nraw);
            std::vector<uint32_t> lev(np);
            try {
                uint32_t* d_out = ctx->stream_out.as<uint32_t>(np);
                lev_run_host_items(ctx, s, items, d_out, nullptr, false);
                DM_CUDA(cudaMemcpyAsync(lev.data(), d_out, np * 4, cudaMemcpyDeviceToHost, ctx->stream));
                DM_CUDA(cudaStreamSynchronize(ctx->stream));
            } catch (...) {
                delete s;
                throw;
            }
            delete s;
            // metrics.cpp:121-166, same order and the same double operations
            rep->p_min = 1.0;
            rep->p_max = 0.0;
            double p_sum = 0.0, ratio_sum = 0.0;
            uint64_t included = 0;
            for (uint64_t t = 0; t < np; ++t) {
                const double p = pc[t].considered == 0
                                     ? 1.0
                                     : (double)pc[t].mismatched / (double)pc[t].considered;  // :29-45
                rep->p_min = std::min(rep->p_min, p);
                rep->p_max = std::max(rep->p_max, p);
                p_sum += p;
                if (lev[t] == 0) {
                    ++rep->zero_distance_pairs;
                } else {
                    ratio_sum += (double)pc[t].hamming / (double)lev[t];
                    ++included;
                }
            }
            rep->p_avg = p_sum / (double)np;
            rep->distortion = included == 0 ? 0.0 : ratio_sum / (double)included;
        }
    }
    rep->time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double gap_percent(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width) {
    if (nrows == 0 || width == 0) throw invalid_argument("gap_percent of an empty alignment");
    uint64_t pitch = 0;
    const uint8_t* d_rows = upload_rows(ctx, rows, nrows, width, &pitch);
    return 100.0 * (double)gap_count(ctx, d_rows, nrows, pitch, width) / ((double)nrows * (double)width);
}

void row_pair_stats(dm_ctx* ctx, const char* a, const char* b, uint64_t len, uint32_t* considered,
                    uint32_t* mismatched, uint32_t* hamming) {
    std::vector<char> two(2 * len);
    std::memcpy(two.data(), a, len);
    std::memcpy(two.data() + len, b, len);
    uint64_t pitch = 0;
    const uint8_t* d_rows = upload_rows(ctx, two.data(), 2, len, &pitch);
    const auto pc = row_pairs(ctx, d_rows, pitch, {0u}, {1u});
    *considered = pc[0].considered;
    *mismatched = pc[0].mismatched;
    *hamming = pc[0].hamming;
}

}  // namespace dm

extern "C" {

int dm_evaluate(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, const uint32_t* row_to_sequence,
                const char* raw, const uint64_t* raw_offsets, uint32_t nraw, uint64_t sample_size,
                uint64_t pair_budget, uint64_t seed, dm_metrics* out) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && out && (rows || nrows == 0) && (row_to_sequence || nrows == 0) && raw_offsets,
                    "null argument");
        dm::evaluate(ctx, rows, nrows, width, row_to_sequence, raw, raw_offsets, nraw, sample_size, pair_budget,
                     seed, out);
    });
}

int dm_gap_percent(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, double* out) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && out, "null argument");
        *out = dm::gap_percent(ctx, rows, nrows, width);
    });
}

int dm_row_pair_stats(dm_ctx* ctx, const char* a, uint64_t na, const char* b, uint64_t nb, uint32_t* considered,
                      uint32_t* mismatched, uint32_t* hamming) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && considered && mismatched && hamming, "null argument");
        if (na != nb) throw dm::invalid_argument("rows must have equal length");
        dm::row_pair_stats(ctx, a, b, na, considered, mismatched, hamming);
    });
}

}  // extern "C"
