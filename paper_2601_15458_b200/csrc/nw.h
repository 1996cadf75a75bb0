// Batched Gotoh NW (nw.cu) — shared by the pairwise C ABI and the merge
// scheduler (msa.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "dm_internal.h"

namespace dm {

// One alignment of a = chars[a_off, a_off+n) against b = chars[b_off, b_off+m).
struct NwJob {
    uint64_t a_off, b_off;
    uint32_t n, m;
    uint64_t t_off;   // trace bytes: m columns x round16(n) rows (filled by nw_run)
    uint64_t ga_off;  // gaps_into_a output (capacity m), path order (descending)
    uint64_t gb_off;  // gaps_into_b output (capacity n), path order (descending)
    uint32_t slot;    // index of the result (set by nw_run)
    uint32_t pad;
};

struct NwRes {
    int64_t score;
    uint32_t final_tag;  // 2 - final state
    uint32_t len;        // aligned length
    uint32_t nga, ngb;   // gap counts
};

// Scoring scheme in device form: chars -> dense codes, 4*score table.
struct NwScheme {
    uint8_t lut[128] = {};
    int K = 0, Kp = 1;
    std::vector<int32_t> table4;  // K x Kp
    std::vector<int16_t> score;   // K x K raw scores (dense codes)
    int64_t open = 0, extend = 0;
    int maxabs = 0;
    bool has[128] = {};
    // Column symbols known to occur (set_columns): the throughput kernel then
    // keeps a per-lane query profile over them (nw_seq.cuh PROF) when KE <= 8.
    int KE = 0;
    uint8_t plut[128] = {};  // char -> profile symbol
    uint8_t pdense[128] = {};  // profile symbol -> dense code
};

NwScheme make_scheme(const int16_t* table, const uint8_t* has_symbol, int open_surcharge, int gap_extend);
// Restrict the column alphabet to the chars flagged in `present` (128
// flags; chars the scheme does not score are ignored).
void set_columns(NwScheme& sc, const bool* present);

// Device outputs of one batch (valid until the next nw_run on this ctx).
struct NwOut {
    NwRes* d_res = nullptr;
    uint32_t* d_gaps = nullptr;
    uint64_t gaps_total = 0;
    float fwd_ms = 0.f, tb_ms = 0.f;
    uint64_t cells = 0;
    uint64_t cells_exec = 0;  // rows padded to whole bands
    uint64_t launches = 0;
};

// Runs forward + traceback over `jobs` (host array; t_off/ga_off/gb_off are
// assigned here). `d_chars` is device memory holding every a and b.
// layout_given: slots / gap offsets are already set and out.d_res / d_gaps
// point at the (shared) result buffers — used by nw_run_sharded.
void nw_run(dm_ctx* ctx, const uint8_t* d_chars, std::vector<NwJob>& jobs, const NwScheme& sc,
            NwOut& out, bool time_kernels, bool layout_given = false);
// Same results, with the jobs split across the context's shards (attached
// ranks or the simulated world) in cost-balanced ranges; the ranks exchange
// the results and compacted gap lists, so every rank holds all of them.
// local: this rank aligns the whole batch (merges inside its own subtrees).
void nw_run_sharded(dm_ctx* ctx, const uint8_t* d_chars, std::vector<NwJob>& jobs, const NwScheme& sc,
                    NwOut& out, bool time_kernels, bool local = false);

// Gathers each job's nga + ngb gap entries (path order, gaps_into_a first)
// into one compact host array; off[k] = start of job k's entries.
void nw_compact_gaps(dm_ctx* ctx, const uint32_t* d_gaps, const std::vector<NwJob>& jobs,
                     const std::vector<NwRes>& res, std::vector<uint32_t>& out, std::vector<uint64_t>& off);

// Index of the first byte of d_bytes[0, n) that is not a symbol of the
// scheme (>= 128 or has[c] false), or UINT64_MAX; one scan on ctx->stream
// and one host sync. (pairwise.cpp:288-297 checks on the host; the batch
// checks the uploaded bytes instead.)
// present (optional, 128 flags): set for every byte value < 128 found in d_bytes.
uint64_t nw_first_bad_symbol(dm_ctx* ctx, const uint8_t* d_bytes, uint64_t n, const bool* has,
                             bool* present = nullptr);

}  // namespace dm
