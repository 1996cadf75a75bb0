// The boundary caller: divmsa::align_sequences
// (pipeline.cpp:78-159) around the GPU tree builder and merge scheduler.
// Host work only: alphabet resolution (alphabet.cpp:37-57), residue
// validation (seq_io.cpp:148-166), scheme coverage check (pipeline.cpp:92-100),
// de-duplication keeping first occurrences (seq_io.cpp:168-186), then
// build_tree + align_all on the device, then duplicate re-expansion in tree or
// input row order (pipeline.cpp:130-146).
#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <string_view>

#include "capi_guard.h"
#include "host_par.h"
#include "nw.h"
#include "pipeline.h"
#include "nvtx.h"

namespace dm {
namespace {

constexpr std::string_view kNucleotide = "ACGTURYSWKMBDHVN";
constexpr std::string_view kProtein = "ARNDCQEGHILKMFPSTWYVBZX*";

int detect_alphabet(const char* data, uint64_t nbytes) {  // alphabet.cpp:37-57; 0 nt, 1 aa
    // counted in parallel chunks (the same totals as the reference's loop)
    const uint64_t chunk = 1 << 20, nc = (nbytes + chunk - 1) / chunk;
    std::vector<uint64_t> tot(nc, 0), ntc(nc, 0);
    host_parallel_for(nc, 1, [&](uint64_t k) {
        uint64_t t = 0, c = 0;
        for (uint64_t i = k * chunk, e = std::min(nbytes, i + chunk); i < e; ++i) {
            const char raw = data[i];
            if (raw == '-') continue;
            ++t;
            switch ((char)std::toupper((unsigned char)raw)) {
                case 'A': case 'C': case 'G': case 'T': case 'U': case 'N': ++c; break;
                default: break;
            }
        }
        tot[k] = t;
        ntc[k] = c;
    });
    uint64_t total = 0, nt = 0;
    for (uint64_t k = 0; k < nc; ++k) {
        total += tot[k];
        nt += ntc[k];
    }
    if (total == 0) return 0;
    return nt * 10 > total * 9 ? 0 : 1;
}

}  // namespace
}  // namespace dm

namespace dm {

// align_sequences (pipeline.cpp:78-159) up to the re-expansion: validation,
// de-duplication, tree + merges on the device. `ids` (optional) names the
// records in error messages; without it they are "seq<i>" (py_module.cpp:134-138).
AlignCore align_core(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                     const std::vector<std::string>* ids, int alphabet, int gap_open, int gap_extend, int flat,
                     const int16_t* custom_table, const uint8_t* custom_has, uint64_t seed, int input_order,
                     dm_stats* st, bool host_rows) {
    AlignCore res;
    NvtxRange nvtx_core("dm align_sequences");
    const auto t0 = std::chrono::steady_clock::now();
    const bool trace = std::getenv("DM_TRACE") != nullptr;
    auto tlast = t0;
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[dm align_sequences] %s %.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - tlast).count());
        tlast = t;
    };
    if (n == 0) throw runtime_error("no sequences to align");
    if (gap_open > gap_extend || gap_extend > 0)
        throw invalid_argument("gap penalties must satisfy gap_open <= gap_extend <= 0");
    const uint64_t base = offsets[0];
    const int kind = alphabet == 1 ? 0 : alphabet == 2 ? 1 : detect_alphabet(data + base, offsets[n] - base);
    auto rec = [ids](uint32_t i) {
        return "record '" + (ids ? (*ids)[i] : "seq" + std::to_string(i)) + "'";
    };
    // One parallel pass over the records: the byte classes each record holds
    // (bit 0: outside the alphabet, validate_residues, seq_io.cpp:148-166;
    // bit 1: not scored by the scheme, pipeline.cpp:92-100) and its hash for
    // de-duplication. Errors are then reported for the first failing record
    // in input order, with messages built sequentially, exactly as the
    // reference's in-order loops report them (alphabet first, then the
    // scheme's own validation, then unscored residues).
    int16_t table[128 * 128];
    uint8_t has[128];
    int osur = 0;
    std::exception_ptr scheme_err;
    if (custom_table) {
        std::memcpy(table, custom_table, sizeof(table));
        std::memcpy(has, custom_has, sizeof(has));
        osur = flat ? 0 : gap_open;
    } else {
        const int rc = dm_scheme_default(kind, gap_open, gap_extend, flat, table, has, &osur);
        if (rc != DM_OK) scheme_err = std::make_exception_ptr(invalid_argument(last_error()));
    }
    bool member[256] = {};
    for (char c : (kind == 0 ? kNucleotide : kProtein)) member[(unsigned char)c] = true;
    uint8_t cls[256];
    for (int c = 0; c < 256; ++c)
        cls[c] = (uint8_t)((!custom_table && !member[c] ? 1 : 0) | (!scheme_err && (c >= 128 || !has[c]) ? 2 : 0));
    std::vector<uint64_t> hv(n);
    std::vector<uint8_t> rcls(n);
    host_parallel_for(n, 256, [&](uint64_t i) {
        const unsigned char* d = reinterpret_cast<const unsigned char*>(data + offsets[i]);
        const uint64_t L = offsets[i + 1] - offsets[i];
        uint8_t acc = 0;
        for (uint64_t p = 0; p < L; ++p) acc |= cls[d[p]];
        rcls[i] = acc;
        hv[i] = std::hash<std::string_view>{}(std::string_view(data + offsets[i], L));
    });
    auto first_with = [&](uint8_t bit) -> uint32_t {
        for (uint32_t i = 0; i < n; ++i)
            if (rcls[i] & bit) return i;
        return UINT32_MAX;
    };
    if (!custom_table) {  // validate_residues (seq_io.cpp:148-166)
        const uint32_t i = first_with(1);
        if (i != UINT32_MAX)
            for (uint64_t p = offsets[i]; p < offsets[i + 1]; ++p) {
                const char c = data[p];
                if (c == '-') throw runtime_error(rec(i) + " contains gap symbol '-' in unaligned input");
                if (!member[(unsigned char)c])
                    throw runtime_error(rec(i) + " contains character '" + std::string(1, c) + "' outside the " +
                                        (kind == 0 ? "nucleotide" : "protein") + " alphabet");
            }
    }
    if (scheme_err) std::rethrow_exception(scheme_err);
    {  // every residue scored by the scheme (pipeline.cpp:92-100)
        const uint32_t i = first_with(2);
        if (i != UINT32_MAX)
            for (uint64_t p = offsets[i]; p < offsets[i + 1]; ++p) {
                const unsigned char c = (unsigned char)data[p];
                if (c >= 128 || !has[c])
                    throw runtime_error(rec(i) + " contains character '" + std::string(1, (char)c) +
                                        "' that the substitution matrix does not score");
            }
    }
    mark("validate");
    // deduplicate: first occurrences in order (seq_io.cpp:168-186) through an
    // open-addressing table of record indices keyed by the hashes above
    uint64_t cap = 16;
    while (cap < 2ull * n) cap <<= 1;
    std::vector<uint32_t> slot_rec(cap, UINT32_MAX), slot_rep(cap, 0);
    std::vector<uint32_t> reps;
    std::vector<std::vector<uint32_t>> dups;
    for (uint32_t i = 0; i < n; ++i) {
        const uint64_t L = offsets[i + 1] - offsets[i];
        uint64_t h = hv[i] & (cap - 1);
        for (;; h = (h + 1) & (cap - 1)) {
            const uint32_t j = slot_rec[h];
            if (j == UINT32_MAX) {  // first occurrence
                slot_rec[h] = i;
                slot_rep[h] = (uint32_t)reps.size();
                reps.push_back(i);
                dups.emplace_back();
                break;
            }
            if (hv[j] == hv[i] && offsets[j + 1] - offsets[j] == L &&
                std::memcmp(data + offsets[j], data + offsets[i], L) == 0) {
                dups[slot_rep[h]].push_back(i);
                break;
            }
        }
    }
    res.reps = reps;
    res.dups = dups;
    mark("dedup");
    dm_seqset* s = nullptr;
    if (reps.size() == n) {  // no duplicates: the caller's buffer as it is
        s = seqset_create(ctx, data, offsets, n);
    } else {  // the distinct sequences, packed (no zero fill: every byte is copied)
        std::vector<uint64_t> roff(reps.size() + 1, 0);
        for (size_t r = 0; r < reps.size(); ++r) roff[r + 1] = roff[r] + (offsets[reps[r] + 1] - offsets[reps[r]]);
        std::unique_ptr<char[]> rdata(new char[std::max<uint64_t>(roff[reps.size()], 1)]);
        host_parallel_for(reps.size(), 256, [&](uint64_t r) {
            std::memcpy(rdata.get() + roff[r], data + offsets[reps[r]], roff[r + 1] - roff[r]);
        });
        s = seqset_create(ctx, rdata.get(), roff.data(), (uint32_t)reps.size());
    }
    mark("seqset");
    try {
        const NwScheme sc = make_scheme(table, has, osur, gap_extend);
        std::vector<dm_node> nodes;
        std::vector<uint32_t> order;
        dm_stats ts{}, as{};
        const auto p0 = std::chrono::steady_clock::now();
        build_tree(ctx, s, seed, 100, nodes, order, st ? &ts : nullptr);
        const auto p1 = std::chrono::steady_clock::now();
        res.msa.reset(align_all(ctx, s, nodes, order, sc, st ? &as : nullptr, nullptr, nullptr, host_rows));
        const auto p2 = std::chrono::steady_clock::now();
        mark("tree+align");
        // re-expand duplicates (pipeline.cpp:130-146): output slot -> (input record, MSA row)
        res.slot_input.assign(n, 0);
        res.slot_row.assign(n, 0);
        uint64_t slot = 0;
        for (size_t r = 0; r < res.msa->row_seq.size(); ++r) {
            const uint32_t rep = res.msa->row_seq[r];
            const auto place = [&](uint32_t orig) {
                const uint64_t at = input_order ? orig : slot++;
                res.slot_input[at] = orig;
                res.slot_row[at] = (uint32_t)r;
            };
            place(reps[rep]);
            for (uint32_t d : dups[rep]) place(d);
        }
        mark("expand");
        res.summary.input_count = n;
        res.summary.unique_count = reps.size();
        res.summary.duplicate_count = n - reps.size();
        uint32_t depth = 0;
        for (const auto& nd : nodes) depth = std::max(depth, nd.depth);
        res.summary.tree_depth = depth;
        res.summary.width = res.msa->width;
        res.summary.alphabet = kind;
        res.summary.elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->cells = ts.cells + as.cells;
            st->cells_executed = ts.cells_executed + as.cells;
            st->kernel_ms = ts.kernel_ms + as.kernel_ms;
            st->launches = ts.launches + as.launches;
            st->nw_calls = as.nw_calls;
            // host wall time of the two phases (both end synchronised: the
            // tree's nodes and the MSA rows are in host memory)
            st->tree_ms = std::chrono::duration<double, std::milli>(p1 - p0).count();
            st->align_ms = std::chrono::duration<double, std::milli>(p2 - p1).count();
            st->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
    } catch (...) {
        delete s;
        throw;
    }
    delete s;
    return res;
}

}  // namespace dm

extern "C" {

int dm_align_sequences(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n, int alphabet,
                       int gap_open, int gap_extend, int flat, const int16_t* custom_table,
                       const uint8_t* custom_has, uint64_t seed, int input_order, char** rows_out,
                       uint64_t* width_out, dm_align_summary* summary, dm_stats* st) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && offsets && rows_out && width_out, "null argument");
        // rows stay on the device; output slot k = MSA row slot_row[k], gathered there
        dm::AlignCore res = dm::align_core(ctx, data, offsets, n, nullptr, alphabet, gap_open, gap_extend, flat,
                                           custom_table, custom_has, seed, input_order, st, false);
        const uint64_t W = res.msa->width;
        char* out = (char*)std::malloc(std::max<uint64_t>((uint64_t)n * W, 1));
        if (!out) throw std::bad_alloc();
        dm::gather_rows_to_host(ctx, (const uint8_t*)ctx->rows_a.p, res.msa->dev_pitch, res.slot_row.data(), n, W,
                                out);
        *rows_out = out;
        *width_out = W;
        if (summary) *summary = res.summary;
    });
}

}  // extern "C"
