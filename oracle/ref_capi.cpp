// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (divmsa, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests, golden-vector generator and bench.py's CPU-baseline /
// `--impl reference` legs call the reference through ctypes. Only tests/,
// __graft_entry__.smoke() and bench.py's reference legs may load it.
//
// Every entry point calls the reference's own public API:
//   ref_levenshtein      -> divmsa::levenshtein            (distance.hpp:11)
//   ref_lev_pairs        -> divmsa::parallel_for + levenshtein, grain 64,
//                           the batching of cluster_tree.cpp:36
//   ref_nw_align         -> divmsa::nw_align               (pairwise.hpp:89)
//   ref_build_tree       -> divmsa::build_tree             (cluster_tree.hpp:66)
//   ref_geometric_median -> divmsa::geometric_median       (cluster_tree.hpp:56)
//   ref_msa              -> build_tree + align_all         (pipeline.cpp:116,128)
//   ref_align            -> divmsa::align_sequences        (pipeline.hpp:59)
//   ref_insert_gap_columns -> divmsa::insert_gap_columns   (msa_merge.hpp:34)
//   ref_evaluate         -> divmsa::evaluate               (metrics.hpp:53-56)
//   ref_run_align        -> divmsa::run_align              (pipeline.hpp:63-64)
//   ref_write_fasta      -> divmsa::write_fasta            (seq_io.hpp:82-83)
//   ref_gap_percent, ref_p_score, ref_hamming_aligned, ref_distortion_pair
//                        -> the metrics helpers            (metrics.hpp:39-49, distance.hpp)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <string_view>
#include <vector>

#include "divmsa/cluster_tree.hpp"
#include "divmsa/distance.hpp"
#include "divmsa/metrics.hpp"
#include "divmsa/msa_merge.hpp"
#include "divmsa/pairwise.hpp"
#include "divmsa/parallel.hpp"
#include "divmsa/pipeline.hpp"
#include "divmsa/seq_io.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

// Error codes mirror the C ABI of the product (include/dm_b200.h).
constexpr int kInvalidArgument = 1;
constexpr int kRuntimeError = 2;

std::vector<std::string_view> views(const char* const* seqs, const std::uint32_t* lens,
                                    std::uint64_t n) {
    std::vector<std::string_view> v(n);
    for (std::uint64_t i = 0; i < n; ++i) v[i] = std::string_view(seqs[i], lens[i]);
    return v;
}

divmsa::ScoringScheme make_scheme(int kind, const char* symbols, const int* matrix,
                                  int gap_open, int gap_extend, int flat) {
    const divmsa::GapMode mode = flat ? divmsa::GapMode::Flat : divmsa::GapMode::Affine;
    if (kind == 0) return divmsa::default_nucleotide_scheme(gap_open, gap_extend, mode);
    if (kind == 1) return divmsa::default_protein_scheme(gap_open, gap_extend, mode);
    const std::size_t n = std::strlen(symbols);
    return divmsa::ScoringScheme(std::string_view(symbols, n),
                                 std::span<const int>(matrix, n * n), gap_open,
                                 gap_extend, mode);
}

} // namespace

struct ref_pw {
    divmsa::PairwiseResult r;
};

struct ref_msa_out {
    divmsa::ClusterTree tree;
    divmsa::Msa msa;
    std::string flat_rows;
    double tree_s = 0, align_s = 0;
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint32_t ref_levenshtein(const char* a, std::uint64_t na, const char* b,
                              std::uint64_t nb) {
    return divmsa::levenshtein(std::string_view(a, na), std::string_view(b, nb));
}

// out[i] = levenshtein(seqs[ia[i]], seqs[ib[i]]) on a divmsa::ThreadPool.
int ref_lev_pairs(const char* const* seqs, const std::uint32_t* lens, std::uint64_t nseq,
                  const std::uint32_t* ia, const std::uint32_t* ib, std::uint64_t npairs,
                  int threads, std::uint32_t* out) {
    try {
        auto v = views(seqs, lens, nseq);
        divmsa::ThreadPool pool(threads > 0 ? threads : 1);
        divmsa::parallel_for(pool, 0, npairs, 64, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t i = lo; i < hi; ++i) out[i] = divmsa::levenshtein(v[ia[i]], v[ib[i]]);
        });
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

int ref_nw_align(const char* a, std::uint64_t na, const char* b, std::uint64_t nb,
                 int kind, const char* symbols, const int* matrix, int gap_open,
                 int gap_extend, int flat, ref_pw** out) {
    try {
        auto scheme = make_scheme(kind, symbols, matrix, gap_open, gap_extend, flat);
        auto* h = new ref_pw;
        h->r = divmsa::nw_align(std::string_view(a, na), std::string_view(b, nb), scheme);
        *out = h;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

// Scheme table export (128*128 int16) so tests can compare table construction.
int ref_scheme_table(int kind, const char* symbols, const int* matrix, int gap_open,
                     int gap_extend, int flat, std::int16_t* table, int* open_surcharge) {
    try {
        auto s = make_scheme(kind, symbols, matrix, gap_open, gap_extend, flat);
        for (int x = 0; x < 128; ++x)
            for (int y = 0; y < 128; ++y)
                table[x * 128 + y] = static_cast<std::int16_t>(s.score(char(x), char(y)));
        *open_surcharge = s.open_surcharge();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

std::int64_t ref_pw_score(const ref_pw* h) { return h->r.score; }
std::uint64_t ref_pw_len(const ref_pw* h) { return h->r.aligned_a.size(); }
const char* ref_pw_a(const ref_pw* h) { return h->r.aligned_a.data(); }
const char* ref_pw_b(const ref_pw* h) { return h->r.aligned_b.data(); }
std::uint64_t ref_pw_ngaps_a(const ref_pw* h) { return h->r.gaps_into_a.size(); }
std::uint64_t ref_pw_ngaps_b(const ref_pw* h) { return h->r.gaps_into_b.size(); }
const std::uint32_t* ref_pw_gaps_a(const ref_pw* h) { return h->r.gaps_into_a.data(); }
const std::uint32_t* ref_pw_gaps_b(const ref_pw* h) { return h->r.gaps_into_b.data(); }
void ref_pw_free(ref_pw* h) { delete h; }

// nodes_out: (2n-1) x 10 int64 = begin,end,center,radius,pole_l,pole_r,left,right,parent,depth
int ref_build_tree(const char* const* seqs, const std::uint32_t* lens, std::uint64_t n,
                   std::uint64_t seed, std::uint64_t cap, int threads,
                   std::int64_t* nodes_out, std::uint64_t* nnodes, std::uint32_t* order_out) {
    try {
        auto v = views(seqs, lens, n);
        divmsa::ThreadPool pool(threads > 0 ? threads : 1);
        divmsa::TreeBuildOptions opt;
        opt.seed = seed;
        opt.median_exact_cap = cap;
        auto t = divmsa::build_tree(v, opt, pool);
        *nnodes = t.nodes.size();
        for (std::size_t i = 0; i < t.nodes.size(); ++i) {
            const auto& nd = t.nodes[i];
            std::int64_t* o = nodes_out + 10 * i;
            o[0] = nd.begin; o[1] = nd.end; o[2] = nd.center; o[3] = nd.radius;
            o[4] = nd.pole_l; o[5] = nd.pole_r; o[6] = nd.left; o[7] = nd.right;
            o[8] = nd.parent; o[9] = nd.depth;
        }
        std::memcpy(order_out, t.order.data(), 4 * n);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

int ref_geometric_median(const char* const* seqs, const std::uint32_t* lens,
                         std::uint64_t nseq, const std::uint32_t* members,
                         std::uint64_t nmembers, std::uint64_t seed, std::uint64_t cap,
                         int threads, std::uint32_t* out) {
    try {
        auto v = views(seqs, lens, nseq);
        divmsa::ThreadPool pool(threads > 0 ? threads : 1);
        *out = divmsa::geometric_median(std::span<const std::uint32_t>(members, nmembers),
                                        v, seed, cap, pool);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

// build_tree then align_all on one pool (pipeline.cpp:113-128), timed separately.
int ref_msa(const char* const* seqs, const std::uint32_t* lens, std::uint64_t n,
            int kind, const char* symbols, const int* matrix, int gap_open,
            int gap_extend, int flat, std::uint64_t seed, int threads, ref_msa_out** out) {
    try {
        auto v = views(seqs, lens, n);
        auto scheme = make_scheme(kind, symbols, matrix, gap_open, gap_extend, flat);
        divmsa::ThreadPool pool(threads > 0 ? threads : 1);
        divmsa::TreeBuildOptions opt;
        opt.seed = seed;
        auto* h = new ref_msa_out;
        auto t0 = std::chrono::steady_clock::now();
        h->tree = divmsa::build_tree(v, opt, pool);
        auto t1 = std::chrono::steady_clock::now();
        h->msa = divmsa::align_all(h->tree, v, scheme, pool);
        auto t2 = std::chrono::steady_clock::now();
        h->tree_s = std::chrono::duration<double>(t1 - t0).count();
        h->align_s = std::chrono::duration<double>(t2 - t1).count();
        h->flat_rows.reserve(h->msa.rows.size() * h->msa.width);
        for (const auto& r : h->msa.rows) h->flat_rows += r;
        *out = h;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

std::uint64_t ref_msa_width(const ref_msa_out* h) { return h->msa.width; }
std::uint64_t ref_msa_rows(const ref_msa_out* h) { return h->msa.rows.size(); }
const char* ref_msa_data(const ref_msa_out* h) { return h->flat_rows.data(); }
const std::uint32_t* ref_msa_row_seq(const ref_msa_out* h) { return h->msa.row_to_sequence.data(); }
double ref_msa_tree_s(const ref_msa_out* h) { return h->tree_s; }
double ref_msa_align_s(const ref_msa_out* h) { return h->align_s; }
std::uint64_t ref_msa_nnodes(const ref_msa_out* h) { return h->tree.nodes.size(); }
void ref_msa_nodes(const ref_msa_out* h, std::int64_t* nodes_out, std::uint32_t* order_out) {
    for (std::size_t i = 0; i < h->tree.nodes.size(); ++i) {
        const auto& nd = h->tree.nodes[i];
        std::int64_t* o = nodes_out + 10 * i;
        o[0] = nd.begin; o[1] = nd.end; o[2] = nd.center; o[3] = nd.radius;
        o[4] = nd.pole_l; o[5] = nd.pole_r; o[6] = nd.left; o[7] = nd.right;
        o[8] = nd.parent; o[9] = nd.depth;
    }
    std::memcpy(order_out, h->tree.order.data(), 4 * h->tree.order.size());
}
void ref_msa_free(ref_msa_out* h) { delete h; }

// divmsa.align of the reference python module (py_module.cpp:120-155):
// RowOrder::Input, ids "seq<i>". rows_out: n * width bytes (caller frees via ref_free).
int ref_align(const char* const* seqs, const std::uint32_t* lens, std::uint64_t n,
              int alphabet, int gap_open, int gap_extend, int flat, std::uint64_t seed,
              int threads, char** rows_out, std::uint64_t* width_out) {
    try {
        divmsa::RunConfig config;
        config.alphabet = alphabet == 0   ? divmsa::AlphabetChoice::Auto
                          : alphabet == 1 ? divmsa::AlphabetChoice::Nucleotide
                                          : divmsa::AlphabetChoice::Protein;
        config.gap_open = gap_open;
        config.gap_extend = gap_extend;
        config.gap_mode = flat ? divmsa::GapMode::Flat : divmsa::GapMode::Affine;
        config.seed = seed;
        config.threads = static_cast<unsigned>(threads);
        config.order = divmsa::RowOrder::Input;
        std::vector<divmsa::Sequence> s(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            s[i].id = "seq" + std::to_string(i);
            s[i].residues.assign(seqs[i], lens[i]);
            s[i].original_index = static_cast<std::uint32_t>(i);
        }
        auto out = divmsa::align_sequences(std::move(s), config);
        const std::uint64_t w = out.summary.width;
        char* buf = new char[n * w + 1];
        for (std::uint64_t i = 0; i < n; ++i) std::memcpy(buf + i * w, out.records[i].row.data(), w);
        *rows_out = buf;
        *width_out = w;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

void ref_free(char* p) { delete[] p; }

// insert_gap_columns over a rows x width block; out: rows x (width + npos).
int ref_insert_gap_columns(const char* rows, std::uint64_t nrows, std::uint64_t width,
                           const std::uint32_t* pos, std::uint64_t npos, char* out) {
    try {
        divmsa::Msa m;
        m.width = width;
        for (std::uint64_t r = 0; r < nrows; ++r) {
            m.rows.emplace_back(rows + r * width, width);
            m.row_to_sequence.push_back(static_cast<std::uint32_t>(r));
        }
        divmsa::ThreadPool pool(1);
        auto o = divmsa::insert_gap_columns(std::move(m),
                                            std::span<const std::uint32_t>(pos, npos), pool);
        for (std::uint64_t r = 0; r < nrows; ++r) std::memcpy(out + r * o.width, o.rows[r].data(), o.width);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}


// Same field order as dm_metrics (include/dm_b200.h).
struct ref_metrics {
    std::uint64_t width;
    double stretch, gap_percent, distortion, p_min, p_avg, p_max;
    std::uint64_t sample_size, pair_count, seed, zero_distance_pairs;
    double time_s;
};

int ref_evaluate(const char* rows, std::uint64_t nrows, std::uint64_t width, const std::uint32_t* row_to_sequence,
                 const char* const* raws, const std::uint32_t* raw_lens, std::uint64_t nraw,
                 std::uint64_t sample_size, std::uint64_t pair_budget, std::uint64_t seed, int threads,
                 ref_metrics* out) {
    try {
        divmsa::Msa m;
        m.width = width;
        for (std::uint64_t r = 0; r < nrows; ++r) {
            m.rows.emplace_back(rows + r * width, width);
            m.row_to_sequence.push_back(row_to_sequence[r]);
        }
        const auto v = views(raws, raw_lens, nraw);
        divmsa::ThreadPool pool(threads > 0 ? (unsigned)threads : 1u);
        const auto t0 = std::chrono::steady_clock::now();
        const divmsa::MetricsReport r = divmsa::evaluate(m, v, sample_size, pair_budget, seed, pool);
        *out = ref_metrics{r.width, r.stretch, r.gap_percent, r.distortion, r.p_min, r.p_avg, r.p_max,
                           r.sample_size, r.pair_count, r.seed, r.zero_distance_pairs,
                           std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count()};
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

int ref_gap_percent(const char* rows, std::uint64_t nrows, std::uint64_t width, double* out) {
    try {
        divmsa::Msa m;
        m.width = width;
        for (std::uint64_t r = 0; r < nrows; ++r) m.rows.emplace_back(rows + r * width, width);
        *out = divmsa::gap_percent(m);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

int ref_p_score(const char* a, std::uint64_t na, const char* b, std::uint64_t nb, double* out) {
    try {
        *out = divmsa::p_score(std::string_view(a, na), std::string_view(b, nb));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    }
}

int ref_hamming_aligned(const char* a, std::uint64_t na, const char* b, std::uint64_t nb, std::uint32_t* out) {
    try {
        *out = divmsa::hamming_aligned(std::string_view(a, na), std::string_view(b, nb));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    }
}

int ref_distortion_pair(const char* a, std::uint64_t na, const char* b, std::uint64_t nb, const char* ra,
                        std::uint64_t nra, const char* rb, std::uint64_t nrb, double* out) {
    try {
        *out = divmsa::distortion_pair(std::string_view(a, na), std::string_view(b, nb), std::string_view(ra, nra),
                                       std::string_view(rb, nrb));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    }
}


int ref_run_align(const char* input, const char* output, int alphabet, int gap_open, int gap_extend, int flat,
                  std::uint64_t seed, int input_order, int threads, const char* dump_tree,
                  const char* dump_dedup) {
    try {
        divmsa::RunConfig c;
        c.alphabet = alphabet == 1   ? divmsa::AlphabetChoice::Nucleotide
                     : alphabet == 2 ? divmsa::AlphabetChoice::Protein
                                     : divmsa::AlphabetChoice::Auto;
        c.gap_open = gap_open;
        c.gap_extend = gap_extend;
        c.gap_mode = flat ? divmsa::GapMode::Flat : divmsa::GapMode::Affine;
        c.seed = seed;
        c.threads = threads > 0 ? (unsigned)threads : 0u;
        c.order = input_order ? divmsa::RowOrder::Input : divmsa::RowOrder::Tree;
        if (dump_tree) c.dump_tree_path = dump_tree;
        if (dump_dedup) c.dump_dedup_path = dump_dedup;
        divmsa::run_align(c, input, output);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, kInvalidArgument);
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

int ref_write_fasta(const char* path, const char* ids, const std::uint64_t* id_off, const char* descs,
                    const std::uint64_t* desc_off, const char* residues, const std::uint64_t* res_off,
                    std::uint64_t n) {
    try {
        std::vector<divmsa::FastaRecordView> v(n);
        for (std::uint64_t k = 0; k < n; ++k)
            v[k] = divmsa::FastaRecordView{std::string_view(ids + id_off[k], id_off[k + 1] - id_off[k]),
                                           std::string_view(descs + desc_off[k], desc_off[k + 1] - desc_off[k]),
                                           std::string_view(residues + res_off[k], res_off[k + 1] - res_off[k])};
        divmsa::write_fasta(v, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, kRuntimeError);
    }
}

} // extern "C"
