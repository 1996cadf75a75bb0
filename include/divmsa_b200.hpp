// divmsa_b200.hpp — header-only C++ drop-in for the reference's hot-path API
// (namespace divmsa, /root/reference/proj/include/divmsa/*.hpp), implemented
// on the C ABI of libdmb200.so (include/dm_b200.h).
//
// Same names, argument meaning, return types and exception types/messages as
// the reference:
//   levenshtein          distance.hpp:11
//   ScoringScheme,       pairwise.hpp:22-52, :64-70
//   default_*_scheme
//   PairwiseResult,      pairwise.hpp:78-90
//   nw_align
//   ClusterNode/-Tree,   cluster_tree.hpp:20-50
//   TreeBuildOptions
//   geometric_median     cluster_tree.hpp:56-59
//   build_tree           cluster_tree.hpp:66-67
//   Msa, align_leaf,     msa_merge.hpp:18-49
//   insert_gap_columns,
//   merge, align_all
// ThreadPool is accepted for signature compatibility and is used for host
// work only (the reference passes it through every call); the GPU does the
// data-parallel work. A process-wide dm_ctx on device 0 (or DM_DEVICE) is
// created on first use.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "dm_b200.h"

namespace divmsa {

inline constexpr std::uint32_t kNoSequence = 0xffffffffu;
inline constexpr std::size_t kMedianExactCap = 100;
constexpr char kGapSymbol = '-';

namespace detail {
inline void check(int rc) {
    if (rc == DM_OK) return;
    const std::string msg = dm_last_error();
    if (rc == DM_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
inline dm_ctx* ctx() {
    static std::once_flag once;
    static dm_ctx* c = nullptr;
    std::call_once(once, [] {
        const char* d = std::getenv("DM_DEVICE");
        check(dm_ctx_create(d ? std::atoi(d) : 0, &c));
    });
    return c;
}
struct SeqsetDeleter {
    void operator()(dm_seqset* s) const { dm_seqset_destroy(s); }
};
using Seqset = std::unique_ptr<dm_seqset, SeqsetDeleter>;
inline Seqset upload(std::span<const std::string_view> seqs) {
    std::string data;
    std::vector<std::uint64_t> off(seqs.size() + 1, 0);
    for (std::size_t i = 0; i < seqs.size(); ++i) {
        data.append(seqs[i]);
        off[i + 1] = data.size();
    }
    dm_seqset* s = nullptr;
    check(dm_seqset_create(ctx(), data.data(), off.data(), static_cast<std::uint32_t>(seqs.size()), &s));
    return Seqset(s);
}
}  // namespace detail

/// Minimal stand-in for divmsa::ThreadPool (parallel.hpp:18-45): accepted by
/// every signature; runs submitted host tasks.
class ThreadPool {
public:
    explicit ThreadPool(std::size_t threads) : n_(std::max<std::size_t>(1, threads)) {}
    std::size_t worker_count() const { return n_; }
    void submit(std::function<void()> task) { task(); }
    void wait_all() {}

private:
    std::size_t n_;
};

/// distance.hpp:11
inline std::uint32_t levenshtein(std::string_view a, std::string_view b) {
    int st = 0;
    const std::uint32_t d = dm_levenshtein(detail::ctx(), a.data(), a.size(), b.data(), b.size(), &st);
    detail::check(st);
    return d;
}

enum class GapMode { Flat, Affine };

/// pairwise.hpp:22-52
class ScoringScheme {
public:
    ScoringScheme(std::string_view symbols, std::span<const int> matrix, int gap_open, int gap_extend,
                  GapMode mode)
        : symbols_(symbols), gap_open_(gap_open), gap_extend_(gap_extend), mode_(mode), table_(128 * 128) {
        if (matrix.size() != symbols.size() * symbols.size() && !symbols.empty())
            throw std::invalid_argument("substitution matrix size does not match symbol count");
        int osur = 0;
        detail::check(dm_scheme_custom(symbols_.data(), static_cast<std::uint32_t>(symbols_.size()),
                                       matrix.data(), gap_open, gap_extend, mode == GapMode::Flat, nullptr, 0,
                                       table_.data(), has_, &osur));
    }
    int score(char x, char y) const {
        return table_[static_cast<unsigned char>(x) * 128 + static_cast<unsigned char>(y)];
    }
    bool has_symbol(char c) const {
        const auto u = static_cast<unsigned char>(c);
        return u < 128 && has_[u] != 0;
    }
    int gap_open() const { return gap_open_; }
    int gap_extend() const { return gap_extend_; }
    GapMode mode() const { return mode_; }
    int open_surcharge() const { return mode_ == GapMode::Affine ? gap_open_ : 0; }
    std::string_view symbols() const { return symbols_; }
    void set_score(char x, char y, int value) {
        if (value < -32768 || value > 32767) throw std::invalid_argument("substitution score out of range");
        table_[static_cast<unsigned char>(x) * 128 + static_cast<unsigned char>(y)] = static_cast<std::int16_t>(value);
        table_[static_cast<unsigned char>(y) * 128 + static_cast<unsigned char>(x)] = static_cast<std::int16_t>(value);
    }
    const std::int16_t* table() const { return table_.data(); }
    const std::uint8_t* has() const { return has_; }

    static ScoringScheme builtin(int kind, int gap_open, int gap_extend, GapMode mode) {
        ScoringScheme s(gap_open, gap_extend, mode, kind == 0 ? "ACGTURYSWKMBDHVN" : "ARNDCQEGHILKMFPSTWYVBZX*");
        int osur = 0;
        detail::check(dm_scheme_default(kind, gap_open, gap_extend, mode == GapMode::Flat, s.table_.data(), s.has_,
                                        &osur));
        return s;
    }

private:
    ScoringScheme(int go, int ge, GapMode mode, std::string_view symbols)
        : symbols_(symbols), gap_open_(go), gap_extend_(ge), mode_(mode), table_(128 * 128) {}
    std::string symbols_;
    int gap_open_, gap_extend_;
    GapMode mode_;
    std::vector<std::int16_t> table_;
    std::uint8_t has_[128] = {};
};

/// pairwise.hpp:64-70
inline ScoringScheme default_nucleotide_scheme(int gap_open = -10, int gap_extend = -1,
                                               GapMode mode = GapMode::Affine) {
    return ScoringScheme::builtin(0, gap_open, gap_extend, mode);
}
inline ScoringScheme default_protein_scheme(int gap_open = -10, int gap_extend = -1,
                                            GapMode mode = GapMode::Affine) {
    return ScoringScheme::builtin(1, gap_open, gap_extend, mode);
}

/// pairwise.hpp:78-84
struct PairwiseResult {
    std::string aligned_a;
    std::string aligned_b;
    std::int64_t score = 0;
    std::vector<std::uint32_t> gaps_into_a;
    std::vector<std::uint32_t> gaps_into_b;
};

/// pairwise.hpp:89-90
inline PairwiseResult nw_align(std::string_view a, std::string_view b, const ScoringScheme& scheme) {
    dm_pw* h = nullptr;
    detail::check(dm_nw_align(detail::ctx(), a.data(), a.size(), b.data(), b.size(), scheme.table(), scheme.has(),
                              scheme.open_surcharge(), scheme.gap_extend(), &h));
    PairwiseResult r;
    const std::uint64_t n = dm_pw_len(h, 0);
    r.aligned_a.resize(n);
    r.aligned_b.resize(n);
    dm_pw_aligned(h, 0, r.aligned_a.data(), r.aligned_b.data());
    r.score = dm_pw_score(h, 0);
    r.gaps_into_a.resize(dm_pw_ngaps_a(h, 0));
    r.gaps_into_b.resize(dm_pw_ngaps_b(h, 0));
    dm_pw_gaps(h, 0, r.gaps_into_a.data(), r.gaps_into_b.data());
    dm_pw_free(h);
    return r;
}

/// cluster_tree.hpp:20-34
struct ClusterNode {
    std::uint32_t begin = 0;
    std::uint32_t end = 0;
    std::uint32_t center = kNoSequence;
    std::uint32_t radius = 0;
    std::uint32_t pole_l = kNoSequence;
    std::uint32_t pole_r = kNoSequence;
    std::int32_t left = -1;
    std::int32_t right = -1;
    std::int32_t parent = -1;
    std::uint32_t depth = 0;
    bool is_leaf() const { return left < 0; }
    std::uint32_t size() const { return end - begin; }
};
static_assert(sizeof(ClusterNode) == sizeof(dm_node), "ClusterNode must mirror dm_node");

/// cluster_tree.hpp:36-45
struct ClusterTree {
    std::vector<ClusterNode> nodes;
    std::vector<std::uint32_t> order;
    std::span<const std::uint32_t> members(const ClusterNode& node) const {
        return std::span(order).subspan(node.begin, node.size());
    }
    std::size_t leaf_count() const {
        return static_cast<std::size_t>(std::count_if(nodes.begin(), nodes.end(), [](auto& n) { return n.is_leaf(); }));
    }
    std::uint32_t max_depth() const {
        std::uint32_t d = 0;
        for (const auto& n : nodes) d = std::max(d, n.depth);
        return d;
    }
};

/// cluster_tree.hpp:47-50
struct TreeBuildOptions {
    std::uint64_t seed = 42;
    std::size_t median_exact_cap = kMedianExactCap;
};

/// cluster_tree.hpp:56-59
inline std::uint32_t geometric_median(std::span<const std::uint32_t> members,
                                      std::span<const std::string_view> seqs, std::uint64_t seed,
                                      std::size_t exact_cap, ThreadPool&) {
    auto s = detail::upload(seqs);
    std::uint32_t out = 0;
    detail::check(dm_geometric_median(detail::ctx(), s.get(), members.data(), members.size(), seed, exact_cap, &out));
    return out;
}

/// cluster_tree.hpp:66-67
inline ClusterTree build_tree(std::span<const std::string_view> seqs, const TreeBuildOptions& options,
                              ThreadPool&) {
    if (seqs.empty()) throw std::runtime_error("cannot build a cluster tree from zero sequences");
    auto s = detail::upload(seqs);
    ClusterTree t;
    t.nodes.resize(2 * seqs.size() - 1);
    t.order.resize(seqs.size());
    std::uint64_t nn = 0;
    detail::check(dm_build_tree(detail::ctx(), s.get(), options.seed, options.median_exact_cap,
                                reinterpret_cast<dm_node*>(t.nodes.data()), &nn, t.order.data(), nullptr));
    t.nodes.resize(nn);
    return t;
}

/// msa_merge.hpp:18-26
struct Msa {
    std::vector<std::string> rows;
    std::vector<std::uint32_t> row_to_sequence;
    std::size_t width = 0;
    std::size_t row_count() const { return rows.size(); }
    std::size_t row_of(std::uint32_t sequence) const {
        for (std::size_t i = 0; i < row_to_sequence.size(); ++i)
            if (row_to_sequence[i] == sequence) return i;
        throw std::invalid_argument("center row for sequence " + std::to_string(sequence) + " not found in alignment");
    }
};

/// msa_merge.hpp:29
inline Msa align_leaf(const ClusterNode& node, std::span<const std::string_view> seqs) {
    if (!node.is_leaf() || node.size() != 1) throw std::invalid_argument("align_leaf requires a singleton leaf node");
    Msa m;
    m.rows.emplace_back(seqs[node.center]);
    m.row_to_sequence.push_back(node.center);
    m.width = m.rows[0].size();
    return m;
}

/// msa_merge.hpp:34-35
inline Msa insert_gap_columns(Msa msa, std::span<const std::uint32_t> positions, ThreadPool&) {
    if (positions.empty()) return msa;
    std::string flat;
    flat.reserve(msa.rows.size() * msa.width);
    for (const auto& r : msa.rows) flat += r;
    const std::size_t nw = msa.width + positions.size();
    std::string out(msa.rows.size() * nw, '\0');
    detail::check(dm_insert_gap_columns(detail::ctx(), flat.data(), msa.rows.size(), msa.width, positions.data(),
                                        positions.size(), out.data()));
    for (std::size_t r = 0; r < msa.rows.size(); ++r) msa.rows[r] = out.substr(r * nw, nw);
    msa.width = nw;
    return msa;
}

/// msa_merge.hpp:40-41
inline Msa merge(const ClusterTree& tree, const ClusterNode& node, Msa left, Msa right,
                 const ScoringScheme& scheme, ThreadPool& pool) {
    if (node.is_leaf()) throw std::invalid_argument("merge requires an internal node");
    const std::size_t lr = left.row_of(tree.nodes[node.left].center);
    const std::size_t rr = right.row_of(tree.nodes[node.right].center);
    const PairwiseResult al = nw_align(left.rows[lr], right.rows[rr], scheme);
    left = insert_gap_columns(std::move(left), al.gaps_into_a, pool);
    right = insert_gap_columns(std::move(right), al.gaps_into_b, pool);
    Msa parent;
    parent.width = al.aligned_a.size();
    parent.rows = std::move(left.rows);
    parent.row_to_sequence = std::move(left.row_to_sequence);
    parent.rows.insert(parent.rows.end(), std::make_move_iterator(right.rows.begin()),
                       std::make_move_iterator(right.rows.end()));
    parent.row_to_sequence.insert(parent.row_to_sequence.end(), right.row_to_sequence.begin(),
                                  right.row_to_sequence.end());
    return parent;
}

using ProgressFn = std::function<void(std::size_t done, std::size_t total)>;

/// msa_merge.hpp:47-49 — the whole bottom-up pass as per-level GPU batches.
inline Msa align_all(const ClusterTree& tree, std::span<const std::string_view> seqs, const ScoringScheme& scheme,
                     ThreadPool&, const ProgressFn& progress = nullptr) {
    auto s = detail::upload(seqs);
    dm_msa_out* h = nullptr;
    detail::check(dm_align_all(detail::ctx(), s.get(), reinterpret_cast<const dm_node*>(tree.nodes.data()),
                               tree.nodes.size(), tree.order.data(), scheme.table(), scheme.has(),
                               scheme.open_surcharge(), scheme.gap_extend(), &h, nullptr));
    Msa m;
    m.width = dm_msa_width(h);
    const std::size_t R = dm_msa_rows(h);
    std::string flat(R * m.width, '\0');
    dm_msa_copy_rows(h, flat.data());
    m.row_to_sequence.resize(R);
    dm_msa_copy_row_seq(h, m.row_to_sequence.data());
    dm_msa_free(h);
    m.rows.reserve(R);
    for (std::size_t r = 0; r < R; ++r) m.rows.push_back(flat.substr(r * m.width, m.width));
    if (progress)
        for (std::size_t i = 1; i <= tree.nodes.size(); ++i) progress(i, tree.nodes.size());
    return m;
}

// ---- quality metrics (metrics.hpp, distance.hpp:hamming_aligned) -------------
/// metrics.hpp:13-35
struct MetricsReport {
    std::size_t width = 0;
    double stretch = 0.0;
    double gap_percent = 0.0;
    double distortion = 0.0;
    double p_min = 0.0;
    double p_avg = 0.0;
    double p_max = 0.0;
    std::size_t sample_size = 0;
    std::size_t pair_count = 0;
    std::uint64_t seed = 0;
    std::size_t zero_distance_pairs = 0;
    double time_s = 0.0;
};

inline constexpr std::size_t kDefaultSampleSize = 10000;
inline constexpr std::size_t kDefaultPairBudget = 100000;

namespace detail {
inline std::string flatten(const Msa& msa) {
    std::string flat;
    flat.reserve(msa.rows.size() * msa.width);
    for (const auto& r : msa.rows) flat += r;
    return flat;
}
inline void row_pair(std::string_view a, std::string_view b, const char* what, std::uint32_t* cons,
                     std::uint32_t* mism, std::uint32_t* ham) {
    if (a.size() != b.size()) throw std::invalid_argument(std::string(what) + " requires equal-length rows");
    check(dm_row_pair_stats(ctx(), a.data(), a.size(), b.data(), b.size(), cons, mism, ham));
}
}  // namespace detail

/// distance.hpp (distance.cpp:50-57)
inline std::uint32_t hamming_aligned(std::string_view a, std::string_view b) {
    std::uint32_t c, m, h;
    detail::row_pair(a, b, "hamming_aligned", &c, &m, &h);
    return h;
}

/// metrics.hpp:37-39 (metrics.cpp:16-27)
inline double gap_percent(const Msa& msa) {
    const std::string flat = detail::flatten(msa);
    double v = 0.0;
    detail::check(dm_gap_percent(detail::ctx(), flat.data(), msa.rows.size(), msa.width, &v));
    return v;
}

/// metrics.hpp:41-43 (metrics.cpp:29-45)
inline double p_score(std::string_view a, std::string_view b) {
    std::uint32_t c, m, h;
    detail::row_pair(a, b, "p_score", &c, &m, &h);
    return c == 0 ? 1.0 : static_cast<double>(m) / static_cast<double>(c);
}

/// metrics.hpp:45-49 (metrics.cpp:47-56)
inline double distortion_pair(std::string_view a_aligned, std::string_view b_aligned, std::string_view a_raw,
                              std::string_view b_raw) {
    const std::uint32_t lev = levenshtein(a_raw, b_raw);
    if (lev == 0) throw std::invalid_argument("distortion is undefined for identical sequences");
    return static_cast<double>(hamming_aligned(a_aligned, b_aligned)) / static_cast<double>(lev);
}

/// metrics.hpp:51-56 (metrics.cpp:84-169); the pair sweep runs on the GPU.
inline MetricsReport evaluate(const Msa& msa, std::span<const std::string_view> raws, std::size_t sample_size,
                              std::size_t pair_budget, std::uint64_t seed, ThreadPool&) {
    const std::string flat = detail::flatten(msa);
    std::string raw;
    std::vector<std::uint64_t> off{0};
    for (auto r : raws) {
        raw += r;
        off.push_back(raw.size());
    }
    dm_metrics m{};
    detail::check(dm_evaluate(detail::ctx(), flat.data(), msa.rows.size(), msa.width, msa.row_to_sequence.data(),
                              raw.data(), off.data(), static_cast<std::uint32_t>(raws.size()), sample_size,
                              pair_budget, seed, &m));
    MetricsReport r;
    r.width = m.width;
    r.stretch = m.stretch;
    r.gap_percent = m.gap_percent;
    r.distortion = m.distortion;
    r.p_min = m.p_min;
    r.p_avg = m.p_avg;
    r.p_max = m.p_max;
    r.sample_size = m.sample_size;
    r.pair_count = m.pair_count;
    r.seed = m.seed;
    r.zero_distance_pairs = m.zero_distance_pairs;
    return r;
}

}  // namespace divmsa
