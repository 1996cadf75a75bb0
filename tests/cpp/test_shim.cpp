// C++ drop-in check: the reference's own known-answer tests, restated against
// include/divmsa_b200.hpp (namespace divmsa on libdmb200.so). Sources of the
// pins: /root/reference/proj/tests/test_distance.cpp:11-28,
// test_pairwise.cpp:137-186, test_cluster_tree.cpp:115-221,
// test_msa_merge.cpp:79-176.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "divmsa_b200.hpp"

using namespace divmsa;

static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
            ++failures;                                                    \
        }                                                                  \
    } while (0)
template <class E, class F>
static bool throws(F&& f, const char* needle = nullptr) {
    try {
        f();
    } catch (const E& e) {
        return !needle || std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    CHECK(levenshtein("KITTEN", "SITTING") == 3);
    CHECK(levenshtein("", "") == 0);
    CHECK(levenshtein("A", "") == 1);
    CHECK(levenshtein("", "ACGT") == 4);
    CHECK(levenshtein("AC", "CA") == 2);
    CHECK(levenshtein("XXXABC", "ABC") == 3);

    const auto affine = default_nucleotide_scheme();
    CHECK(affine.score('A', 'R') == 1 && affine.score('A', 'Y') == -1 && affine.score('-', '-') == 0);
    CHECK(default_protein_scheme().score('W', 'W') == 11);
    {
        const auto r = nw_align("ACGT", "AGT", affine);
        CHECK(r.score == -8 && r.aligned_a == "ACGT" && r.aligned_b == "A-GT");
        CHECK(r.gaps_into_a.empty() && r.gaps_into_b == std::vector<std::uint32_t>{1});
    }
    {
        const auto r = nw_align("AA", "A", affine);
        CHECK(r.score == -10 && r.aligned_b == "-A" && r.gaps_into_b == std::vector<std::uint32_t>{0});
    }
    {
        const auto r = nw_align("A-G", "AG", affine);
        CHECK(r.score == -9 && r.aligned_b == "A-G");
        CHECK(nw_align("A-G", "A-G", affine).score == 2);
    }
    CHECK(nw_align("ACGT", "AGT", default_nucleotide_scheme(-10, -1, GapMode::Flat)).score == 2);
    CHECK(throws<std::invalid_argument>([&] { nw_align("", "A", affine); }));
    CHECK(throws<std::invalid_argument>([&] { nw_align("AQ", "A", affine); }));
    const std::vector<int> asym{1, -1, -2, 1};
    CHECK(throws<std::invalid_argument>([&] { ScoringScheme("AC", asym, -5, -1, GapMode::Affine); }, "not symmetric"));

    ThreadPool pool(2);
    {
        const std::vector<std::string_view> seqs{"AAAA", "AAAT", "TTTT"};
        const std::vector<std::uint32_t> members{0, 1, 2};
        CHECK(geometric_median(members, seqs, 42, kMedianExactCap, pool) == 1);
        const auto tree = build_tree(seqs, {}, pool);
        const ClusterNode& root = tree.nodes[0];
        CHECK(root.center == 1 && root.pole_l == 2 && root.pole_r == 0 && root.radius == 3);
        const auto lm = tree.members(tree.nodes[root.left]);
        CHECK(lm.size() == 1 && lm[0] == 2);
        CHECK(tree.leaf_count() == 3 && tree.nodes.size() == 5);
        const Msa m = align_all(tree, seqs, affine, pool);
        CHECK(m.row_to_sequence == tree.order && m.rows.size() == 3);
    }
    {
        const std::vector<std::string_view> dup{"ACGT", "ACGT", "TTTT"};
        CHECK(throws<std::runtime_error>([&] { build_tree(dup, {}, pool); }, "de-duplicated"));
    }
    {
        Msa m;
        m.rows = {"AC", "GT"};
        m.row_to_sequence = {0, 1};
        m.width = 2;
        const std::vector<std::uint32_t> p{1};
        const Msa o = insert_gap_columns(m, p, pool);
        CHECK(o.rows == (std::vector<std::string>{"A-C", "G-T"}) && o.width == 3);
        Msa ab;
        ab.rows = {"AB"};
        ab.row_to_sequence = {0};
        ab.width = 2;
        const std::vector<std::uint32_t> p2{0, 0, 2};
        CHECK(insert_gap_columns(ab, p2, pool).rows[0] == "--AB-");
        const std::vector<std::uint32_t> p3{3};
        CHECK(throws<std::invalid_argument>([&] { insert_gap_columns(ab, p3, pool); }, "width"));
    }
    {
        // merge ACGT + AGT through a two-leaf tree (test_msa_merge.cpp:146-163)
        const std::vector<std::string_view> seqs{"ACGT", "AGT"};
        ClusterTree t;
        t.order = {0, 1};
        t.nodes.resize(3);
        t.nodes[0] = ClusterNode{0, 2, 0, 0, kNoSequence, kNoSequence, 1, 2, -1, 0};
        t.nodes[1] = ClusterNode{0, 1, 0, 0, kNoSequence, kNoSequence, -1, -1, 0, 1};
        t.nodes[2] = ClusterNode{1, 2, 1, 0, kNoSequence, kNoSequence, -1, -1, 0, 1};
        const Msa p = merge(t, t.nodes[0], align_leaf(t.nodes[1], seqs), align_leaf(t.nodes[2], seqs), affine, pool);
        CHECK(p.width == 4 && p.rows[0] == "ACGT" && p.rows[1] == "A-GT");
    }
    {
        // metrics (test_metrics.cpp:74-128)
        Msa m;
        m.rows = {"AC-T", "AG-T"};
        m.row_to_sequence = {0, 1};
        m.width = 4;
        CHECK(std::abs(gap_percent(m) - 25.0) < 1e-12);
        CHECK(std::abs(p_score("AC-T", "AG-T") - 1.0 / 3) < 1e-12 && p_score("A---", "-CCC") == 1.0);
        CHECK(hamming_aligned("ACGT", "A-GT") == 1);
        CHECK(distortion_pair("AC--", "--GT", "AC", "GT") == 2.0);
        CHECK(throws<std::invalid_argument>([&] { p_score("AC", "A"); }, "equal-length"));
        CHECK(throws<std::invalid_argument>([&] { distortion_pair("ACGT", "ACGT", "ACGT", "ACGT"); }, "identical"));
        const std::vector<std::string_view> raws{"ACT", "AGT"};
        const MetricsReport r = evaluate(m, raws, 100, 100, 42, pool);
        CHECK(r.width == 4 && r.sample_size == 2 && r.pair_count == 1 && r.seed == 42);
        CHECK(std::abs(r.stretch - 4.0 / 3) < 1e-12 && std::abs(r.p_avg - 1.0 / 3) < 1e-12 && r.distortion == 1.0);
        CHECK(throws<std::invalid_argument>([&] { evaluate(Msa{}, raws, 10, 10, 1, pool); }, "empty alignment"));
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "all shim checks passed", failures);
    return failures ? 1 : 0;
}
