// GPU drop-in for the reference's include/divmsa/cluster_tree.hpp
// (/root/reference/proj/include/divmsa/cluster_tree.hpp:16-74): the same
// node/tree structs and functions; geometric_median and build_tree run on
// libdmb200 (distance engine + level-batched divisive builder), dump_tree
// formats the reference's NDJSON (nlohmann key order) in the library.
#pragma once

#include <algorithm>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <iosfwd>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "divmsa/b200_runtime.hpp"
#include "divmsa/parallel.hpp"  // the reference's ThreadPool (host work only here)

namespace divmsa {

inline constexpr std::uint32_t kNoSequence = 0xffffffffu;
inline constexpr std::size_t kMedianExactCap = 100;

/// cluster_tree.hpp:20-34 (layout mirrors dm_node, handed to the library as is)
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

/// cluster_tree.hpp:36-45 (leaf_count / max_depth: cluster_tree.cpp:236-250)
struct ClusterTree {
    std::vector<ClusterNode> nodes;
    std::vector<std::uint32_t> order;

    std::span<const std::uint32_t> members(const ClusterNode& node) const {
        return std::span(order).subspan(node.begin, node.size());
    }
    std::size_t leaf_count() const {
        return static_cast<std::size_t>(
            std::count_if(nodes.begin(), nodes.end(), [](const ClusterNode& n) { return n.is_leaf(); }));
    }
    std::uint32_t max_depth() const {
        std::uint32_t d = 0;
        for (const ClusterNode& n : nodes) d = std::max(d, n.depth);
        return d;
    }
};

/// cluster_tree.hpp:47-50
struct TreeBuildOptions {
    std::uint64_t seed = 42;
    std::size_t median_exact_cap = kMedianExactCap;
};

/// cluster_tree.hpp:56-59 (cluster_tree.cpp:115-166)
inline std::uint32_t geometric_median(std::span<const std::uint32_t> members, std::span<const std::string_view> seqs,
                                      std::uint64_t seed, std::size_t exact_cap, ThreadPool& /*pool*/) {
    if (members.empty()) throw std::invalid_argument("geometric_median of an empty member set");
    auto s = b200::upload(seqs);
    std::uint32_t out = 0;
    b200::check(dm_geometric_median(b200::ctx(), s.get(), members.data(), members.size(), seed, exact_cap, &out));
    return out;
}

/// cluster_tree.hpp:66-67 (cluster_tree.cpp:168-235): every level's median
/// candidates, distance sweeps and splits as GPU batches; same nodes, same
/// BFS numbering, same order permutation, same errors.
inline ClusterTree build_tree(std::span<const std::string_view> seqs, const TreeBuildOptions& options,
                              ThreadPool& /*pool*/) {
    if (seqs.empty()) throw std::runtime_error("cannot build a cluster tree from zero sequences");
    auto s = b200::upload(seqs);
    ClusterTree t;
    t.nodes.resize(2 * seqs.size() - 1);
    t.order.resize(seqs.size());
    std::uint64_t nn = 0;
    b200::check(dm_build_tree(b200::ctx(), s.get(), options.seed, options.median_exact_cap,
                              reinterpret_cast<dm_node*>(t.nodes.data()), &nn, t.order.data(), nullptr));
    t.nodes.resize(nn);
    return t;
}

/// cluster_tree.hpp:70-71 (cluster_tree.cpp:253-270)
inline void dump_tree(const ClusterTree& tree, std::span<const std::string> ids, std::ostream& out) {
    std::string flat;
    std::vector<std::uint64_t> off{0};
    for (const std::string& id : ids) {
        flat += id;
        off.push_back(flat.size());
    }
    char* text = nullptr;
    std::uint64_t len = 0;
    b200::check(dm_format_tree(reinterpret_cast<const dm_node*>(tree.nodes.data()), tree.nodes.size(), flat.data(),
                               off.data(), ids.size(), &text, &len));
    out.write(text, static_cast<std::streamsize>(len));
    dm_free(text);
}

/// cluster_tree.hpp:72-73 (cluster_tree.cpp:272-280)
inline void dump_tree(const ClusterTree& tree, std::span<const std::string> ids, const std::filesystem::path& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open tree dump file: " + path.string());
    dump_tree(tree, ids, out);
    if (!out.flush()) throw std::runtime_error("failed writing tree dump: " + path.string());
}

}  // namespace divmsa
