// GPU drop-in for the reference's include/divmsa/metrics.hpp
// (/root/reference/proj/include/divmsa/metrics.hpp:11-58): the same
// MetricsReport and functions; the gap census, the sampled row-pair column
// statistics and the pairs' Levenshtein distances run on libdmb200
// (dm_evaluate, csrc/metrics.cu), the report is bit-identical to
// metrics.cpp:84-169. Serialisation (to_json / to_csv_row / csv_header)
// restates metrics.cpp:171-203 on the same nlohmann header the reference
// builds with.
#pragma once

#include <cstdint>
#include <cstdio>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include <json.hpp>

#include "divmsa/b200_runtime.hpp"
#include "divmsa/distance.hpp"
#include "divmsa/msa_merge.hpp"
#include "divmsa/parallel.hpp"

namespace divmsa {

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

    std::string to_json() const {
        nlohmann::json j{
            {"width", width},           {"stretch", stretch},         {"gap_percent", gap_percent},
            {"distortion", distortion}, {"p_min", p_min},             {"p_avg", p_avg},
            {"p_max", p_max},           {"sample_size", sample_size}, {"pair_count", pair_count},
            {"seed", seed},             {"zero_distance_pairs", zero_distance_pairs}, {"time_s", time_s},
        };
        return j.dump();
    }
    std::string to_csv_row() const {
        const auto g6 = [](double v) {
            char buf[64];
            std::snprintf(buf, sizeof(buf), "%.6g", v);
            return std::string(buf);
        };
        return g6(time_s) + "," + std::to_string(width) + "," + g6(stretch) + "," + g6(gap_percent) + "," +
               g6(distortion) + "," + g6(p_min) + "," + g6(p_avg) + "," + g6(p_max);
    }
    static std::string csv_header() { return "time_s,width,stretch,gap_percent,distortion,p_min,p_avg,p_max"; }
};

namespace b200 {
inline std::string flatten(const Msa& msa) {
    std::string flat;
    flat.reserve(msa.rows.size() * msa.width);
    for (const std::string& r : msa.rows) {
        if (r.size() != msa.width) throw std::invalid_argument("alignment rows differ from the alignment width");
        flat += r;
    }
    return flat;
}
}  // namespace b200

/// metrics.hpp:37-39 (metrics.cpp:16-27)
inline double gap_percent(const Msa& msa) {
    if (msa.rows.empty() || msa.width == 0) throw std::invalid_argument("gap_percent of an empty alignment");
    const std::string flat = b200::flatten(msa);
    double v = 0.0;
    b200::check(dm_gap_percent(b200::ctx(), flat.data(), msa.rows.size(), msa.width, &v));
    return v;
}

/// metrics.hpp:41-43 (metrics.cpp:29-45)
inline double p_score(std::string_view a, std::string_view b) {
    if (a.size() != b.size()) throw std::invalid_argument("p_score requires equal-length rows");
    std::uint32_t considered = 0, mismatched = 0, hamming = 0;
    b200::check(dm_row_pair_stats(b200::ctx(), a.data(), a.size(), b.data(), b.size(), &considered, &mismatched,
                                  &hamming));
    return considered == 0 ? 1.0 : static_cast<double>(mismatched) / static_cast<double>(considered);
}

/// metrics.hpp:45-49 (metrics.cpp:47-56)
inline double distortion_pair(std::string_view a_aligned, std::string_view b_aligned, std::string_view a_raw,
                              std::string_view b_raw) {
    const std::uint32_t lev = levenshtein(a_raw, b_raw);
    if (lev == 0) throw std::invalid_argument("distortion is undefined for identical sequences");
    return static_cast<double>(hamming_aligned(a_aligned, b_aligned)) / static_cast<double>(lev);
}

/// metrics.hpp:51-56 (metrics.cpp:84-169): one GPU call for the whole sample.
inline MetricsReport evaluate(const Msa& msa, std::span<const std::string_view> raws, std::size_t sample_size,
                              std::size_t pair_budget, std::uint64_t seed, ThreadPool& /*pool*/) {
    if (msa.rows.empty()) throw std::invalid_argument("cannot evaluate an empty alignment");
    const std::string flat = b200::flatten(msa);
    std::string raw;
    std::vector<std::uint64_t> off{0};
    for (std::string_view r : raws) {
        raw += r;
        off.push_back(raw.size());
    }
    dm_metrics m{};
    b200::check(dm_evaluate(b200::ctx(), flat.data(), msa.rows.size(), msa.width, msa.row_to_sequence.data(),
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

inline constexpr std::size_t kDefaultSampleSize = 10000;
inline constexpr std::size_t kDefaultPairBudget = 100000;

}  // namespace divmsa
