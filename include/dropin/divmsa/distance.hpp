// GPU drop-in for the reference's include/divmsa/distance.hpp
// (/root/reference/proj/include/divmsa/distance.hpp:8-16): same declarations,
// bodies on libdmb200 (include/dm_b200.h). Put include/dropin ahead of the
// reference's include/ on the include path.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string_view>

#include "divmsa/b200_runtime.hpp"

namespace divmsa {

/// distance.hpp:11 (distance.cpp:9-48): exact Levenshtein distance, computed
/// by the bit-parallel distance engine (any length).
inline std::uint32_t levenshtein(std::string_view a, std::string_view b) {
    int st = 0;
    const std::uint32_t d = dm_levenshtein(b200::ctx(), a.data(), a.size(), b.data(), b.size(), &st);
    b200::check(st);
    return d;
}

/// distance.hpp:16 (distance.cpp:50-57): differing columns of two equal-length
/// gapped rows.
inline std::uint32_t hamming_aligned(std::string_view a, std::string_view b) {
    if (a.size() != b.size()) throw std::invalid_argument("hamming_aligned requires equal-length rows");
    std::uint32_t considered = 0, mismatched = 0, hamming = 0;
    b200::check(dm_row_pair_stats(b200::ctx(), a.data(), a.size(), b.data(), b.size(), &considered, &mismatched,
                                  &hamming));
    return hamming;
}

}  // namespace divmsa
