// align_sequences core shared by the C ABI entry points (pipeline.cpp,
// fasta.cu).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "dm_internal.h"

namespace dm {

struct AlignCore {
    std::unique_ptr<dm_msa_out> msa;   // unique rows in tree order (rows also in ctx->rows_a, dev_pitch)
    std::vector<uint32_t> slot_input;  // output slot -> input record index
    std::vector<uint32_t> slot_row;    // output slot -> MSA row (duplicates share their representative's)
    dm_align_summary summary{};
    std::vector<uint32_t> reps;               // input index of each distinct sequence (tree leaf ids)
    std::vector<std::vector<uint32_t>> dups;  // input indices collapsed onto each representative
};

AlignCore align_core(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                     const std::vector<std::string>* ids, int alphabet, int gap_open, int gap_extend, int flat,
                     const int16_t* custom_table, const uint8_t* custom_has, uint64_t seed, int input_order,
                     dm_stats* st, bool host_rows = true);

}  // namespace dm
