// The reference's file pipeline (pipeline.cpp run_align, compiled unmodified
// from /root/reference/proj/src) linked against the GPU drop-in headers:
//   run_align_b200 IN.fa OUT.fa [--alphabet auto|nt|aa] [--gap-open N]
//                  [--gap-extend N] [--flat] [--seed N] [--order tree|input]
//                  [--dump-tree PATH] [--dump-dedup PATH] [--matrix PATH]
// prints the AlignSummary JSON (pipeline.cpp AlignSummary::to_json).
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "divmsa/pipeline.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s IN.fa OUT.fa [options]\n", argv[0]);
        return 2;
    }
    divmsa::RunConfig cfg;
    for (int i = 3; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
            return argv[++i];
        };
        if (a == "--alphabet") {
            const std::string v = next();
            cfg.alphabet = v == "nt" ? divmsa::AlphabetChoice::Nucleotide
                           : v == "aa" ? divmsa::AlphabetChoice::Protein
                                       : divmsa::AlphabetChoice::Auto;
        } else if (a == "--gap-open") {
            cfg.gap_open = std::atoi(next().c_str());
        } else if (a == "--gap-extend") {
            cfg.gap_extend = std::atoi(next().c_str());
        } else if (a == "--flat") {
            cfg.gap_mode = divmsa::GapMode::Flat;
        } else if (a == "--seed") {
            cfg.seed = std::strtoull(next().c_str(), nullptr, 10);
        } else if (a == "--order") {
            cfg.order = next() == "input" ? divmsa::RowOrder::Input : divmsa::RowOrder::Tree;
        } else if (a == "--dump-tree") {
            cfg.dump_tree_path = next();
        } else if (a == "--dump-dedup") {
            cfg.dump_dedup_path = next();
        } else if (a == "--matrix") {
            cfg.matrix_path = next();
        } else if (a == "--progress") {
            cfg.progress = true;
        } else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 2;
        }
    }
    try {
        const divmsa::AlignSummary s = divmsa::run_align(cfg, argv[1], argv[2]);
        std::printf("%s\n", s.to_json().c_str());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
