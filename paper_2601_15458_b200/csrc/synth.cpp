// Seeded synthetic inputs for the five BASELINE configs (SURVEY.md
// Appendix C). They stand in for the paper's GreenGenes / PDB / Pfam corpora
// (PAPER.md:219-241), which are not available; only shapes, lengths and
// mutation processes are modelled.
//
// RNG primitives follow the reference's portable draws: std::mt19937_64 with
// rejection-sampled bounded draws (rng.hpp:27-35), uniform doubles
// (x >> 11) * 2^-53, geometric lengths k=1; while (u >= 1/mu) ++k.
// cfg1 pairs are generated in parallel, pair i from its own engine seeded
// with combine_seed(S_1, i) (rng.hpp:21-23), so the set is independent of the
// thread count.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "dm_b200.h"
#include "rng.h"

namespace {

using dm::rng::combine_seed;

struct Rng {
    std::mt19937_64 g;
    explicit Rng(uint64_t s) : g(s) {}
    uint64_t bounded(uint64_t bound) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t v;
        do v = g(); while (v >= limit);
        return v % bound;
    }
    double u() { return (double)(g() >> 11) * (1.0 / 9007199254740992.0); }
    uint32_t geom(double mean) {
        uint32_t k = 1;
        while (u() >= 1.0 / mean) ++k;
        return k;
    }
};

struct Law {
    bool protein = false;
    char draw(Rng& r) const {
        if (!protein) return "ACGT"[r.bounded(4)];
        // background weights w_k = 20 - k over ARNDCQEGHILKMFPSTWYV (sum 210)
        static const char kAA[] = "ARNDCQEGHILKMFPSTWYV";
        const uint64_t t = r.bounded(210);
        uint64_t cum = 0;
        for (int k = 0; k < 20; ++k) {
            cum += 20 - k;
            if (cum > t) return kAA[k];
        }
        return kAA[19];
    }
};

struct Rates {
    double sub, ins, del, mean;
};

std::string random_seq(Rng& r, const Law& law, size_t len) {
    std::string s(len, 'A');
    for (auto& c : s) c = law.draw(r);
    return s;
}

std::string evolve(Rng& r, const Law& law, const std::string& s, const Rates& k) {
    std::string out;
    out.reserve(s.size() + s.size() / 16 + 8);
    size_t i = 0;
    while (i < s.size()) {
        if (r.u() < k.del) {
            i += r.geom(k.mean);
            continue;
        }
        char c = s[i];
        if (r.u() < k.sub) {
            char d;
            do d = law.draw(r); while (d == c);
            c = d;
        }
        out.push_back(c);
        if (r.u() < k.ins) {
            const uint32_t g = r.geom(k.mean);
            for (uint32_t t = 0; t < g; ++t) out.push_back(law.draw(r));
        }
        ++i;
    }
    if (out.empty()) out.push_back(law.draw(r));
    return out;
}

void yule(Rng& r, const Law& law, size_t leaves_wanted, size_t root_len, const Rates& k,
          std::vector<std::string>& out) {
    std::vector<std::string> leaves{random_seq(r, law, root_len)};
    while (leaves.size() < leaves_wanted) {
        const size_t idx = r.bounded(leaves.size());
        const std::string p = leaves[idx];
        leaves[idx] = evolve(r, law, p, k);
        leaves.push_back(evolve(r, law, p, k));
    }
    for (auto& s : leaves) out.push_back(std::move(s));
}

}  // namespace

extern "C" int dm_synth(int cfg, double scale, uint64_t seed, char** data, uint64_t** offsets,
                        uint64_t* n) {
    if (cfg < 0 || cfg > 4 || !(scale > 0) || !data || !offsets || !n) return DM_EINVAL;
    const uint64_t S = seed ? seed : 2601154580ULL + (uint64_t)cfg;
    auto scaled = [&](double full) { return std::max<size_t>(2, (size_t)(full * scale + 0.5)); };
    std::vector<std::string> seqs;
    const Law dna{false}, aa{true};
    if (cfg == 0) {
        Rng r(S);
        yule(r, dna, scaled(1000), 300, {0.02, 0.005, 0.005, 3.0}, seqs);
    } else if (cfg == 1) {
        const size_t pairs = scaled(1000000);
        seqs.resize(2 * pairs);
        unsigned nt = std::max(1u, std::thread::hardware_concurrency());
        nt = std::min<unsigned>(nt, 64);
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (size_t i = t; i < pairs; i += nt) {
                    Rng r(combine_seed(S, i));
                    const size_t L = 500 + r.bounded(1001);
                    seqs[2 * i] = random_seq(r, dna, L);
                    seqs[2 * i + 1] = evolve(r, dna, seqs[2 * i], {0.05, 0.005, 0.005, 3.0});
                }
            });
        for (auto& x : th) x.join();
    } else if (cfg == 2) {
        Rng r(S);
        yule(r, dna, scaled(10000), 1500, {0.03, 0.004, 0.004, 3.0}, seqs);
    } else if (cfg == 3) {
        Rng r(S);
        yule(r, aa, scaled(20000), 350, {0.10, 0.005, 0.005, 2.0}, seqs);
    } else {
        const size_t per = scaled(2000);
        for (uint64_t c = 0; c < 50; ++c) {
            Rng r(combine_seed(S, c));
            yule(r, dna, per, 1500, {0.03, 0.004, 0.004, 3.0}, seqs);
        }
    }
    uint64_t total = 0;
    for (auto& s : seqs) total += s.size();
    char* d = (char*)std::malloc(total + 1);
    uint64_t* o = (uint64_t*)std::malloc((seqs.size() + 1) * sizeof(uint64_t));
    if (!d || !o) {
        std::free(d);
        std::free(o);
        return DM_ENOMEM;
    }
    uint64_t p = 0;
    for (size_t i = 0; i < seqs.size(); ++i) {
        o[i] = p;
        std::memcpy(d + p, seqs[i].data(), seqs[i].size());
        p += seqs[i].size();
    }
    o[seqs.size()] = p;
    *data = d;
    *offsets = o;
    *n = seqs.size();
    return DM_OK;
}
