// Scoring schemes: the 128x128 int16 table the aligner
// reads, built with the reference's semantics — ScoringScheme
// (pairwise.cpp:59-120), default_nucleotide_scheme (extended IUPAC
// intersection, :20-25, :122-137), default_protein_scheme (BLOSUM62, :27-55,
// :139-142) — including its validation messages (:67-99, :112-115).
#include <cstring>
#include <string>

#include "capi_guard.h"

namespace {

constexpr char kGap = '-';

struct Table {
    int16_t t[128 * 128] = {};
    uint8_t has[128] = {};
};

void set_score(Table& T, char x, char y, int v) {
    if (v < -32768 || v > 32767) throw dm::invalid_argument("substitution score out of range");
    T.t[(unsigned char)x * 128 + (unsigned char)y] = (int16_t)v;
    T.t[(unsigned char)y * 128 + (unsigned char)x] = (int16_t)v;
}

// ScoringScheme constructor semantics (pairwise.cpp:59-108).
void build(Table& T, const char* symbols, size_t n, const int* matrix, int gap_open, int gap_extend) {
    if (n == 0) throw dm::invalid_argument("scoring scheme needs at least one symbol");
    if (!matrix) throw dm::invalid_argument("substitution matrix size does not match symbol count");
    if (gap_open > 0 || gap_extend > 0) throw dm::invalid_argument("gap penalties must be <= 0");
    if (gap_open > gap_extend) throw dm::invalid_argument("gap_open must be <= gap_extend");
    for (size_t i = 0; i < n; ++i) {
        const unsigned char c = (unsigned char)symbols[i];
        if (c >= 128) throw dm::invalid_argument("substitution symbols must be ASCII");
        if (symbols[i] == kGap) throw dm::invalid_argument("the gap symbol cannot appear in the residue alphabet");
        if (T.has[c]) throw dm::invalid_argument(std::string("duplicate symbol '") + symbols[i] + "' in substitution matrix");
        T.has[c] = 1;
    }
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) {
            if (matrix[i * n + j] != matrix[j * n + i])
                throw dm::invalid_argument(std::string("substitution matrix is not symmetric at '") + symbols[i] +
                                           "'/'" + symbols[j] + "'");
            set_score(T, symbols[i], symbols[j], matrix[i * n + j]);
        }
    T.has[(unsigned char)kGap] = 1;
    set_score(T, kGap, kGap, 0);
    for (size_t i = 0; i < n; ++i) set_score(T, kGap, symbols[i], gap_extend);
}

const char kIupacSym[] = "ACGTURYSWKMBDHVN";
const unsigned kIupacMask[16] = {1, 2, 4, 8, 8, 5, 10, 6, 9, 12, 3, 14, 13, 11, 7, 15};
const char kBloSym[] = "ARNDCQEGHILKMFPSTWYVBZX*";
// BLOSUM62, the standard published matrix, row-major over kBloSym.
const signed char kBlo[24][24] = {
    {4, -1, -2, -2, 0, -1, -1, 0, -2, -1, -1, -1, -1, -2, -1, 1, 0, -3, -2, 0, -2, -1, 0, -4},
    {-1, 5, 0, -2, -3, 1, 0, -2, 0, -3, -2, 2, -1, -3, -2, -1, -1, -3, -2, -3, -1, 0, -1, -4},
    {-2, 0, 6, 1, -3, 0, 0, 0, 1, -3, -3, 0, -2, -3, -2, 1, 0, -4, -2, -3, 3, 0, -1, -4},
    {-2, -2, 1, 6, -3, 0, 2, -1, -1, -3, -4, -1, -3, -3, -1, 0, -1, -4, -3, -3, 4, 1, -1, -4},
    {0, -3, -3, -3, 9, -3, -4, -3, -3, -1, -1, -3, -1, -2, -3, -1, -1, -2, -2, -1, -3, -3, -2, -4},
    {-1, 1, 0, 0, -3, 5, 2, -2, 0, -3, -2, 1, 0, -3, -1, 0, -1, -2, -1, -2, 0, 3, -1, -4},
    {-1, 0, 0, 2, -4, 2, 5, -2, 0, -3, -3, 1, -2, -3, -1, 0, -1, -3, -2, -2, 1, 4, -1, -4},
    {0, -2, 0, -1, -3, -2, -2, 6, -2, -4, -4, -2, -3, -3, -2, 0, -2, -2, -3, -3, -1, -2, -1, -4},
    {-2, 0, 1, -1, -3, 0, 0, -2, 8, -3, -3, -1, -2, -1, -2, -1, -2, -2, 2, -3, 0, 0, -1, -4},
    {-1, -3, -3, -3, -1, -3, -3, -4, -3, 4, 2, -3, 1, 0, -3, -2, -1, -3, -1, 3, -3, -3, -1, -4},
    {-1, -2, -3, -4, -1, -2, -3, -4, -3, 2, 4, -2, 2, 0, -3, -2, -1, -2, -1, 1, -4, -3, -1, -4},
    {-1, 2, 0, -1, -3, 1, 1, -2, -1, -3, -2, 5, -1, -3, -1, 0, -1, -3, -2, -2, 0, 1, -1, -4},
    {-1, -1, -2, -3, -1, 0, -2, -3, -2, 1, 2, -1, 5, 0, -2, -1, -1, -1, -1, 1, -3, -1, -1, -4},
    {-2, -3, -3, -3, -2, -3, -3, -3, -1, 0, 0, -3, 0, 6, -4, -2, -2, 1, 3, -1, -3, -3, -1, -4},
    {-1, -2, -2, -1, -3, -1, -1, -2, -2, -3, -3, -1, -2, -4, 7, -1, -1, -4, -3, -2, -2, -1, -2, -4},
    {1, -1, 1, 0, -1, 0, 0, 0, -1, -2, -2, 0, -1, -2, -1, 4, 1, -3, -2, -2, 0, 0, 0, -4},
    {0, -1, 0, -1, -1, -1, -1, -2, -2, -1, -1, -1, -1, -2, -1, 1, 5, -2, -2, 0, -1, -1, 0, -4},
    {-3, -3, -4, -4, -2, -2, -3, -2, -2, -3, -2, -3, -1, 1, -4, -3, -2, 11, 2, -3, -4, -3, -2, -4},
    {-2, -2, -2, -3, -2, -1, -2, -3, 2, -1, -1, -2, -1, 3, -3, -2, -2, 2, 7, -1, -3, -2, -1, -4},
    {0, -3, -3, -3, -1, -2, -2, -3, -3, 3, 1, -2, 1, -1, -2, -2, 0, -3, -1, 4, -3, -2, -1, -4},
    {-2, -1, 3, 4, -3, 0, 1, -1, 0, -3, -4, 0, -3, -3, -2, 0, -1, -4, -3, -3, 4, 1, -1, -4},
    {-1, 0, 0, 1, -3, 3, 4, -2, 0, -3, -3, 1, -1, -3, -1, 0, -1, -3, -2, -2, 1, 4, -1, -4},
    {0, -1, -1, -1, -2, -1, -1, -1, -1, -1, -1, -1, -1, -1, -2, 0, 0, -2, -1, -1, -1, -1, -1, -4},
    {-4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, 1},
};

void emit(const Table& T, int gap_open, int flat, int16_t* table, uint8_t* has, int* open_surcharge) {
    std::memcpy(table, T.t, sizeof(T.t));
    std::memcpy(has, T.has, sizeof(T.has));
    if (open_surcharge) *open_surcharge = flat ? 0 : gap_open;  // pairwise.hpp:36-38
}

}  // namespace

extern "C" {

// kind 0: default_nucleotide_scheme, 1: default_protein_scheme.
int dm_scheme_default(int kind, int gap_open, int gap_extend, int flat, int16_t* table, uint8_t* has_symbol,
                      int* open_surcharge) {
    return dm::guard([&] {
        dm::require(table && has_symbol, "null argument");
        Table T;
        if (kind == 0) {
            int m[16 * 16];
            for (int i = 0; i < 16; ++i)
                for (int j = 0; j < 16; ++j) m[i * 16 + j] = (kIupacMask[i] & kIupacMask[j]) ? 1 : -1;
            build(T, kIupacSym, 16, m, gap_open, gap_extend);
        } else if (kind == 1) {
            int m[24 * 24];
            for (int i = 0; i < 24; ++i)
                for (int j = 0; j < 24; ++j) m[i * 24 + j] = kBlo[i][j];
            build(T, kBloSym, 24, m, gap_open, gap_extend);
        } else {
            throw dm::invalid_argument("unknown built-in scheme");
        }
        emit(T, gap_open, flat, table, has_symbol, open_surcharge);
    });
}

// ScoringScheme(symbols, matrix, gap_open, gap_extend, mode); optional gap
// column overrides (parse_scoring_matrix, pairwise.cpp:243-250): gap_scores
// (length nsym, may be NULL) sets score('-', symbols[i]).
int dm_scheme_custom(const char* symbols, uint32_t nsym, const int* matrix, int gap_open, int gap_extend, int flat,
                     const int* gap_scores, int gap_gap, int16_t* table, uint8_t* has_symbol, int* open_surcharge) {
    return dm::guard([&] {
        dm::require(table && has_symbol, "null argument");
        Table T;
        build(T, symbols, nsym, matrix, gap_open, gap_extend);
        if (gap_scores) {
            for (uint32_t i = 0; i < nsym; ++i) set_score(T, kGap, symbols[i], gap_scores[i]);
            set_score(T, kGap, kGap, gap_gap);
        }
        emit(T, gap_open, flat, table, has_symbol, open_surcharge);
    });
}

}  // extern "C"
