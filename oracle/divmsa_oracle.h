/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference (divmsa) hot path, written from the
 * reference's documented behaviour and pinned against its known-answer tests
 * and the compiled reference itself (oracle/_ref, see oracle/Makefile).
 * Each function cites the reference lines it restates; paths are relative to
 * /root/reference/proj. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may call it.
 */
#ifndef DIVMSA_ORACLE_H
#define DIVMSA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:14-23 */
uint64_t orc_mix_seed(uint64_t x);
uint64_t orc_combine_seed(uint64_t seed, uint64_t salt);

/* std::mt19937_64 (the engine rng.hpp and cluster_tree.cpp:134 use). */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);

/* rng.hpp:27-35 */
uint64_t orc_bounded_draw(orc_mt64* g, uint64_t bound);
/* rng.hpp:39-59: k distinct of [0,n), sorted ascending; returns count written. */
uint64_t orc_sample_distinct(orc_mt64* g, uint64_t n, uint64_t k, uint64_t* out);

/* distance.cpp:9-48 */
uint32_t orc_levenshtein(const char* a, size_t na, const char* b, size_t nb);

/* cluster_tree.cpp:18-27 */
uint64_t orc_hash_members(const uint32_t* members, size_t n);

/* cluster_tree.cpp:115-166; returns 0 or -1 on empty members. */
int orc_geometric_median(const uint32_t* members, size_t n, const char* const* seqs,
                         const uint32_t* lens, uint64_t seed, size_t exact_cap,
                         uint32_t* out);

/* One ClusterNode (cluster_tree.hpp:20-34). */
typedef struct {
    uint32_t begin, end, center, radius, pole_l, pole_r;
    int32_t left, right, parent;
    uint32_t depth;
} orc_node;

/* cluster_tree.cpp:168-235. nodes: capacity 2n-1. Returns 0, 1 (empty input)
 * or 2 (pole_l == pole_r: "input was not de-duplicated", :89-92). */
int orc_build_tree(const char* const* seqs, const uint32_t* lens, size_t n,
                   uint64_t seed, size_t exact_cap, orc_node* nodes, size_t* nnodes,
                   uint32_t* order);

/* Scoring tables (pairwise.cpp:20-55, :59-142): 128x128 int16 indexed by char. */
void orc_nucleotide_table(int gap_extend, int16_t* table);
void orc_protein_table(int gap_extend, int16_t* table);

/* pairwise.cpp:301-415 (nw_align). aligned_a/_b: capacity na+nb; gaps: capacity
 * nb (into a) / na (into b). Returns 0, or 1 on empty input. */
int orc_nw_align(const char* a, size_t na, const char* b, size_t nb,
                 const int16_t* table, int open_surcharge, int gap_extend,
                 int64_t* score, char* aligned_a, char* aligned_b, size_t* aligned_len,
                 uint32_t* gaps_a, size_t* ngaps_a, uint32_t* gaps_b, size_t* ngaps_b);

/* msa_merge.cpp:31-70. rows: nrows x width; out: nrows x (width+npos).
 * Returns 0, 1 (position exceeds width) or 2 (unsorted). */
int orc_insert_gap_columns(const char* rows, size_t nrows, size_t width,
                           const uint32_t* pos, size_t npos, char* out);

/* msa_merge.cpp:107-158 (align_all) over a tree from orc_build_tree.
 * rows_out: n x width (malloc'd by callee; free with orc_free). Row r carries
 * sequence order[r] (test_msa_merge.cpp:198). */
int orc_align_all(const orc_node* nodes, size_t nnodes, const uint32_t* order,
                  const char* const* seqs, const uint32_t* lens, size_t n,
                  const int16_t* table, int open_surcharge, int gap_extend,
                  char** rows_out, size_t* width_out);
void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
