/* dm_b200.h — C ABI of the B200-native MuSAlS hot path (libdmb200.so).
 *
 * Plain pointers and sizes only; no exceptions and no C++/torch types cross
 * this boundary. Every call returns a status (DM_OK = 0); on failure
 * dm_last_error() returns a thread-local message whose text matches the
 * reference exception it replaces (e.g. "...not de-duplicated",
 * "...exceeds alignment width ..."), and the status says which exception
 * type the reference throws: DM_EINVAL <-> std::invalid_argument,
 * DM_ERUNTIME <-> std::runtime_error.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   dm_levenshtein / dm_lev_pairs   divmsa::levenshtein          include/divmsa/distance.hpp:11
 *   dm_lev_one_to_many              distance_scan                src/cluster_tree.cpp:31-41
 *   dm_geometric_median             divmsa::geometric_median     include/divmsa/cluster_tree.hpp:56-59
 *   dm_build_tree                   divmsa::build_tree           include/divmsa/cluster_tree.hpp:66-67
 *   dm_nw_align / dm_nw_batch       divmsa::nw_align             include/divmsa/pairwise.hpp:89-90
 *   dm_insert_gap_columns           divmsa::insert_gap_columns   include/divmsa/msa_merge.hpp:34-35
 *   dm_align_all                    divmsa::align_all            include/divmsa/msa_merge.hpp:47-49
 *   dm_msa                          build_tree + align_all       src/pipeline.cpp:113-128
 * Python FFI that binds these today: python/py_module.cpp:77-155.
 */
#ifndef DM_B200_H
#define DM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DM_OK 0
#define DM_EINVAL 1   /* std::invalid_argument in the reference */
#define DM_ERUNTIME 2 /* std::runtime_error in the reference */
#define DM_ECUDA 3    /* CUDA failure (no device, launch error, ...) */
#define DM_ENOMEM 4

typedef struct dm_ctx dm_ctx;       /* one CUDA device + stream + scratch */
typedef struct dm_seqset dm_seqset; /* device-resident residues + bit-plane profiles */
typedef struct dm_pw dm_pw;         /* one PairwiseResult */
typedef struct dm_msa_out dm_msa_out;

/* Mirrors divmsa::ClusterNode (cluster_tree.hpp:20-34), 40 bytes. */
typedef struct {
    uint32_t begin, end, center, radius, pole_l, pole_r;
    int32_t left, right, parent;
    uint32_t depth;
} dm_node;

/* Per-call device timing and work counters (filled when non-NULL). */
typedef struct {
    double kernel_ms;        /* device time of the hot kernels (CUDA events) */
    double total_ms;         /* device time of the whole call incl. copies */
    uint64_t cells;          /* oracle-equivalent cells: sum |a|*|b| (untrimmed) */
    uint64_t cells_executed; /* cells the kernels actually computed (padding incl.) */
    uint64_t launches;       /* kernels launched */
    double tree_ms, align_ms; /* dm_msa: phase times; dm_nw_*: align_ms = forward-pass kernel time */
    uint64_t lev_calls, nw_calls;
    uint64_t h2d_bytes, d2h_bytes; /* dm_lev_pairs_packed: bytes that crossed PCIe */
    uint64_t cells_reused;   /* guide tree (ABI 2): cells of distance jobs answered from the
                                build's table of pairs already computed (not in `cells`) */
} dm_stats;

const char* dm_last_error(void);
int dm_abi_version(void);

/* ---- context ---------------------------------------------------------- */
/* A context owns a CUDA stream and scratch memory on one device. Calls on one
 * context are serialised by a per-context lock, so a context may be shared by
 * host threads (as the reference's reentrant functions are); dm_ctx_destroy
 * must not race with other calls on the same context. Errors: the status
 * code of the call plus dm_last_error() on the calling thread. */
int dm_ctx_create(int device, dm_ctx** out);
int dm_ctx_destroy(dm_ctx* ctx);
int dm_ctx_sync(dm_ctx* ctx);
/* Issue all further work of ctx on `stream` (a cudaStream_t), e.g. a torch
 * stream, so callers can time with events on their own stream. */
int dm_ctx_set_stream(dm_ctx* ctx, void* stream);
/* INT32 lane-op peak of this device (mode 0 LOP3 (ALU), 1 IMAD (FMA), 2 LOP3+IMAD). */
int dm_int32_peak(dm_ctx* ctx, int mode, double* lane_ops_per_s);
/* Multi-GPU (one process per GPU): rank 0 makes an NCCL unique id, the caller
 * broadcasts its 128 bytes (e.g. torch.distributed), every rank attaches.
 * Afterwards dm_build_tree / dm_align_all / dm_msa / dm_align_sequences
 * split the work across the ranks: the top tree levels' distance batches
 * and the top merge levels' NW batches in work-balanced ranges (results
 * all-gathered), and below a split level whole subtrees per rank (tree
 * nodes, order slices and MSA row blocks all-gathered once); every rank
 * ends with the full, identical tree and MSA. */
int dm_nccl_unique_id(uint8_t* id128);
int dm_ctx_attach_nccl(dm_ctx* ctx, const uint8_t* id128, int rank, int world);
/* The same sharded execution with the collectives done by the caller on
 * host memory: fn all-gathers `bytes_per_rank` bytes from every rank into
 * recv (rank order) and returns 0 on success. Lets several processes share
 * one GPU in tests (torch.distributed over gloo), or a caller bring its own
 * transport. */
typedef int (*dm_allgather_fn)(const void* send, void* recv, uint64_t bytes_per_rank, void* user);
int dm_ctx_attach_host_comm(dm_ctx* ctx, int rank, int world, dm_allgather_fn fn, void* user);
/* The shard plan the library uses, for callers and tests: bounds[0..world]
 * splits n jobs of the given costs into contiguous, cost-balanced ranges;
 * owner[i] assigns n whole items to ranks, largest cost first to the least
 * loaded rank (ties to the lower rank). Pure host functions. */
int dm_shard_bounds(const uint64_t* cost, uint64_t n, int world, uint64_t* bounds);
/* Counters of this context since creation: out4 = {collective calls, bytes
 * this rank contributed to them, subtrees it owned in guide trees, subtrees
 * it owned in merge passes}. */
int dm_ctx_comm_stats(dm_ctx* ctx, uint64_t* out4);
int dm_assign_owners(const uint64_t* cost, uint64_t n, int world, int32_t* owner);
/* Run the sharded code path with `world` shards on this one GPU (tests). */
int dm_ctx_simulate_world(dm_ctx* ctx, int world);
/* Record (rank, world) without a communicator (independent shards, e.g. the
 * cfg1 pair batches). */
int dm_ctx_set_shard(dm_ctx* ctx, int rank, int world);

/* ---- sequences -------------------------------------------------------- */
/* Residues of n sequences, concatenated in `data`; sequence i is
 * data[offsets[i], offsets[i+1]). Raw bytes are compared. */
int dm_seqset_create(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                     dm_seqset** out);
int dm_seqset_destroy(dm_seqset* s);
uint32_t dm_seqset_count(const dm_seqset* s);
int dm_seqset_planes(const dm_seqset* s); /* bit-planes used by the distance engine */

/* ---- distance engine (Levenshtein) ------------------------------------ */
uint32_t dm_levenshtein(dm_ctx* ctx, const char* a, uint64_t na, const char* b, uint64_t nb,
                        int* status);
/* out[i] = levenshtein(seq ia[i], seq ib[i]); host arrays. */
int dm_lev_pairs(dm_ctx* ctx, const dm_seqset* s, const uint32_t* ia, const uint32_t* ib,
                 uint64_t n, uint32_t* out, dm_stats* st);
/* Same with DEVICE arrays (ia, ib, out resident in HBM); no host copies. */
int dm_lev_pairs_device(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                        const uint32_t* d_ib, uint64_t n, uint32_t* d_out, dm_stats* st);
/* End-to-end batch from HOST memory: pair i = (sequence 2i, sequence 2i+1)
 * of `data` / `offsets` (2*npairs+1 entries). Uploads and computes in
 * overlapped chunks (copy stream + compute stream). Chunks holding only
 * A/C/G/T bytes cross PCIe as 2-bit codes (packed by host threads into
 * pinned slots); with a pinned `data`, part of the chunks go up raw while
 * the host packs the rest (planned as A/C/G/T, verified on the device,
 * recomputed exactly if the check fails). Results are identical either way.
 * st->h2d_bytes / d2h_bytes report the bytes copied. Env: DM_STREAM_PACK=0
 * disables packing, DM_STREAM_RAW_FRAC sets the raw share, DM_HOST_THREADS
 * sizes the host pool. out: host uint32[npairs]. */
int dm_lev_pairs_packed(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint64_t npairs,
                        uint32_t* out, dm_stats* st);
/* The packer alone (no device needed): residue j of src -> bits 2(j%4).. of
 * dst[j/4], codes A0 C1 G2 T3, last byte zero-padded; DM_EINVAL if src holds
 * any other byte. dst: (n+3)/4 bytes. */
int dm_pack_nt(const char* src, uint64_t n, uint8_t* dst);
/* Per-sequence form, the streamed path's upload layout: sequence i of
 * data[offsets[i], offsets[i+1]) (n sequences) takes 32*ceil(L/128) bytes
 * (residue j at bits 2(j%16) of little-endian 32-bit word j/16, zero pad),
 * back to back; *bytes = total. dst: 32-B aligned, sum of L/4 + 32 bytes
 * suffices. */
int dm_pack_nt_seqs(const char* data, const uint64_t* offsets, uint64_t n, uint8_t* dst, uint64_t* bytes);
/* distance_scan: out[i] = levenshtein(seq from, seq members[i]). */
int dm_lev_one_to_many(dm_ctx* ctx, const dm_seqset* s, uint32_t from, const uint32_t* members,
                       uint64_t n, uint32_t* out, dm_stats* st);
int dm_geometric_median(dm_ctx* ctx, const dm_seqset* s, const uint32_t* members, uint64_t n,
                        uint64_t seed, uint64_t exact_cap, uint32_t* out);

/* ---- quality metrics (divmsa::evaluate, metrics.cpp:84-169) ------------ */
/* Mirrors divmsa::MetricsReport (metrics.hpp:13-35). */
typedef struct {
    uint64_t width;
    double stretch, gap_percent, distortion, p_min, p_avg, p_max;
    uint64_t sample_size, pair_count, seed, zero_distance_pairs;
    double time_s;
} dm_metrics;
/* rows: nrows x width bytes (row r = msa.rows[r]); row_to_sequence[r] indexes
 * the raw sequences (raw, raw_offsets[nraw + 1]). Seeded sampling identical
 * to the reference (sample_size rows, then pair_budget pairs); every field is
 * bit-identical to divmsa::evaluate. DM_EINVAL "cannot evaluate an empty
 * alignment" / "gap_percent of an empty alignment". */
int dm_evaluate(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, const uint32_t* row_to_sequence,
                const char* raw, const uint64_t* raw_offsets, uint32_t nraw, uint64_t sample_size,
                uint64_t pair_budget, uint64_t seed, dm_metrics* out);
/* divmsa::gap_percent (metrics.cpp:16-27). */
int dm_gap_percent(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, double* out);
/* Column counts of two equal-length aligned rows: columns where both carry a
 * residue, mismatches among those (p_score = mismatched / considered, 1.0
 * when considered == 0; metrics.cpp:29-45) and differing columns
 * (hamming_aligned, distance.cpp:50-57). DM_EINVAL on unequal lengths. */
int dm_row_pair_stats(dm_ctx* ctx, const char* a, uint64_t na, const char* b, uint64_t nb, uint32_t* considered,
                      uint32_t* mismatched, uint32_t* hamming);

/* ---- guide tree ------------------------------------------------------- */
/* nodes: capacity 2n-1; order: n. Errors: DM_ERUNTIME "cannot build a cluster
 * tree from zero sequences" / "...input was not de-duplicated". */
int dm_build_tree(dm_ctx* ctx, const dm_seqset* s, uint64_t seed, uint64_t exact_cap,
                  dm_node* nodes, uint64_t* nnodes, uint32_t* order, dm_stats* st);

/* ---- pairwise aligner (Gotoh NW) -------------------------------------- */
/* table: 128x128 int16 indexed by char (ScoringScheme::score, pairwise.hpp:30);
 * has_symbol: 128 flags (ScoringScheme::has_symbol); open_surcharge: gap_open
 * in affine mode, 0 in flat mode (pairwise.hpp:36-38). */
int dm_nw_align(dm_ctx* ctx, const char* a, uint64_t na, const char* b, uint64_t nb,
                const int16_t* table, const uint8_t* has_symbol, int open_surcharge,
                int gap_extend, dm_pw** out);
/* Batched: job k aligns a_k = A[a_off[k], a_off[k+1]) against b_k likewise. */
int dm_nw_batch(dm_ctx* ctx, const char* A, const uint64_t* a_off, const char* B,
                const uint64_t* b_off, uint32_t njobs, const int16_t* table,
                const uint8_t* has_symbol, int open_surcharge, int gap_extend, dm_pw** out,
                dm_stats* st);
int64_t dm_pw_score(const dm_pw* p, uint32_t k);
uint64_t dm_pw_len(const dm_pw* p, uint32_t k);
int dm_pw_aligned(const dm_pw* p, uint32_t k, char* a_out, char* b_out);
uint64_t dm_pw_ngaps_a(const dm_pw* p, uint32_t k);
uint64_t dm_pw_ngaps_b(const dm_pw* p, uint32_t k);
int dm_pw_gaps(const dm_pw* p, uint32_t k, uint32_t* gaps_a, uint32_t* gaps_b);
void dm_pw_free(dm_pw* p);

/* ---- MSA builder ------------------------------------------------------ */
/* rows: nrows x width; out: nrows x (width + npos). Errors as msa_merge.cpp:37-44. */
int dm_insert_gap_columns(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width,
                          const uint32_t* pos, uint64_t npos, char* out);
/* align_all over a tree from dm_build_tree (or the reference). */
int dm_align_all(dm_ctx* ctx, const dm_seqset* s, const dm_node* nodes, uint64_t nnodes,
                 const uint32_t* order, const int16_t* table, const uint8_t* has_symbol,
                 int open_surcharge, int gap_extend, dm_msa_out** out, dm_stats* st);
/* Progress callback of align_all (ProgressFn, msa_merge.hpp:43-49): called
 * once per tree node as it completes, done = 1..nnodes, on the calling
 * thread (leaves first, then each merge level's nodes once that level's
 * alignments are known). */
typedef void (*dm_progress_fn)(uint64_t done, uint64_t total, void* user);
int dm_align_all_progress(dm_ctx* ctx, const dm_seqset* s, const dm_node* nodes, uint64_t nnodes,
                          const uint32_t* order, const int16_t* table, const uint8_t* has_symbol,
                          int open_surcharge, int gap_extend, dm_progress_fn progress, void* user,
                          dm_msa_out** out, dm_stats* st);
/* dump_tree (cluster_tree.hpp:70-72) into memory: the NDJSON text of the
 * tree (one record per node, nlohmann key order), *text malloc'd (dm_free).
 * ids: node centers' names, ids + id_off[k] .. id_off[k+1]. */
int dm_format_tree(const dm_node* nodes, uint64_t nnodes, const char* ids, const uint64_t* id_off, uint64_t nids,
                   char** text, uint64_t* len);
/* build_tree + align_all, device-resident between the two. */
int dm_msa(dm_ctx* ctx, const dm_seqset* s, uint64_t seed, uint64_t exact_cap,
           const int16_t* table, const uint8_t* has_symbol, int open_surcharge,
           int gap_extend, dm_msa_out** out, dm_stats* st);
uint64_t dm_msa_width(const dm_msa_out* m);
uint64_t dm_msa_rows(const dm_msa_out* m);
/* rows in tree order (row r carries sequence order[r]); buf: rows x width. */
int dm_msa_copy_rows(const dm_msa_out* m, char* buf);
int dm_msa_copy_row_seq(const dm_msa_out* m, uint32_t* row_to_sequence);
uint64_t dm_msa_nnodes(const dm_msa_out* m);
int dm_msa_copy_tree(const dm_msa_out* m, dm_node* nodes, uint32_t* order);
void dm_msa_free(dm_msa_out* m);

/* ---- scoring schemes (pairwise.cpp:59-142) ----------------------------- */
/* kind 0: default_nucleotide_scheme (IUPAC), 1: default_protein_scheme
 * (BLOSUM62). Outputs the 128x128 table, the has_symbol flags and the open
 * surcharge (gap_open, or 0 when flat). Validation errors as the reference. */
int dm_scheme_default(int kind, int gap_open, int gap_extend, int flat, int16_t* table,
                      uint8_t* has_symbol, int* open_surcharge);
/* ScoringScheme(symbols, matrix, gap_open, gap_extend, mode); gap_scores
 * (nsym entries, or NULL) overrides score('-', symbol) as a matrix file's
 * gap column does (pairwise.cpp:243-250), gap_gap overrides score('-','-'). */
int dm_scheme_custom(const char* symbols, uint32_t nsym, const int* matrix, int gap_open,
                     int gap_extend, int flat, const int* gap_scores, int gap_gap, int16_t* table,
                     uint8_t* has_symbol, int* open_surcharge);

/* ---- pipeline (align_sequences, pipeline.cpp:78-159) -------------------- */
typedef struct {
    uint64_t input_count, unique_count, duplicate_count;
    uint32_t tree_depth;
    uint64_t width;
    int alphabet; /* 0 nucleotide, 1 protein */
    double elapsed_s;
} dm_align_summary;
/* alphabet: 0 auto, 1 nucleotide, 2 protein. custom_table/custom_has: a
 * scheme from dm_scheme_custom (NULL: built-in for the alphabet; residue
 * validation is skipped for custom schemes, as with --matrix). Record ids in
 * error messages are "seq<i>" (py_module.cpp:134-138). input_order: 1 rows
 * parallel to the input (RowOrder::Input), 0 tree order. rows_out: n x width,
 * free with dm_free. */
int dm_align_sequences(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                       int alphabet, int gap_open, int gap_extend, int flat,
                       const int16_t* custom_table, const uint8_t* custom_has, uint64_t seed,
                       int input_order, char** rows_out, uint64_t* width_out,
                       dm_align_summary* summary, dm_stats* st);

/* ---- FASTA in / out (seq_io.cpp:44-225, pipeline.cpp:160-187) ---------- */
/* divmsa::run_align: parse `input_path` (alphabet 0 auto = structural parse,
 * 1/2 = validate while parsing), align_sequences (record ids in errors),
 * write the aligned FASTA (80-column lines, formatted on the device) to
 * "<output_path>.partial" and rename it into place. input_order: 1 rows in
 * input order, 0 tree order (RowOrder::Tree, the CLI default); non-empty
 * dump paths write the tree NDJSON / the duplicates TSV (RunConfig dump_*).
 * Errors:
 * DM_ERUNTIME with the reference's messages ("<file>:<line>: ..."). */
int dm_run_align(dm_ctx* ctx, const char* input_path, const char* output_path, int alphabet, int gap_open,
                 int gap_extend, int flat, const int16_t* custom_table, const uint8_t* custom_has, uint64_t seed,
                 int input_order, const char* dump_tree_path, const char* dump_dedup_path,
                 dm_align_summary* summary, dm_stats* st);
/* divmsa::dump_tree (cluster_tree.cpp:253-280): NDJSON, one line per node;
 * ids[node.center] names the center. Host I/O. */
int dm_dump_tree(const dm_node* nodes, uint64_t nnodes, const char* ids, const uint64_t* id_off, uint64_t nids,
                 const char* path);
/* divmsa::write_fasta over n records given as packed (data, offsets[n+1])
 * id / description / residue arrays; the text is assembled on the device. */
int dm_write_fasta(dm_ctx* ctx, const char* path, const char* ids, const uint64_t* id_off, const char* descs,
                   const uint64_t* desc_off, const char* residues, const uint64_t* res_off, uint64_t n);
/* divmsa::parse_fasta (alphabet 0 none, 1 nucleotide, 2 protein; allow_gaps =
 * ParseOptions::allow_gaps). Outputs packed arrays, each freed with dm_free. */
int dm_parse_fasta(const char* path, int alphabet, int allow_gaps, char** ids, uint64_t** id_off, char** descs,
                   uint64_t** desc_off, char** residues, uint64_t** res_off, uint64_t* n);

/* ---- synthetic inputs --------------------------- */
/* cfg 0..4 at `scale` (1.0 = full size). Returns concatenated residues +
 * offsets (free with dm_free). For cfg 1, sequence 2i / 2i+1 form pair i. */
int dm_synth(int cfg, double scale, uint64_t seed, char** data, uint64_t** offsets,
             uint64_t* n);
void dm_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
