// extern "C" boundary, part 2: pairwise aligner and MSA builder.
#include <algorithm>
#include <cstring>
#include <string>

#include "capi_guard.h"
#include "host_par.h"
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include "nw.h"
#include "host_copy.h"

// One batch of PairwiseResults (pairwise.hpp:78-84).
struct dm_pw {
    struct One {
        int64_t score = 0;
        std::string a, b;
        std::vector<uint32_t> gaps_a, gaps_b;  // ascending, pre-insertion coordinates
    };
    std::vector<One> r;
};

namespace {
using dm::guard;

// pairwise.cpp:288-297
void check_symbols(const char* s, uint64_t n, const dm::NwScheme& sc, const char* which) {
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned char c = (unsigned char)s[i];
        if (c >= 128 || !sc.has[c])
            throw dm::invalid_argument(std::string("sequence ") + which + " contains symbol '" + (char)c +
                                       "' absent from the substitution table");
    }
}

// s with a '-' inserted before residue asc[p] for each p (asc ascending; a
// value n appends at the end), as runs of memcpy between the gaps
std::string with_gaps(const char* s, uint64_t n, const std::vector<uint32_t>& asc) {
    std::string out(n + asc.size(), '-');
    char* o = out.data();
    uint64_t c = 0;
    for (const uint32_t g : asc) {
        const uint64_t upto = std::min<uint64_t>(g, n);
        if (upto > c) {
            std::memcpy(o, s + c, upto - c);
            o += upto - c;
            c = upto;
        }
        ++o;  // the gap (already '-')
    }
    if (n > c) std::memcpy(o, s + c, n - c);
    return out;
}

// A caller-supplied ClusterTree must be a well-formed divisive tree over
// `order` (cluster_tree.hpp:20-45) before the merge scheduler indexes with it.
void validate_tree(const std::vector<dm_node>& nodes, const std::vector<uint32_t>& order, uint32_t n) {
    auto bad = [](const char* why) { throw dm::invalid_argument(std::string("invalid cluster tree: ") + why); };
    if (n == 0 || nodes.size() != 2ull * n - 1) bad("expected 2n-1 nodes");
    std::vector<uint8_t> seen(n, 0);
    for (uint32_t v : order) {
        if (v >= n || seen[v]) bad("order is not a permutation");
        seen[v] = 1;
    }
    if (nodes[0].begin != 0 || nodes[0].end != n) bad("root does not cover every sequence");
    for (size_t v = 0; v < nodes.size(); ++v) {
        const dm_node& nd = nodes[v];
        if (nd.begin >= nd.end || nd.end > n || nd.center >= n) bad("node slice or center out of range");
        if (nd.left < 0 || nd.right < 0) {
            if (nd.left != -1 || nd.right != -1 || nd.end - nd.begin != 1) bad("leaf with children or width != 1");
            continue;
        }
        if ((size_t)nd.left >= nodes.size() || (size_t)nd.right >= nodes.size() || (size_t)nd.left <= v ||
            (size_t)nd.right <= v)
            bad("child index out of range");
        const dm_node& l = nodes[nd.left];
        const dm_node& r = nodes[nd.right];
        if (l.begin != nd.begin || l.end != r.begin || r.end != nd.end) bad("children do not partition the parent");
    }
}

void run_batch(dm_ctx* ctx, const char* A, const uint64_t* a_off, const char* B, const uint64_t* b_off,
               uint32_t njobs, const dm::NwScheme& sc, dm_pw* pw, dm_stats* st) {
    const bool trace = std::getenv("DM_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        DM_CUDA(cudaStreamSynchronize(ctx->stream));
        std::fprintf(stderr, "[dm nw_batch] %s %.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };
    for (uint32_t k = 0; k < njobs; ++k)
        if (a_off[k + 1] == a_off[k] || b_off[k + 1] == b_off[k])
            throw dm::invalid_argument("nw_align requires non-empty inputs");
    const uint64_t abytes = a_off[njobs] - a_off[0], bbytes = b_off[njobs] - b_off[0];
    uint8_t* d_in = (uint8_t*)ctx->rows_b.get(abytes + bbytes + 16);
    dm::upload_host(ctx, d_in, A + a_off[0], abytes, ctx->stream);
    dm::upload_host(ctx, d_in + abytes, B + b_off[0], bbytes, ctx->stream);
    mark("uploaded");
    // symbols (pairwise.cpp:288-297), checked on the uploaded bytes: the first
    // pair in batch order with a bad symbol reports it, a before b
    const uint64_t bad_a = dm::nw_first_bad_symbol(ctx, d_in, abytes, sc.has);
    bool present[128] = {};
    const uint64_t bad_b = dm::nw_first_bad_symbol(ctx, d_in + abytes, bbytes, sc.has, present);
    if (bad_a != UINT64_MAX || bad_b != UINT64_MAX) {
        auto job_of = [](const uint64_t* off, uint32_t nj, uint64_t pos) {  // pair holding byte off[0] + pos
            return (uint32_t)(std::upper_bound(off, off + nj + 1, off[0] + pos) - off - 1);
        };
        const uint32_t ka = bad_a != UINT64_MAX ? job_of(a_off, njobs, bad_a) : UINT32_MAX;
        const uint32_t kb = bad_b != UINT64_MAX ? job_of(b_off, njobs, bad_b) : UINT32_MAX;
        if (ka <= kb) check_symbols(A + a_off[ka], a_off[ka + 1] - a_off[ka], sc, "a");
        else check_symbols(B + b_off[kb], b_off[kb + 1] - b_off[kb], sc, "b");
        throw dm::cuda_error("internal error: symbol check disagrees with the host");
    }
    mark("checked");
    std::vector<dm::NwJob> jobs(njobs);
    for (uint32_t k = 0; k < njobs; ++k) {
        jobs[k].a_off = a_off[k] - a_off[0];
        jobs[k].n = (uint32_t)(a_off[k + 1] - a_off[k]);
        jobs[k].b_off = abytes + (b_off[k] - b_off[0]);
        jobs[k].m = (uint32_t)(b_off[k + 1] - b_off[k]);
    }
    dm::NwScheme scb = sc;  // the column symbols b actually holds (query profiles)
    dm::set_columns(scb, present);
    dm::NwOut no;
    dm::nw_run(ctx, d_in, jobs, scb, no, st != nullptr);
    mark("aligned");
    std::vector<dm::NwRes> res(njobs);
    if (njobs)
        DM_CUDA(cudaMemcpyAsync(res.data(), no.d_res, njobs * sizeof(dm::NwRes), cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    // only the nga + ngb used entries of each job's gap capacity come back
    std::vector<uint32_t> gaps;
    std::vector<uint64_t> goff;
    dm::nw_compact_gaps(ctx, no.d_gaps, jobs, res, gaps, goff);
    mark("gaps back");
    pw->r.resize(njobs);
    dm::host_parallel_for(njobs, 64, [&](uint64_t k) {
        auto& o = pw->r[k];
        o.score = res[k].score;
        const uint32_t* g = gaps.data() + goff[k];
        o.gaps_a.assign(g, g + res[k].nga);
        o.gaps_b.assign(g + res[k].nga, g + res[k].nga + res[k].ngb);
        std::reverse(o.gaps_a.begin(), o.gaps_a.end());  // pairwise.cpp:410-413
        std::reverse(o.gaps_b.begin(), o.gaps_b.end());
        o.a = with_gaps(A + a_off[k], jobs[k].n, o.gaps_a);
        o.b = with_gaps(B + b_off[k], jobs[k].m, o.gaps_b);
    });
    mark("results assembled");
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->kernel_ms = no.fwd_ms + no.tb_ms;
        st->align_ms = no.fwd_ms;
        st->cells = no.cells;
        st->cells_executed = no.cells_exec;
        st->launches = no.launches;
        st->nw_calls = njobs;
    }
}

}  // namespace

extern "C" {

int dm_nw_align(dm_ctx* ctx, const char* a, uint64_t na, const char* b, uint64_t nb, const int16_t* table,
                const uint8_t* has_symbol, int open_surcharge, int gap_extend, dm_pw** out) {
    return guard(ctx, [&] {
        if (!ctx || !table || !has_symbol || !out) throw dm::invalid_argument("null argument");
        const dm::NwScheme sc = dm::make_scheme(table, has_symbol, open_surcharge, gap_extend);
        auto* pw = new dm_pw;
        uint64_t ao[2] = {0, na}, bo[2] = {0, nb};
        try {
            run_batch(ctx, a, ao, b, bo, 1, sc, pw, nullptr);
        } catch (...) {
            delete pw;
            throw;
        }
        *out = pw;
    });
}

int dm_nw_batch(dm_ctx* ctx, const char* A, const uint64_t* a_off, const char* B, const uint64_t* b_off,
                uint32_t njobs, const int16_t* table, const uint8_t* has_symbol, int open_surcharge, int gap_extend,
                dm_pw** out, dm_stats* st) {
    return guard(ctx, [&] {
        if (!ctx || !table || !has_symbol || !out || !a_off || !b_off) throw dm::invalid_argument("null argument");
        const dm::NwScheme sc = dm::make_scheme(table, has_symbol, open_surcharge, gap_extend);
        auto* pw = new dm_pw;
        try {
            run_batch(ctx, A, a_off, B, b_off, njobs, sc, pw, st);
        } catch (...) {
            delete pw;
            throw;
        }
        *out = pw;
    });
}

int64_t dm_pw_score(const dm_pw* p, uint32_t k) { return p->r.at(k).score; }
uint64_t dm_pw_len(const dm_pw* p, uint32_t k) { return p->r.at(k).a.size(); }
int dm_pw_aligned(const dm_pw* p, uint32_t k, char* a_out, char* b_out) {
    const auto& o = p->r.at(k);
    std::memcpy(a_out, o.a.data(), o.a.size());
    std::memcpy(b_out, o.b.data(), o.b.size());
    return DM_OK;
}
uint64_t dm_pw_ngaps_a(const dm_pw* p, uint32_t k) { return p->r.at(k).gaps_a.size(); }
uint64_t dm_pw_ngaps_b(const dm_pw* p, uint32_t k) { return p->r.at(k).gaps_b.size(); }
int dm_pw_gaps(const dm_pw* p, uint32_t k, uint32_t* gaps_a, uint32_t* gaps_b) {
    const auto& o = p->r.at(k);
    if (gaps_a && !o.gaps_a.empty()) std::memcpy(gaps_a, o.gaps_a.data(), o.gaps_a.size() * 4);
    if (gaps_b && !o.gaps_b.empty()) std::memcpy(gaps_b, o.gaps_b.data(), o.gaps_b.size() * 4);
    return DM_OK;
}
void dm_pw_free(dm_pw* p) { delete p; }

int dm_insert_gap_columns(dm_ctx* ctx, const char* rows, uint64_t nrows, uint64_t width, const uint32_t* pos,
                          uint64_t npos, char* out) {
    return guard(ctx, [&] {
        if (!ctx) throw dm::invalid_argument("null context");
        dm::insert_gap_columns(ctx, rows, nrows, width, pos, npos, out);
    });
}

int dm_align_all_progress(dm_ctx* ctx, const dm_seqset* s, const dm_node* nodes, uint64_t nnodes,
                          const uint32_t* order, const int16_t* table, const uint8_t* has_symbol, int open_surcharge,
                          int gap_extend, dm_progress_fn progress, void* user, dm_msa_out** out, dm_stats* st) {
    return guard(ctx, [&] {
        if (!ctx || !s || !nodes || !order || !table || !has_symbol || !out) throw dm::invalid_argument("null argument");
        const dm::NwScheme sc = dm::make_scheme(table, has_symbol, open_surcharge, gap_extend);
        std::vector<dm_node> nv(nodes, nodes + nnodes);
        std::vector<uint32_t> ov(order, order + s->n);
        validate_tree(nv, ov, s->n);
        if (st) std::memset(st, 0, sizeof(*st));
        cudaEvent_t t0, t1;
        DM_CUDA(cudaEventCreate(&t0));
        DM_CUDA(cudaEventCreate(&t1));
        DM_CUDA(cudaEventRecord(t0, ctx->stream));
        dm_msa_out* m = dm::align_all(ctx, s, nv, ov, sc, st, progress, user);
        DM_CUDA(cudaEventRecord(t1, ctx->stream));
        DM_CUDA(cudaEventSynchronize(t1));
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        if (st) {
            st->align_ms = ms;
            st->total_ms = ms;
        }
        *out = m;
    });
}

int dm_align_all(dm_ctx* ctx, const dm_seqset* s, const dm_node* nodes, uint64_t nnodes, const uint32_t* order,
                 const int16_t* table, const uint8_t* has_symbol, int open_surcharge, int gap_extend,
                 dm_msa_out** out, dm_stats* st) {
    return dm_align_all_progress(ctx, s, nodes, nnodes, order, table, has_symbol, open_surcharge, gap_extend,
                                 nullptr, nullptr, out, st);
}

int dm_msa(dm_ctx* ctx, const dm_seqset* s, uint64_t seed, uint64_t exact_cap, const int16_t* table,
           const uint8_t* has_symbol, int open_surcharge, int gap_extend, dm_msa_out** out, dm_stats* st) {
    return guard(ctx, [&] {
        if (!ctx || !s || !table || !has_symbol || !out) throw dm::invalid_argument("null argument");
        const dm::NwScheme sc = dm::make_scheme(table, has_symbol, open_surcharge, gap_extend);
        if (st) std::memset(st, 0, sizeof(*st));
        cudaEvent_t t0, t1, t2;
        DM_CUDA(cudaEventCreate(&t0));
        DM_CUDA(cudaEventCreate(&t1));
        DM_CUDA(cudaEventCreate(&t2));
        DM_CUDA(cudaEventRecord(t0, ctx->stream));
        std::vector<dm_node> nodes;
        std::vector<uint32_t> order;
        dm_stats tree_st{};
        dm::build_tree(ctx, s, seed, exact_cap, nodes, order, st ? &tree_st : nullptr);
        DM_CUDA(cudaEventRecord(t1, ctx->stream));
        dm_stats al_st{};
        dm_msa_out* m = dm::align_all(ctx, s, nodes, order, sc, st ? &al_st : nullptr);
        DM_CUDA(cudaEventRecord(t2, ctx->stream));
        DM_CUDA(cudaEventSynchronize(t2));
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, t0, t1);
        cudaEventElapsedTime(&b, t1, t2);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        cudaEventDestroy(t2);
        if (st) {
            st->tree_ms = a;
            st->align_ms = b;
            st->total_ms = a + b;
            st->cells = tree_st.cells + al_st.cells;
            st->cells_executed = tree_st.cells_executed + al_st.cells;
            st->launches = tree_st.launches + al_st.launches;
            st->kernel_ms = tree_st.kernel_ms + al_st.kernel_ms;
            st->nw_calls = al_st.nw_calls;
            st->lev_calls = tree_st.lev_calls;
        }
        *out = m;
    });
}

uint64_t dm_msa_width(const dm_msa_out* m) { return m->width; }
uint64_t dm_msa_rows(const dm_msa_out* m) { return m->row_seq.size(); }
int dm_msa_copy_rows(const dm_msa_out* m, char* buf) {
    if (!m->rows.empty()) std::memcpy(buf, m->rows.data(), m->rows.size());
    return DM_OK;
}
int dm_msa_copy_row_seq(const dm_msa_out* m, uint32_t* r) {
    std::memcpy(r, m->row_seq.data(), m->row_seq.size() * 4);
    return DM_OK;
}
uint64_t dm_msa_nnodes(const dm_msa_out* m) { return m->nodes.size(); }
int dm_msa_copy_tree(const dm_msa_out* m, dm_node* nodes, uint32_t* order) {
    std::memcpy(nodes, m->nodes.data(), m->nodes.size() * sizeof(dm_node));
    std::memcpy(order, m->order.data(), m->order.size() * 4);
    return DM_OK;
}
void dm_msa_free(dm_msa_out* m) { delete m; }

}  // extern "C"
