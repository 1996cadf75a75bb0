// extern "C" boundary of libdmb200.so (include/dm_b200.h). Maps internal
// exceptions onto status codes + a thread-local message, so no C++ exception
// ever crosses the ABI.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "capi_guard.h"
#include "comm.h"

namespace dm {
std::string& last_error() {
    thread_local std::string e;
    return e;
}

void trace_bytes(const char* kernel, uint64_t read, uint64_t written) {
    static const bool on = std::getenv("DM_TRACE_BYTES") != nullptr;
    if (on)
        std::fprintf(stderr, "[dm bytes] %s %llu %llu\n", kernel, (unsigned long long)read,
                     (unsigned long long)written);
}

int occupancy(const void* kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, size_t>, int> occ;
    static std::map<std::pair<const void*, int>, size_t> optin;  // smem limit set per (kernel, device)
    int dev = 0;
    DM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(kern, dev, threads, smem);
    auto it = occ.find(key);
    if (it != occ.end()) return it->second;
    if (smem > 32 * 1024) {  // dynamic + static above 48 KB needs the opt-in
        size_t& lim = optin[{kern, dev}];
        if (smem > lim) {
            DM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            lim = smem;
        }
    }
    int o = 0;
    DM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem));
    if (o < 1) throw runtime_error("kernel does not fit on an SM (" + std::to_string(smem) + " B shared memory)");
    occ[key] = o;
    return o;
}
}  // namespace dm

namespace {
using dm::guard;
using dm::require;
}  // namespace

extern "C" {

const char* dm_last_error(void) { return dm::last_error().c_str(); }
int dm_abi_version(void) { return 2; }

int dm_ctx_create(int device, dm_ctx** out) {
    return guard([&] {
        require(out != nullptr, "null output pointer");
        int count = 0;
        DM_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) throw dm::cuda_error("CUDA device " + std::to_string(device) + " not present");
        DM_CUDA(cudaSetDevice(device));
        auto* c = new dm_ctx;
        c->device = device;
        cudaDeviceProp prop;
        DM_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) {
            delete c;
            throw dm::cuda_error(std::string("libdmb200 is built for sm_100a; device is ") + prop.name);
        }
        c->sm_count = prop.multiProcessorCount;
        {
            size_t fr = 0, tot = 0;
            DM_CUDA(cudaMemGetInfo(&fr, &tot));
            c->free_at_create = fr;
        }
        // sequence sets are stream-ordered allocations: keep freed memory in the
        // pool so repeated create/destroy (one per batch) never returns to the driver
        cudaMemPool_t pool;
        DM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        DM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        DM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = c->stream;
        {
            int least = 0, greatest = 0;
            DM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            c->side_prio = greatest;
        }
        DM_CUDA(cudaEventCreate(&c->ev0));
        DM_CUDA(cudaEventCreate(&c->ev1));
        dm::lev_warm();
        dm::nw_warm();
        if (const char* sw = std::getenv("DM_SIM_WORLD")) c->sim_world = std::max(1, std::atoi(sw));
        *out = c;
    });
}

int dm_ctx_destroy(dm_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        auto destroy_aux = [](dm_ctx*& p) {  // planner / background contexts
            if (!p) return;
            cudaStreamSynchronize(p->stream);
            for (int k = 0; k < dm_ctx::kLevSide; ++k) {
                if (p->lev_side[k]) {
                    cudaStreamSynchronize(p->lev_side[k]);
                    cudaStreamDestroy(p->lev_side[k]);
                }
                if (p->lev_join[k]) cudaEventDestroy(p->lev_join[k]);
            }
            if (p->lev_fork) cudaEventDestroy(p->lev_fork);
            p->detach_buffers();
            cudaEventDestroy(p->ev0);
            cudaEventDestroy(p->ev1);
            cudaStreamDestroy(p->own_stream);
            delete p;
            p = nullptr;
        };
        for (dm_ctx*& p : ctx->prep) destroy_aux(p);  // planner contexts of the streamed path
        destroy_aux(ctx->tree_bg);
        for (int k = 0; k < dm_ctx::kLevSide; ++k) {
            if (ctx->lev_side[k]) {
                cudaStreamSynchronize(ctx->lev_side[k]);
                cudaStreamDestroy(ctx->lev_side[k]);
            }
            if (ctx->lev_join[k]) cudaEventDestroy(ctx->lev_join[k]);
        }
        if (ctx->lev_fork) cudaEventDestroy(ctx->lev_fork);
        ctx->detach_buffers();  // scratch is freed synchronously once the stream is gone
        dm::comm_destroy(ctx);
        cudaEventDestroy(ctx->ev0);
        for (cudaEvent_t e : ctx->stage_ev)
            if (e) cudaEventDestroy(e);
        cudaEventDestroy(ctx->ev1);
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
        delete ctx;
    });
}

int dm_ctx_sync(dm_ctx* ctx) {
    return guard(ctx, [&] { DM_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int dm_ctx_set_stream(dm_ctx* ctx, void* stream) {
    return guard(ctx, [&] {
        require(ctx != nullptr, "null context");
        DM_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->own_stream) {
            DM_CUDA(cudaStreamDestroy(ctx->own_stream));
            ctx->own_stream = nullptr;
        }
        ctx->stream = static_cast<cudaStream_t>(stream);
    });
}

int dm_int32_peak(dm_ctx* ctx, int mode, double* lane_ops_per_s) {
    return guard(ctx, [&] {
        require(ctx && lane_ops_per_s, "null argument");
        require(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
        *lane_ops_per_s = dm::int32_peak(ctx, mode);
    });
}

int dm_ctx_set_shard(dm_ctx* ctx, int rank, int world) {
    return guard(ctx, [&] {
        require(world >= 1 && rank >= 0 && rank < world, "invalid shard (rank, world)");
        ctx->rank = rank;
        ctx->world = world;
    });
}

int dm_seqset_create(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                     dm_seqset** out) {
    return guard(ctx, [&] {
        require(ctx && out && offsets, "null argument");
        DM_CUDA(cudaSetDevice(ctx->device));
        *out = dm::seqset_create(ctx, data, offsets, n);
    });
}

int dm_seqset_destroy(dm_seqset* s) {
    return guard(s ? s->ctx : nullptr, [&] { delete s; });
}

uint32_t dm_seqset_count(const dm_seqset* s) { return s ? s->n : 0; }
int dm_seqset_planes(const dm_seqset* s) { return s ? s->planes : 0; }

static void fill_stats(dm_stats* st, dm::LevTotals& t, float total_ms) {
    dm::lev_finish_timing(t);
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->kernel_ms = t.kernel_ms;
    st->total_ms = total_ms;
    st->cells = t.cells;
    st->cells_executed = t.cells_exec;
    st->launches = t.launches;
}

uint32_t dm_levenshtein(dm_ctx* ctx, const char* a, uint64_t na, const char* b, uint64_t nb,
                        int* status) {
    uint32_t d = 0;
    int rc = guard(ctx, [&] {
        require(ctx != nullptr, "null context");
        std::string buf;
        buf.append(a, na);
        buf.append(b, nb);
        uint64_t off[3] = {0, na, na + nb};
        dm_seqset* s = dm::seqset_create(ctx, buf.data(), off, 2);
        std::vector<dm::LevItem> items{{0, 1, 0}};
        uint32_t* d_out = ctx->out.as<uint32_t>(1);
        try {
            dm::lev_run_host_items(ctx, s, items, d_out, nullptr, false);
            DM_CUDA(cudaMemcpyAsync(&d, d_out, 4, cudaMemcpyDeviceToHost, ctx->stream));
            DM_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete s;
            throw;
        }
        delete s;
    });
    if (status) *status = rc;
    return d;
}

int dm_lev_pairs(dm_ctx* ctx, const dm_seqset* s, const uint32_t* ia, const uint32_t* ib,
                 uint64_t n, uint32_t* out, dm_stats* st) {
    return guard(ctx, [&] {
        require(ctx && s, "null argument");
        for (uint64_t i = 0; i < n; ++i)
            require(ia[i] < s->n && ib[i] < s->n, "sequence index out of range");
        cudaStream_t stream = ctx->stream;
        cudaEvent_t t0, t1;
        DM_CUDA(cudaEventCreate(&t0));
        DM_CUDA(cudaEventCreate(&t1));
        DM_CUDA(cudaEventRecord(t0, stream));
        uint32_t* d_ab = ctx->aux3.as<uint32_t>(2 * n + 1);
        uint32_t* d_out = ctx->out.as<uint32_t>(n + 1);
        if (n) {
            DM_CUDA(cudaMemcpyAsync(d_ab, ia, n * 4, cudaMemcpyHostToDevice, stream));
            DM_CUDA(cudaMemcpyAsync(d_ab + n, ib, n * 4, cudaMemcpyHostToDevice, stream));
        }
        dm::LevTotals tot;
        dm::lev_run_device_pairs(ctx, s, d_ab, d_ab + n, n, d_out, &tot, st != nullptr);
        if (n) DM_CUDA(cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, stream));
        DM_CUDA(cudaEventRecord(t1, stream));
        DM_CUDA(cudaEventSynchronize(t1));
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        fill_stats(st, tot, ms);
    });
}

int dm_lev_pairs_device(dm_ctx* ctx, const dm_seqset* s, const uint32_t* d_ia,
                        const uint32_t* d_ib, uint64_t n, uint32_t* d_out, dm_stats* st) {
    return guard(ctx, [&] {
        require(ctx && s, "null argument");
        cudaEvent_t t0, t1;
        DM_CUDA(cudaEventCreate(&t0));
        DM_CUDA(cudaEventCreate(&t1));
        DM_CUDA(cudaEventRecord(t0, ctx->stream));
        dm::LevTotals tot;
        dm::lev_run_device_pairs(ctx, s, d_ia, d_ib, n, d_out, &tot, st != nullptr);
        DM_CUDA(cudaEventRecord(t1, ctx->stream));
        DM_CUDA(cudaEventSynchronize(t1));
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        fill_stats(st, tot, ms);
    });
}

int dm_lev_one_to_many(dm_ctx* ctx, const dm_seqset* s, uint32_t from, const uint32_t* members,
                       uint64_t n, uint32_t* out, dm_stats* st) {
    return guard(ctx, [&] {
        require(ctx && s, "null argument");
        require(from < s->n, "sequence index out of range");
        std::vector<dm::LevItem> items(n);
        for (uint64_t i = 0; i < n; ++i) {
            require(members[i] < s->n, "sequence index out of range");
            items[i] = dm::LevItem{from, members[i], (uint32_t)i};
        }
        uint32_t* d_out = ctx->out.as<uint32_t>(n + 1);
        dm::LevTotals tot;
        dm::lev_run_host_items(ctx, s, items, d_out, &tot, st != nullptr);
        if (n) DM_CUDA(cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        DM_CUDA(cudaStreamSynchronize(ctx->stream));
        fill_stats(st, tot, 0.f);
    });
}

int dm_geometric_median(dm_ctx* ctx, const dm_seqset* s, const uint32_t* members, uint64_t n,
                        uint64_t seed, uint64_t exact_cap, uint32_t* out) {
    return guard(ctx, [&] {
        require(ctx && s && out, "null argument");
        *out = dm::geometric_median(ctx, s, members, n, seed, exact_cap);
    });
}

int dm_build_tree(dm_ctx* ctx, const dm_seqset* s, uint64_t seed, uint64_t exact_cap,
                  dm_node* nodes, uint64_t* nnodes, uint32_t* order, dm_stats* st) {
    return guard(ctx, [&] {
        require(ctx && s && nodes && nnodes && order, "null argument");
        std::vector<dm_node> nv;
        std::vector<uint32_t> ov;
        if (st) std::memset(st, 0, sizeof(*st));
        cudaEvent_t t0, t1;
        DM_CUDA(cudaEventCreate(&t0));
        DM_CUDA(cudaEventCreate(&t1));
        DM_CUDA(cudaEventRecord(t0, ctx->stream));
        dm::build_tree(ctx, s, seed, exact_cap, nv, ov, st);
        DM_CUDA(cudaEventRecord(t1, ctx->stream));
        DM_CUDA(cudaEventSynchronize(t1));
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        if (st) {
            st->tree_ms = ms;
            st->total_ms = ms;
        }
        std::memcpy(nodes, nv.data(), nv.size() * sizeof(dm_node));
        std::memcpy(order, ov.data(), ov.size() * sizeof(uint32_t));
        *nnodes = nv.size();
    });
}

void dm_free(void* p) { std::free(p); }

}  // extern "C"
