// Multi-GPU plumbing: one process per GPU, an NCCL
// communicator per dm_ctx. NCCL is loaded at attach time with dlopen (the
// same libnccl.so.2 torch has already loaded, or the system one), so
// single-GPU use has no NCCL dependency.
//
// Sharding contract used by the tree builder and the merge scheduler: a
// batch of jobs is split in contiguous, cost-balanced ranges (shard_bounds:
// sum |a||b| per range ~ 1/W of the batch); decisions stay replicated, so the
// only data exchanged are the per-job results (all-gathers of distances, NW
// results and compacted gap lists). Below a split level whole subtrees are
// assigned to ranks (assign_lpt) and exchanged once (tree.cu, msa.cu).
// DM_SIM_WORLD=k (k > 1) runs the range-sharded code path on ONE GPU,
// executing the k ranges in turn — how the single-GPU test box checks the
// partition/gather logic; dm_ctx_attach_host_comm runs the real multi-rank
// path with the collectives done by a host callback (several processes
// sharing one GPU in the tests).
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "capi_guard.h"
#include "comm.h"

namespace dm {
namespace {

// Minimal NCCL ABI (nccl.h, stable across 2.x).
typedef struct {
    char internal[128];
} NcclUid;
typedef void* NcclComm;
enum { kNcclUint8 = 1, kNcclUint32 = 3, kNcclInt64 = 4 };
enum { kNcclSum = 0 };

struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(NcclUid*) = nullptr;
    int (*commInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
    int (*commDestroy)(NcclComm) = nullptr;
    int (*allGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    const char* (*errStr)(int) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw cuda_error(std::string("cannot load NCCL: ") + dlerror());
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) throw cuda_error(std::string("NCCL symbol missing: ") + n);
            return p;
        };
        api.getUniqueId = (int (*)(NcclUid*))sym("ncclGetUniqueId");
        api.commInitRank = (int (*)(NcclComm*, int, NcclUid, int))sym("ncclCommInitRank");
        api.commDestroy = (int (*)(NcclComm))sym("ncclCommDestroy");
        api.allGather = (int (*)(const void*, void*, size_t, int, NcclComm, cudaStream_t))sym("ncclAllGather");
        api.allReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))sym("ncclAllReduce");
        api.errStr = (const char* (*)(int))sym("ncclGetErrorString");
        api.h = h;
    }
    return api;
}

void nccl_check(int rc, const char* what) {
    if (rc != 0) throw cuda_error(std::string(what) + ": " + nccl().errStr(rc));
}

}  // namespace

int shard_world(const dm_ctx* ctx) { return ctx->world > 1 ? ctx->world : std::max(1, ctx->sim_world); }

void shard_bounds(const uint64_t* cost, uint64_t n, int w, std::vector<uint64_t>& bounds) {
    bounds.assign((size_t)w + 1, n);
    bounds[0] = 0;
    long double total = 0;
    for (uint64_t i = 0; i < n; ++i) total += (long double)std::max<uint64_t>(cost[i], 1);
    // shard r starts at the first job whose preceding cost reaches r/w of the total
    long double acc = 0;
    int r = 1;
    for (uint64_t i = 0; i < n && r < w; ++i) {
        while (r < w && acc >= total * r / w) bounds[r++] = i;
        acc += (long double)std::max<uint64_t>(cost[i], 1);
    }
    for (; r < w; ++r) bounds[r] = n;
    for (int k = 1; k <= w; ++k) bounds[k] = std::max(bounds[k], bounds[k - 1]);
}

void assign_lpt(const uint64_t* cost, uint64_t n, int w, std::vector<int>& owner) {
    std::vector<uint64_t> idx(n);
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) { return cost[a] > cost[b]; });
    std::vector<long double> load((size_t)w, 0);
    owner.assign(n, 0);
    for (uint64_t i : idx) {
        int best = 0;
        for (int r = 1; r < w; ++r)
            if (load[r] < load[best]) best = r;
        owner[i] = best;
        load[best] += (long double)std::max<uint64_t>(cost[i], 1);
    }
}

namespace {
uint8_t* comm_stage(dm_ctx* ctx, size_t bytes) {
    if (!ctx->comm_pin) ctx->comm_pin = new PinnedBuf;
    return (uint8_t*)ctx->comm_pin->get(std::max<size_t>(bytes, 16));
}
void host_gather(dm_ctx* ctx, const void* send, void* recv, size_t bytes) {
    if (ctx->host_allgather(send, recv, bytes, ctx->host_comm_user) != 0)
        throw cuda_error("host all-gather callback failed");
}
}  // namespace

void comm_allgather(dm_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
    ++ctx->coll_calls;
    ctx->coll_bytes += bytes_per_rank;
    if (ctx->nccl) {
        nccl_check(nccl().allGather(send, recv, bytes_per_rank, kNcclUint8, ctx->nccl, ctx->stream), "ncclAllGather");
        return;
    }
    if (!ctx->host_allgather) throw runtime_error("no communicator attached");
    // staged through pinned host memory: [send | recv]
    const size_t w = (size_t)ctx->world;
    uint8_t* h = comm_stage(ctx, bytes_per_rank * (w + 1));
    DM_CUDA(cudaMemcpyAsync(h, send, bytes_per_rank, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    host_gather(ctx, h, h + bytes_per_rank, bytes_per_rank);
    DM_CUDA(cudaMemcpyAsync(recv, h + bytes_per_rank, bytes_per_rank * w, cudaMemcpyHostToDevice, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void comm_allgather_host(dm_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
    if (ctx->host_allgather) {
        ++ctx->coll_calls;
        ctx->coll_bytes += bytes_per_rank;
        host_gather(ctx, send, recv, bytes_per_rank);
        return;
    }
    if (!ctx->nccl) throw runtime_error("no communicator attached");
    const size_t w = (size_t)ctx->world;
    uint8_t* d = (uint8_t*)ctx->comm_dev.get(bytes_per_rank * (w + 1) + 16);
    DM_CUDA(cudaMemcpyAsync(d, send, bytes_per_rank, cudaMemcpyHostToDevice, ctx->stream));
    comm_allgather(ctx, d, d + bytes_per_rank, bytes_per_rank);
    DM_CUDA(cudaMemcpyAsync(recv, d + bytes_per_rank, bytes_per_rank * w, cudaMemcpyDeviceToHost, ctx->stream));
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void comm_allgatherv_host(dm_ctx* ctx, const std::vector<uint8_t>& mine, std::vector<std::vector<uint8_t>>& out) {
    const int w = ctx->world;
    uint64_t my = mine.size();
    std::vector<uint64_t> sizes((size_t)w);
    comm_allgather_host(ctx, &my, sizes.data(), sizeof(uint64_t));
    uint64_t mx = 16;
    for (uint64_t x : sizes) mx = std::max(mx, x);
    std::vector<uint8_t> send(mx, 0), recv(mx * (size_t)w);
    if (my) std::memcpy(send.data(), mine.data(), my);
    comm_allgather_host(ctx, send.data(), recv.data(), mx);
    out.assign((size_t)w, {});
    for (int r = 0; r < w; ++r) out[r].assign(recv.begin() + (size_t)r * mx, recv.begin() + (size_t)r * mx + sizes[r]);
}

void comm_destroy(dm_ctx* ctx) {
    if (ctx->nccl) nccl().commDestroy(ctx->nccl);
    ctx->nccl = nullptr;
    ctx->host_allgather = nullptr;
    ctx->host_comm_user = nullptr;
    delete ctx->comm_pin;
    ctx->comm_pin = nullptr;
}

}  // namespace dm

extern "C" {

int dm_nccl_unique_id(uint8_t* id128) {
    return dm::guard([&] {
        dm::require(id128 != nullptr, "null argument");
        dm::NcclUid uid;
        dm::nccl_check(dm::nccl().getUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(id128, &uid, 128);
    });
}

int dm_ctx_attach_nccl(dm_ctx* ctx, const uint8_t* id128, int rank, int world) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && id128, "null argument");
        dm::require(world >= 1 && rank >= 0 && rank < world, "invalid shard (rank, world)");
        DM_CUDA(cudaSetDevice(ctx->device));
        dm::comm_destroy(ctx);
        if (world > 1) {
            dm::NcclUid uid;
            std::memcpy(&uid, id128, 128);
            dm::NcclComm c = nullptr;
            dm::nccl_check(dm::nccl().commInitRank(&c, world, uid, rank), "ncclCommInitRank");
            ctx->nccl = c;
        }
        ctx->rank = rank;
        ctx->world = world;
    });
}

int dm_ctx_attach_host_comm(dm_ctx* ctx, int rank, int world, dm_allgather_fn fn, void* user) {
    return dm::guard(ctx, [&] {
        dm::require(ctx != nullptr, "null context");
        dm::require(world >= 1 && rank >= 0 && rank < world, "invalid shard (rank, world)");
        dm::require(world == 1 || fn != nullptr, "null all-gather callback");
        dm::comm_destroy(ctx);
        ctx->host_allgather = world > 1 ? fn : nullptr;
        ctx->host_comm_user = user;
        ctx->rank = rank;
        ctx->world = world;
    });
}

int dm_ctx_comm_stats(dm_ctx* ctx, uint64_t* out4) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && out4, "null argument");
        out4[0] = ctx->coll_calls;
        out4[1] = ctx->coll_bytes;
        out4[2] = ctx->own_tree;
        out4[3] = ctx->own_msa;
    });
}

int dm_shard_bounds(const uint64_t* cost, uint64_t n, int world, uint64_t* bounds) {
    return dm::guard([&] {
        dm::require(bounds && (cost || n == 0) && world >= 1, "invalid argument");
        std::vector<uint64_t> b;
        dm::shard_bounds(cost, n, world, b);
        std::memcpy(bounds, b.data(), b.size() * sizeof(uint64_t));
    });
}

int dm_assign_owners(const uint64_t* cost, uint64_t n, int world, int32_t* owner) {
    return dm::guard([&] {
        dm::require(owner && (cost || n == 0) && world >= 1, "invalid argument");
        std::vector<int> o;
        dm::assign_lpt(cost, n, world, o);
        for (uint64_t i = 0; i < n; ++i) owner[i] = o[i];
    });
}

int dm_ctx_simulate_world(dm_ctx* ctx, int world) {
    return dm::guard(ctx, [&] {
        dm::require(ctx != nullptr, "null context");
        dm::require(world >= 1 && world <= 64, "simulated world must be in [1, 64]");
        ctx->sim_world = world;
    });
}

}  // extern "C"
