// Multi-GPU plumbing: one process per GPU, an NCCL
// communicator per dm_ctx. NCCL is loaded at attach time with dlopen (the
// same libnccl.so.2 torch has already loaded, or the system one), so
// single-GPU use has no NCCL dependency.
//
// Sharding contract used by the tree builder and the merge scheduler: a
// batch of I jobs is split in contiguous ranges, rank r owning
// [I*r/W, I*(r+1)/W) (shard_range); decisions stay replicated, so the only
// data exchanged are the per-job results (all-gather of distances, all-reduce
// of zero-initialised NW result/gap buffers). DM_SIM_WORLD=k (k > 1) runs the
// same sharded code path on ONE GPU, executing the k ranges in turn and
// exchanging through local copies — how the single-GPU test box checks the
// partition/gather logic.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>

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

void shard_range(uint64_t n, int r, int w, uint64_t* lo, uint64_t* hi) {
    *lo = n * (uint64_t)r / (uint64_t)w;
    *hi = n * (uint64_t)(r + 1) / (uint64_t)w;
}

void comm_allgather(dm_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
    nccl_check(nccl().allGather(send, recv, bytes_per_rank, kNcclUint8, ctx->nccl, ctx->stream), "ncclAllGather");
}

void comm_allreduce_sum_u32(dm_ctx* ctx, void* buf, size_t count) {
    nccl_check(nccl().allReduce(buf, buf, count, kNcclUint32, kNcclSum, ctx->nccl, ctx->stream), "ncclAllReduce");
}

void comm_allreduce_sum_i64(dm_ctx* ctx, void* buf, size_t count) {
    nccl_check(nccl().allReduce(buf, buf, count, kNcclInt64, kNcclSum, ctx->nccl, ctx->stream), "ncclAllReduce");
}

void comm_destroy(dm_ctx* ctx) {
    if (ctx->nccl) nccl().commDestroy(ctx->nccl);
    ctx->nccl = nullptr;
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

int dm_ctx_simulate_world(dm_ctx* ctx, int world) {
    return dm::guard(ctx, [&] {
        dm::require(ctx != nullptr, "null context");
        dm::require(world >= 1 && world <= 64, "simulated world must be in [1, 64]");
        ctx->sim_world = world;
    });
}

}  // extern "C"
