// Multi-GPU plumbing (comm.cpp): the collectives libdmb200 uses between the
// ranks of one job, over NCCL (dm_ctx_attach_nccl) or over a caller-supplied
// host all-gather (dm_ctx_attach_host_comm: tests run several processes on
// one GPU through torch.distributed/gloo), and the work-balanced shard plan.
#pragma once

#include <vector>

#include "dm_internal.h"

namespace dm {

// Number of shards a batch is split into: the attached world, or the
// simulated world (one GPU, DM_SIM_WORLD / dm_ctx_simulate_world, tests).
int shard_world(const dm_ctx* ctx);
// True when this process is one of several attached ranks.
inline bool comm_real(const dm_ctx* ctx) { return ctx->world > 1; }

// Work-balanced contiguous shards: bounds[0] = 0 <= ... <= bounds[w] = n,
// shard r = [bounds[r], bounds[r+1]) holding ~1/w of sum(cost); identical on
// every rank for the same costs.
void shard_bounds(const uint64_t* cost, uint64_t n, int w, std::vector<uint64_t>& bounds);
// Largest-processing-time assignment of items to w ranks by cost (ties to
// the lower rank; deterministic).
void assign_lpt(const uint64_t* cost, uint64_t n, int w, std::vector<int>& owner);

// All-gather on DEVICE buffers (recv = w * bytes_per_rank), on ctx->stream.
void comm_allgather(dm_ctx* ctx, const void* d_send, void* d_recv, size_t bytes_per_rank);
// All-gather on HOST buffers (synchronous).
void comm_allgather_host(dm_ctx* ctx, const void* h_send, void* h_recv, size_t bytes_per_rank);
// Variable-size all-gather of host blobs: out[r] = rank r's blob.
void comm_allgatherv_host(dm_ctx* ctx, const std::vector<uint8_t>& mine, std::vector<std::vector<uint8_t>>& out);
void comm_destroy(dm_ctx* ctx);

}  // namespace dm
