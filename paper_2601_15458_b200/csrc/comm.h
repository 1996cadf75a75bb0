// Multi-GPU sharding helpers (comm.cpp).
#pragma once

#include "dm_internal.h"

namespace dm {

// Number of shards a batch is split into: the NCCL world, or the simulated
// world (single GPU, DM_SIM_WORLD / dm_ctx_simulate_world) used by the tests.
int shard_world(const dm_ctx* ctx);
// Rank r of w owns jobs [n*r/w, n*(r+1)/w).
void shard_range(uint64_t n, int r, int w, uint64_t* lo, uint64_t* hi);

void comm_allgather(dm_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank);
void comm_allreduce_sum_u32(dm_ctx* ctx, void* buf, size_t count);
void comm_allreduce_sum_i64(dm_ctx* ctx, void* buf, size_t count);
void comm_destroy(dm_ctx* ctx);

}  // namespace dm
