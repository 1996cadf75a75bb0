"""Multi-GPU plumbing: one process per GPU (torchrun), an NCCL communicator
inside libdmb200 per rank.

The sharding contract mirrors csrc/comm.cpp: a batch of n jobs is split in
contiguous ranges, rank r owning ``shard_range(n, r, w)``; results are
exchanged (all-gather of distances, all-reduce of zeroed NW result buffers)
so every rank keeps identical, replicated decisions.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import check, lib


def shard_range(n: int, r: int, w: int):
    """Jobs [n*r//w, n*(r+1)//w) belong to rank r (comm.cpp shard_range)."""
    return n * r // w, n * (r + 1) // w


def owner_of(i: int, n: int, w: int) -> int:
    """Rank owning job i (the scatter rule of lev.cu scatter_shards)."""
    r = 0
    while r + 1 < w and n * (r + 1) // w <= i:
        r += 1
    return r


def gather_sharded(parts, n: int, w: int, maxc: int | None = None) -> np.ndarray:
    """Reassemble per-rank result rows (rank r: its range, padded to maxc)
    into job order — what scatter_shards does on the device."""
    out = np.empty(n, dtype=parts[0].dtype)
    for r in range(w):
        lo, hi = shard_range(n, r, w)
        out[lo:hi] = parts[r][: hi - lo]
    return out


def env_rank():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().dm_nccl_unique_id(buf))
    return bytes(buf)


def attach(ctx, rank: int, world: int, uid: bytes):
    """Attach an NCCL communicator (uid from rank 0) to a Context."""
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    check(lib().dm_ctx_attach_nccl(ctx.handle, buf, rank, world))


def attach_from_torch(ctx):
    """Inside torchrun with torch.distributed initialised: rank 0 creates the
    NCCL id, it is broadcast over the default process group, all attach."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    attach(ctx, rank, world, obj[0])
    return rank, world


def simulate_world(ctx, world: int):
    """Run the sharded code path with `world` shards on this one GPU."""
    check(lib().dm_ctx_simulate_world(ctx.handle, int(world)))
