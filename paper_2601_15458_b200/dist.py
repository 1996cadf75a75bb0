"""Multi-GPU plumbing: one process per GPU (torchrun), an NCCL communicator
inside libdmb200 per rank.

The sharding contract lives in csrc/comm.cpp (exported as dm_shard_bounds /
dm_assign_owners): a batch is split in contiguous cost-balanced ranges whose
results are all-gathered, and below a split level whole subtrees go to
ranks and are exchanged once, so every rank keeps identical, replicated
decisions. Collectives run over NCCL (attach /
attach_from_torch) or over torch.distributed on host memory
(attach_host_comm).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import check, lib


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


# dm_allgather_fn (include/dm_b200.h)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


def attach_host_comm(ctx, group=None):
    """Attach the library's collectives to torch.distributed (any backend,
    e.g. gloo on CPU tensors): the sharded tree / merge path then runs across
    the group's processes, which may share one GPU (tests), with every
    exchange an all-gather of host bytes through this callback."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)

    def _allgather(send, recv, nbytes, _user):
        try:
            n = int(nbytes)
            src = torch.empty(max(n, 1), dtype=torch.uint8)
            if n:
                C.memmove(src.data_ptr(), send, n)
            parts = [torch.empty(max(n, 1), dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, src, group=group)
            for r, t in enumerate(parts):
                if n:
                    C.memmove(recv + r * n, t.data_ptr(), n)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    cb = ALLGATHER_FN(_allgather)
    ctx._host_comm = cb  # the library keeps the pointer: keep the thunk alive
    check(lib().dm_ctx_attach_host_comm(ctx.handle, rank, world, C.cast(cb, C.c_void_p), None))
    return rank, world


def comm_stats(ctx) -> dict:
    """Collective calls / bytes and owned subtrees of this rank (dm_ctx_comm_stats)."""
    out = np.zeros(4, dtype=np.uint64)
    check(lib().dm_ctx_comm_stats(ctx.handle, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return {"collectives": int(out[0]), "bytes": int(out[1]), "owned_tree_subtrees": int(out[2]),
            "owned_merge_subtrees": int(out[3])}


def shard_bounds(costs, world: int) -> np.ndarray:
    """The library's cost-balanced contiguous split (dm_shard_bounds)."""
    c = np.ascontiguousarray(costs, dtype=np.uint64)
    out = np.zeros(world + 1, dtype=np.uint64)
    check(lib().dm_shard_bounds(c.ctypes.data_as(C.POINTER(C.c_uint64)), len(c), world,
                                out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def assign_owners(costs, world: int) -> np.ndarray:
    """The library's subtree-to-rank assignment (dm_assign_owners, LPT)."""
    c = np.ascontiguousarray(costs, dtype=np.uint64)
    out = np.zeros(len(c), dtype=np.int32)
    check(lib().dm_assign_owners(c.ctypes.data_as(C.POINTER(C.c_uint64)), len(c), world,
                                 out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def simulate_world(ctx, world: int):
    """Run the sharded code path with `world` shards on this one GPU."""
    check(lib().dm_ctx_simulate_world(ctx.handle, int(world)))
