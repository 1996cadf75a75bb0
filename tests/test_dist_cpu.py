"""CPU, world_size 2 over gloo: the host side of the multi-GPU sharding.

Each rank computes its contiguous range of a distance batch (here with the
CPU oracle standing in for the GPU kernel), the ranges are all-gathered with
padding exactly as comm.cpp / lev.cu do with ncclAllGather, every rank
routes the rows back to job order (scatter_shards) and must hold the full,
identical result. The NW result exchange (zeroed buffers + sum all-reduce)
and the NCCL-id broadcast are exercised the same way."""
import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2601_15458_b200.dist import gather_sharded, owner_of, shard_range
        orc = oracle.restatement()
        rng = random.Random(17)
        seqs = ["".join(rng.choice("ACGT") for _ in range(rng.randint(0, 60))) for _ in range(80)]
        jobs = [(rng.randrange(80), rng.randrange(80)) for _ in range(101)]  # odd count: uneven shards
        n = len(jobs)
        maxc = max(shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world))
        lo, hi = shard_range(n, rank, world)
        mine = np.zeros(maxc, dtype=np.int64)
        for k, (a, b) in enumerate(jobs[lo:hi]):
            mine[k] = orc.levenshtein(seqs[a], seqs[b])
        parts = [torch.zeros(maxc, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        got = gather_sharded([p.numpy() for p in parts], n, world)
        want = np.array([orc.levenshtein(seqs[a], seqs[b]) for a, b in jobs])
        ok_lev = bool(np.array_equal(got, want))
        ok_owner = all(shard_range(n, owner_of(i, n, world), world)[0] <= i <
                       shard_range(n, owner_of(i, n, world), world)[1] for i in range(n))
        # NW-style exchange: each rank writes its slots into a zeroed buffer, sum all-reduce
        buf = torch.zeros(n, dtype=torch.int64)
        for i in range(lo, hi):
            buf[i] = int(want[i]) - 7  # signed values survive the sum
        dist.all_reduce(buf)
        ok_sum = bool(np.array_equal(buf.numpy(), want - 7))
        # NCCL-id broadcast path (128 opaque bytes from rank 0)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ok_uid = obj[0] == bytes(range(128))
        q.put((rank, ok_lev, ok_owner, ok_sum, ok_uid))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    results = sorted(q.get(timeout=5) for _ in range(world))
    assert [r[0] for r in results] == list(range(world))
    for rank, ok_lev, ok_owner, ok_sum, ok_uid in results:
        assert ok_lev and ok_owner and ok_sum and ok_uid, (rank, ok_lev, ok_owner, ok_sum, ok_uid)


def test_shard_range_matches_device_rule():
    from paper_2601_15458_b200.dist import owner_of, shard_range
    for n in (0, 1, 5, 101, 4950):
        for w in (1, 2, 3, 8):
            covered = []
            for r in range(w):
                lo, hi = shard_range(n, r, w)
                covered.extend(range(lo, hi))
                for i in range(lo, hi):
                    assert owner_of(i, n, w) == r
            assert covered == list(range(n))
