"""CPU, world_size 2/3 over gloo: the host side of the multi-GPU sharding,
driven by the library's own plan functions (libdmb200 dm_shard_bounds /
dm_assign_owners, pure host code). Each rank computes its cost-balanced
range of a distance batch (the CPU oracle standing in for the kernel), the
ranges are all-gathered with padding as comm.cpp / lev.cu do, and every
rank must hold the full, identical result; subtree ownership must be
identical and balanced on every rank; compacted variable-length gap lists
go through the padded all-gather nw.cu uses. The full multi-rank GPU path
(these collectives inside libdmb200, several processes on one GPU) is
tests/test_multirank_gpu.py."""
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
        from paper_2601_15458_b200.dist import assign_owners, shard_bounds
        orc = oracle.restatement()
        rng = random.Random(17)
        seqs = ["".join(rng.choice("ACGT") for _ in range(rng.randint(0, 60))) for _ in range(80)]
        jobs = [(rng.randrange(80), rng.randrange(80)) for _ in range(101)]  # odd count: uneven shards
        n = len(jobs)
        # the library's own plan (dm_shard_bounds), cost |a| * |b| as lev.cu uses
        cost = np.array([len(seqs[a]) * len(seqs[b]) for a, b in jobs], dtype=np.uint64)
        bounds = shard_bounds(cost, world)
        plans = [None] * world
        dist.all_gather_object(plans, bounds.tolist())
        ok_plan = all(p == bounds.tolist() for p in plans) and bounds[0] == 0 and bounds[-1] == n
        maxc = int(max(bounds[r + 1] - bounds[r] for r in range(world)))
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        mine = np.zeros(max(maxc, 1), dtype=np.int64)
        for k, (a, b) in enumerate(jobs[lo:hi]):
            mine[k] = orc.levenshtein(seqs[a], seqs[b])
        parts = [torch.zeros(max(maxc, 1), dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        got = np.empty(n, dtype=np.int64)  # lev.cu scatter_shards: rank r's row -> its range
        for r in range(world):
            b0, b1 = int(bounds[r]), int(bounds[r + 1])
            got[b0:b1] = parts[r].numpy()[: b1 - b0]
        want = np.array([orc.levenshtein(seqs[a], seqs[b]) for a, b in jobs])
        ok_lev = bool(np.array_equal(got, want))
        # subtree ownership (dm_assign_owners): identical on every rank, LPT balanced
        sizes = np.array([rng.randint(2, 5000) for _ in range(40)], dtype=np.uint64)
        own = assign_owners(sizes, world)
        owns = [None] * world
        dist.all_gather_object(owns, own.tolist())
        load = [int(sizes[own == r].sum()) for r in range(world)]
        ok_own = all(o == own.tolist() for o in owns) and max(load) - min(load) <= int(sizes.max())
        # the compacted-gap exchange of nw.cu: variable lengths, padded all-gather
        mygaps = np.arange(rank * 7, rank * 7 + 3 + rank, dtype=np.int64)
        sz = [None] * world
        dist.all_gather_object(sz, len(mygaps))
        mx = max(sz)
        pad = np.zeros(mx, dtype=np.int64)
        pad[: len(mygaps)] = mygaps
        gp = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gp, torch.from_numpy(pad))
        ok_gaps = all(np.array_equal(gp[r].numpy()[: sz[r]], np.arange(r * 7, r * 7 + 3 + r)) for r in range(world))
        q.put((rank, ok_plan, ok_lev, ok_own, ok_gaps))
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
    for rank, ok_plan, ok_lev, ok_own, ok_gaps in results:
        assert ok_plan and ok_lev and ok_own and ok_gaps, (rank, ok_plan, ok_lev, ok_own, ok_gaps)


def test_shard_bounds_balance_cost():
    """dm_shard_bounds: contiguous, complete, each range ~1/w of the cost."""
    from paper_2601_15458_b200.dist import shard_bounds
    rng = np.random.default_rng(3)
    for n in (0, 1, 5, 101, 4950):
        for w in (1, 2, 3, 8):
            cost = rng.integers(1, 10**6, n).astype(np.uint64)
            b = shard_bounds(cost, w)
            assert b[0] == 0 and b[-1] == n and all(b[k] <= b[k + 1] for k in range(w))
            if n >= 50 * w:
                parts = [int(cost[b[k]:b[k + 1]].sum()) for k in range(w)]
                assert max(parts) - min(parts) <= 2 * int(cost.max())
