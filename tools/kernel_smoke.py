#!/usr/bin/env python
"""Drives every kernel of libdmb200 on tiny inputs in one process (a
compute-sanitizer target: `compute-sanitizer --tool memcheck|racecheck|
synccheck|initcheck python tools/kernel_smoke.py`; the tool is closed on the
round-1 GPU pool, so the parity tests' small/edge cases stand in).

Covers: seqset census/recode/planes, the distance planner and kernels
(DNA / protein / 94-symbol alphabets, several buckets), the streamed host
path, the tree kernels (big levels, sampled medians, subtrees), NW forward
(1 / 4 / 8 warps per alignment, int32 and int64) and traceback, the merge
scheduler, gap-column insertion, metrics, the FASTA formatter and the
sharded path (simulated world)."""
import os
import random
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def rs(rng, n, alpha="ACGT"):
    return "".join(rng.choice(alpha) for _ in range(n))


def main():
    import paper_2601_15458_b200 as dm
    from paper_2601_15458_b200.dist import simulate_world
    rng = random.Random(1)
    ctx = dm.Context(0)
    for alpha in ("ACGT", "ARNDCQEGHILKMFPSTWYV", "".join(chr(c) for c in range(33, 127))):
        seqs = [rs(rng, rng.randint(0, 700), alpha) for _ in range(40)]
        ss = dm.SeqSet(seqs, ctx)
        ia = np.arange(20) * 2
        dm.lev_pairs(ss, ia, ia + 1)
    data, offs = dm.synth(1, scale=0.0005)
    os.environ["DM_STREAM_CHUNK_BYTES"] = "60000"
    dm.lev_pairs_packed(data, offs, ctx)
    del os.environ["DM_STREAM_CHUNK_BYTES"]
    # tree + MSA (cfg0 slice has big nodes and small subtrees), protein too
    data, offs = dm.synth(0, scale=0.25)
    seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide())
    dm.evaluate(m, seqs, 200, 500, 3, ctx)
    prot = list(dict.fromkeys(rs(rng, rng.randint(20, 120), "ARNDCQEGHILKMFPSTWYV") for _ in range(60)))
    dm.msa(dm.SeqSet(prot, ctx), dm.ScoringScheme.protein(), exact_cap=16)
    # NW: one, four and eight bands; the int64 path via a wide custom scheme
    pairs = [(rs(rng, n), rs(rng, n + rng.randint(-20, 20))) for n in (30, 600, 1500, 3000)]
    dm.nw_batch(pairs, dm.ScoringScheme.nucleotide(), ctx)
    wide = dm.ScoringScheme.custom("ACGT", [30000 if i == j else -30000 for i in range(4) for j in range(4)],
                                   -10, -1)
    dm.nw_batch(pairs[2:], wide, ctx)
    dm.insert_gap_columns(["ACGT", "A-GT"], [0, 2, 2, 4], ctx)
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "in.fa")
        with open(src, "w") as f:
            for i, s in enumerate(seqs[:50] + seqs[:5]):
                f.write(f">r{i} d\n{s}\n")
        dm.run_align(src, os.path.join(d, "out.fa"), dump_tree=os.path.join(d, "t"), dump_dedup=os.path.join(d, "u"),
                     ctx=ctx)
    c2 = dm.Context(0)
    simulate_world(c2, 3)
    dm.msa(dm.SeqSet(seqs[:120], c2), dm.ScoringScheme.nucleotide())
    print("kernel smoke done")


if __name__ == "__main__":
    main()
