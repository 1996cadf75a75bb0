#!/usr/bin/env python
"""`pairs` alignments of ~L x L (DNA, 10 % substitutions) through dm.nw_batch:
profiling target for the mid-size batches of the merge levels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2601_15458_b200 as dm  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 400
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2500
rng = np.random.default_rng(5)
alpha = np.frombuffer(b"ACGT", dtype=np.uint8)
pairs = []
for _ in range(P):
    x = alpha[rng.integers(0, 4, L)]
    y = x.copy()
    k = rng.integers(0, L, L // 10)
    y[k] = alpha[rng.integers(0, 4, len(k))]
    pairs.append((x.tobytes().decode(), y.tobytes().decode()))
for _ in range(2):
    _, st = dm.nw_batch(pairs, dm.ScoringScheme.nucleotide(), stats=True)
print(f"forward {st['align_ms']:.3f} ms, {st['cells'] / st['align_ms'] / 1e6:.0f} GCUPS")
