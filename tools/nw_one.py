#!/usr/bin/env python
"""One long alignment through dm.nw_batch (profiling target for the latency kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2601_15458_b200 as dm  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2600
rng = np.random.default_rng(3)
alpha = np.frombuffer(b"ACGT", dtype=np.uint8)
x = alpha[rng.integers(0, 4, L)]
y = x.copy()
k = rng.integers(0, L, L // 10)
y[k] = alpha[rng.integers(0, 4, len(k))]
for _ in range(3):
    _, st = dm.nw_batch([(x.tobytes().decode(), y.tobytes().decode())], dm.ScoringScheme.nucleotide(), stats=True)
print(f"forward {st['align_ms']:.3f} ms")
