#!/usr/bin/env python
"""Profiling driver for the pairwise aligner: `pairs` alignments of ~L x L
(DNA, mutated pairs) through dm.nw_batch; prints forward/traceback GCUPS."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=1300)
    ap.add_argument("--len", type=int, default=1600)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import paper_2601_15458_b200 as dm
    rng = np.random.default_rng(2)
    alpha = np.frombuffer(b"ACGT", dtype=np.uint8)
    pairs = []
    for _ in range(a.pairs):
        x = alpha[rng.integers(0, 4, a.len)]
        y = x.copy()
        k = rng.integers(0, a.len, a.len // 20)
        y[k] = alpha[rng.integers(0, 4, len(k))]
        pairs.append((x.tobytes(), y[: a.len - rng.integers(0, 30)].tobytes()))
    sc = dm.ScoringScheme.nucleotide()
    for r in range(a.reps):
        _, st = dm.nw_batch(pairs, sc, stats=True)
        print(f"rep {r}: {st['cells']:.3e} cells kernel {st['kernel_ms']:.3f} ms "
              f"-> {st['cells'] / st['kernel_ms'] / 1e6:.1f} GCUPS, launches {st['launches']}")


if __name__ == "__main__":
    main()
