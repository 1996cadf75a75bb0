#!/usr/bin/env python
"""Latency of a few long alignments (the top merge levels): forward-kernel ms
of `pairs` alignments of ~L x L through dm.nw_batch, for the ring kernel
(DM_NW_CLU=0) and the cluster kernel (DM_NW_CLU=2/4/8)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=1)
    ap.add_argument("--len", type=int, default=2600)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import paper_2601_15458_b200 as dm
    rng = np.random.default_rng(3)
    alpha = np.frombuffer(b"ACGT", dtype=np.uint8)
    pairs = []
    for _ in range(a.pairs):
        x = alpha[rng.integers(0, 4, a.len)]
        y = x.copy()
        k = rng.integers(0, a.len, a.len // 10)
        y[k] = alpha[rng.integers(0, 4, len(k))]
        pairs.append((x.tobytes().decode(), y.tobytes().decode()))
    sc = dm.ScoringScheme.nucleotide()
    os.environ["DM_NW_SEQ"] = "0"
    for clu in ("0", "2", "4", "8"):
        os.environ["DM_NW_CLU"] = clu
        best = None
        for _ in range(a.reps):
            _, st = dm.nw_batch(pairs, sc, stats=True)
            f = st["align_ms"]  # forward pass (dm_nw_batch)
            best = f if best is None else min(best, f)
        print(f"pairs {a.pairs} len {a.len} DM_NW_CLU={clu}: forward {best:.3f} ms "
              f"({st['cells'] / best / 1e6:.1f} GCUPS)", flush=True)


if __name__ == "__main__":
    main()
