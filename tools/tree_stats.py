#!/usr/bin/env python
"""Per-depth cluster statistics of a config's guide tree (cardinality, radius),
i.e. how far apart the sequences the distance engine compares at each level
are (input to the banded-distance decision in DESIGN.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    import paper_2601_15458_b200 as dm
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    data, offs = dm.synth(cfg, scale)
    seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
    L = np.mean([len(s) for s in seqs])
    nodes, order = dm.build_tree(dm.SeqSet(seqs))
    f = {k: i for i, k in enumerate(dm.NODE_FIELDS)}
    card = nodes[:, f["end"]] - nodes[:, f["begin"]]
    print(f"cfg{cfg}@{scale}: n={len(seqs)} mean L={L:.0f}")
    for d in range(int(nodes[:, f["depth"]].max()) + 1):
        sel = (nodes[:, f["depth"]] == d) & (card > 1)
        if not sel.any():
            continue
        r = nodes[sel, f["radius"]]
        print(f"depth {d:2d}: nodes {sel.sum():5d} members {card[sel].sum():6d} radius median {np.median(r):6.0f} "
              f"p10 {np.percentile(r, 10):6.0f} max {r.max():6.0f} (radius/L median {np.median(r) / L:.2f})")


if __name__ == "__main__":
    main()
