#!/usr/bin/env python
"""Generate golden vectors by running the UNMODIFIED reference (oracle/_ref,
built from /root/reference by oracle/Makefile) in this container.

The vectors pin the oracle restatement (tests/test_oracle.py, CPU) and the
GPU path (tests/test_golden_gpu.py) on the GPU box, where /root/reference
does not exist. Inputs are regenerated from the seeds stored next to the
outputs (Python `random` for small cases, dm.synth for the BASELINE configs),
so only outputs (or their SHA-256 for full-size MSAs) are committed.

    python tests/golden/make_golden.py            # small vectors (seconds)
    python tests/golden/make_golden.py --big      # + cfg0/cfg2/cfg3 full MSAs (~40 min on 8 cores)
"""
import argparse
import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402


def rand_str(rng, n, alphabet):
    return "".join(rng.choice(alphabet) for _ in range(n))


def lev_cases():
    rng = random.Random(2024)
    cases = []
    for alpha in ("ACGT", "ACGTURYSWKMBDHVN", "ARNDCQEGHILKMFPSTWYV"):
        for _ in range(150):
            la = rng.choice([0, 1, 5, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 300, 700])
            a = rand_str(rng, la, alpha)
            b = list(a)
            for _ in range(rng.randrange(max(1, la // 5) + 1)):
                if b and rng.random() < 0.5:
                    b[rng.randrange(len(b))] = rng.choice(alpha)
                elif rng.random() < 0.5 and b:
                    del b[rng.randrange(len(b))]
                else:
                    b.insert(rng.randrange(len(b) + 1), rng.choice(alpha))
            cases.append([a, "".join(b)])
    return cases


def nw_cases():
    rng = random.Random(4048)
    out = []
    for kind, alpha in (("nt", "ACGTN-"), ("aa", "ARNDCQEGHILKMFPSTWYV-")):
        for go, ge, flat in ((-10, -1, False), (-3, -2, False), (-10, -1, True)):
            for _ in range(40):
                a = rand_str(rng, rng.randint(1, 80), alpha)
                b = rand_str(rng, rng.randint(1, 80), alpha)
                out.append(dict(kind=kind, go=go, ge=ge, flat=flat, a=a, b=b))
    return out


def tree_cases():
    rng = random.Random(8096)
    out = []
    for it in range(10):
        n = rng.randint(2, 260)
        seqs = list(dict.fromkeys(rand_str(rng, rng.randint(4, 40), "ACGT") for _ in range(n)))
        out.append(dict(seqs=seqs, seed=it, cap=rng.choice([100, 16, 2, 7])))
    return out


def sha(rows):
    h = hashlib.sha256()
    for r in rows:
        h.update(r.encode() if isinstance(r, str) else r)
        h.update(b"\n")
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default="", help="comma list of big-config keys to add (e.g. cfg4@1.0); skips the small vectors")
    args = ap.parse_args()
    ref = oracle.reference()
    if args.only:
        keys = [k for k in args.only.split(",") if k]
        if "cfg1@1.0" in keys:
            keys.remove("cfg1@1.0")
            cfg1_distances(ref)
        return big_configs(ref, keys) if keys else None

    lev = [[a, b, ref.levenshtein(a, b)] for a, b in lev_cases()]
    with open(os.path.join(HERE, "lev.json"), "w") as f:
        json.dump(lev, f, separators=(",", ":"))

    nw = []
    for c in nw_cases():
        r = ref.nw_align(c["a"], c["b"], c["kind"], c["go"], c["ge"], c["flat"])
        nw.append(dict(c, **r))
    with open(os.path.join(HERE, "nw.json"), "w") as f:
        json.dump(nw, f, separators=(",", ":"))

    trees = []
    for c in tree_cases():
        nodes, order = ref.build_tree(c["seqs"], seed=c["seed"], cap=c["cap"])
        trees.append(dict(c, nodes=nodes.tolist(), order=order.tolist()))
    with open(os.path.join(HERE, "tree.json"), "w") as f:
        json.dump(trees, f, separators=(",", ":"))

    msas = []
    rng = random.Random(16192)
    for it in range(6):
        alpha, kind = ("ACGT", "nt") if it % 2 == 0 else ("ARNDCQEGHILKMFPSTWYV", "aa")
        seqs = list(dict.fromkeys(rand_str(rng, rng.randint(5, 90), alpha) for _ in range(rng.randint(3, 120))))
        r = ref.msa(seqs, kind=kind, seed=it)
        msas.append(dict(seqs=seqs, kind=kind, seed=it, width=r["width"], rows=r["rows"],
                         order=r["order"].tolist()))
    with open(os.path.join(HERE, "msa_small.json"), "w") as f:
        json.dump(msas, f, separators=(",", ":"))

    if args.big:
        big_configs(ref, ["cfg0@1.0", "cfg3@1.0", "cfg2@0.1", "cfg2@1.0"])


def cfg1_distances(ref):
    """BASELINE configs[1] pinned in full: the reference's levenshtein
    (distance.cpp:9-48) over all 10^6 synth(1) pairs (2i, 2i+1), stored as the
    SHA-256 of the little-endian uint32 vector, one SHA per 65,536-pair block
    (to localise a mismatch), the sum and a histogram."""
    import paper_2601_15458_b200 as dm
    data, offs = dm.synth(1)
    seqs = dm.split(data, offs)
    n = len(seqs) // 2
    ia = np.arange(n, dtype=np.uint32) * 2
    t0 = time.time()
    d = ref.lev_pairs(seqs, ia, ia + 1, threads=os.cpu_count())
    wall = time.time() - t0
    d = np.ascontiguousarray(d, dtype="<u4")
    blk = 65536
    hist, edges = np.histogram(d, bins=64, range=(0, 1600))
    out = dict(cfg=1, pairs=int(n), sha256=hashlib.sha256(d.tobytes()).hexdigest(),
               block=blk, block_sha256=[hashlib.sha256(d[i:i + blk].tobytes()).hexdigest() for i in range(0, n, blk)],
               sum=int(d.astype(np.uint64).sum()), min=int(d.min()), max=int(d.max()),
               hist_range=[0, 1600], hist=hist.tolist(), first16=d[:16].tolist(),
               threads=os.cpu_count(), wall_s=wall,
               cells=int(sum((int(offs[2 * i + 1] - offs[2 * i]) * int(offs[2 * i + 2] - offs[2 * i + 1])) for i in range(n))))
    with open(os.path.join(HERE, "lev_cfg1.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("cfg1", {k: v for k, v in out.items() if k not in ("block_sha256", "hist")}, flush=True)


def big_configs(ref, keys):
    """Full-size reference MSAs (SHA-256 of rows / order / nodes) for the GPU
    golden tests; cfg4@1.0 takes hours on 8 cores and runs once per input."""
    import paper_2601_15458_b200 as dm
    big = {}
    path = os.path.join(HERE, "msa_configs.json")
    if os.path.exists(path):
        with open(path) as f:
            big = json.load(f)
    for key in keys:
        cfg, scale = int(key[3]), float(key.split("@")[1])
        kind = "aa" if cfg == 3 else "nt"
        if key in big:
            continue
        data, offs = dm.synth(cfg, scale)
        seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
        t0 = time.time()
        r = ref.msa(seqs, kind=kind, seed=42)
        big[key] = dict(cfg=cfg, scale=scale, kind=kind, n=len(seqs), width=r["width"],
                        rows_sha256=sha(r["rows"]), order_sha256=hashlib.sha256(r["order"].tobytes()).hexdigest(),
                        nodes_sha256=hashlib.sha256(np.ascontiguousarray(r["nodes"], dtype=np.int64).tobytes()).hexdigest(),
                        tree_s=r["tree_s"], align_s=r["align_s"], threads=os.cpu_count(),
                        wall_s=time.time() - t0)
        print(key, big[key], flush=True)
        with open(path, "w") as f:
            json.dump(big, f, indent=1)


if __name__ == "__main__":
    main()
