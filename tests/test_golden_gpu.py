"""GPU path against golden vectors produced by the unmodified reference
(tests/golden/make_golden.py). These run on the GPU box, where
/root/reference is absent: the fixtures are the reference there."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not generated")
    with open(p) as f:
        return json.load(f)


def test_lev_golden(dm, ctx):
    cases = load("lev.json")
    seqs = [s for a, b, _ in cases for s in (a, b)]
    ss = dm.SeqSet(seqs, ctx)
    ia = np.arange(0, len(seqs), 2)
    got = dm.lev_pairs(ss, ia, ia + 1)
    assert [int(x) for x in got] == [d for _, _, d in cases]


def test_nw_golden(dm, ctx):
    cases = load("nw.json")
    groups = {}
    for c in cases:
        groups.setdefault((c["kind"], c["go"], c["ge"], c["flat"]), []).append(c)
    for (kind, go, ge, flat), cs in groups.items():
        ctor = dm.ScoringScheme.nucleotide if kind == "nt" else dm.ScoringScheme.protein
        sc = ctor(go, ge, "flat" if flat else "affine")
        got = dm.nw_batch([(c["a"], c["b"]) for c in cs], sc, ctx)
        for c, r in zip(cs, got):
            assert (r.score, r.aligned_a, r.aligned_b, r.gaps_into_a, r.gaps_into_b) == (
                c["score"], c["aligned_a"], c["aligned_b"], c["gaps_into_a"], c["gaps_into_b"])


def test_tree_golden(dm, ctx):
    for c in load("tree.json"):
        nodes, order = dm.build_tree(dm.SeqSet(c["seqs"], ctx), seed=c["seed"], exact_cap=c["cap"])
        assert nodes.tolist() == c["nodes"]
        assert order.tolist() == c["order"]


def test_msa_golden(dm, ctx):
    for c in load("msa_small.json"):
        sc = dm.ScoringScheme.nucleotide() if c["kind"] == "nt" else dm.ScoringScheme.protein()
        m = dm.msa(dm.SeqSet(c["seqs"], ctx), sc, seed=c["seed"])
        assert m.width == c["width"] and m.rows == c["rows"]
        assert m.order.tolist() == c["order"]


def _sha_rows(rows):
    h = hashlib.sha256()
    for r in rows:
        h.update(r.encode())
        h.update(b"\n")
    return h.hexdigest()


@pytest.mark.parametrize("key", ["cfg0@1.0", "cfg3@1.0", "cfg2@0.1", "cfg2@1.0", "cfg4@1.0"])
def test_config_msa_golden(dm, ctx, key):
    """Full-size BASELINE configs: tree and MSA bytes equal the reference's (by SHA-256)."""
    big = load("msa_configs.json")
    if key not in big:
        pytest.skip(f"{key} not generated")
    c = big[key]
    data, offs = dm.synth(c["cfg"], c["scale"])
    seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
    assert len(seqs) == c["n"]
    sc = dm.ScoringScheme.nucleotide() if c["kind"] == "nt" else dm.ScoringScheme.protein()
    m = dm.msa(dm.SeqSet(seqs, ctx), sc, seed=42)
    assert hashlib.sha256(np.ascontiguousarray(m.nodes, dtype=np.int64).tobytes()).hexdigest() == c["nodes_sha256"]
    assert hashlib.sha256(m.order.tobytes()).hexdigest() == c["order_sha256"]
    assert m.width == c["width"]
    assert _sha_rows(m.rows) == c["rows_sha256"]
