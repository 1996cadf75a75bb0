"""Parity of the GPU guide tree with the reference build_tree.

Pins restate /root/reference/proj/tests/test_cluster_tree.cpp:115-236; every
random case compares all node fields and `order` with the compiled
reference (oracle/_ref) or the C restatement."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand_str(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


def unique(seqs):
    out, seen = [], set()
    for s in seqs:
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


def mutation_families(rng, families, per, base_len, rate, alphabet="ACGT"):
    out = []
    for _ in range(families):
        anc = rand_str(rng, base_len, alphabet)
        for _ in range(per):
            s = list(anc)
            for _ in range(max(1, int(rate * base_len))):
                k = rng.randrange(3)
                p = rng.randrange(len(s))
                if k == 0:
                    s[p] = rng.choice(alphabet)
                elif k == 1 and len(s) > 4:
                    del s[p]
                else:
                    s.insert(p, rng.choice(alphabet))
            out.append("".join(s))
    return out


def test_geometric_median_pins(dm, ctx):
    ss = dm.SeqSet(["AAAA", "AAAT", "TTTT"], ctx)
    assert dm.geometric_median(ss, [0, 1, 2], 42) == 1
    pair = dm.SeqSet(["AAAA", "TTTT"], ctx)
    assert dm.geometric_median(pair, [0, 1], 42) == 0
    assert dm.geometric_median(pair, [1, 0], 42) == 0
    one = dm.SeqSet(["ACGT"], ctx)
    assert dm.geometric_median(one, [0], 42) == 0
    with pytest.raises(ValueError):
        dm.geometric_median(one, [], 42)


def test_sampled_median_matches_reference(dm, ctx, ref):
    rng = random.Random(21)
    seqs = unique([rand_str(rng, rng.randint(8, 20)) for _ in range(60)])
    ss = dm.SeqSet(seqs, ctx)
    members = list(range(len(seqs)))
    for seed, cap in [(7, 16), (8, 16), (7, len(seqs)), (99, len(seqs) + 50), (3, 2), (5, 1)]:
        assert dm.geometric_median(ss, members, seed, cap) == ref.geometric_median(seqs, members, seed, cap)


def test_three_sequence_pins(dm, ctx):
    nodes, order = dm.build_tree(dm.SeqSet(["AAAA", "AAAT", "TTTT"], ctx))
    root = nodes[0]
    assert root[2] == 1 and root[4] == 2 and root[5] == 0 and root[3] == 3
    left, right = nodes[root[6]], nodes[root[7]]
    assert list(order[left[0]:left[1]]) == [2]
    assert sorted(order[right[0]:right[1]]) == [0, 1]


def test_two_member_split(dm, ctx):
    nodes, order = dm.build_tree(dm.SeqSet(["ACGT", "AGT"], ctx))
    root = nodes[0]
    assert (root[2], root[4], root[5]) == (0, 1, 0)
    assert order[nodes[root[6]][0]] == 1 and order[nodes[root[7]][0]] == 0


def test_duplicates_rejected(dm, ctx):
    with pytest.raises(RuntimeError, match="de-duplicated"):
        dm.build_tree(dm.SeqSet(["ACGT", "ACGT", "TTTT"], ctx))
    # duplicates deep inside a big (sampled) node
    rng = random.Random(4)
    seqs = unique([rand_str(rng, 30) for _ in range(400)])
    seqs.append(seqs[17])
    with pytest.raises(RuntimeError, match="de-duplicated"):
        dm.build_tree(dm.SeqSet(seqs, ctx))


def test_empty_and_single(dm, ctx):
    with pytest.raises(RuntimeError):
        dm.build_tree(dm.SeqSet([], ctx))
    nodes, order = dm.build_tree(dm.SeqSet(["ACGT"], ctx))
    assert nodes.shape[0] == 1 and nodes[0][2] == 0 and nodes[0][6] == -1 and list(order) == [0]


def _same(a, b):
    (na, oa), (nb, ob) = a, b
    assert na.shape == nb.shape
    bad = np.nonzero((na != nb).any(axis=1))[0]
    assert len(bad) == 0, f"first differing node {bad[:3]}: {na[bad[0]]} vs {nb[bad[0]]}"
    assert np.array_equal(oa, ob)


@pytest.mark.parametrize("it", range(8))
def test_random_small_vs_restatement(dm, ctx, orc, it):
    # test_cluster_tree.cpp:223-236 (seed 31)
    rng = random.Random(31 + it)
    seqs = unique([rand_str(rng, rng.randint(4, 24)) for _ in range(2 + rng.randrange(40))])
    if len(seqs) < 2:
        return
    _same(dm.build_tree(dm.SeqSet(seqs, ctx), seed=100 + it), orc.build_tree(seqs, seed=100 + it))


@pytest.mark.parametrize("cap", [100, 16, 2, 5, 128, 200])
def test_caps_vs_reference(dm, ctx, ref, cap):
    rng = random.Random(cap)
    seqs = unique(mutation_families(rng, 6, 60, 60, 0.2))
    ss = dm.SeqSet(seqs, ctx)
    _same(dm.build_tree(ss, seed=5, exact_cap=cap), ref.build_tree(seqs, seed=5, cap=cap))


def test_families_determinism(dm, ctx, ref):
    # test_cluster_tree.cpp:238-265 (seed 41)
    rng = random.Random(41)
    seqs = unique(mutation_families(rng, 6, 25, 30, 0.2))
    ss = dm.SeqSet(seqs, ctx)
    t1 = dm.build_tree(ss, seed=5)
    t2 = dm.build_tree(ss, seed=5)
    _same(t1, t2)
    _same(t1, ref.build_tree(seqs, seed=5))


@pytest.mark.parametrize("bg", ["1", "0"])
@pytest.mark.parametrize("alphabet", ["ACGT", "ARNDCQEGHILKMFPSTWYV"])
def test_medium_vs_reference(dm, ctx, ref, alphabet, bg, monkeypatch):
    """bg: the small subtrees' matrices on the background worker (default) or
    in the foreground after the levels (DM_TREE_BG=0)."""
    monkeypatch.setenv("DM_TREE_BG", bg)
    rng = random.Random(77)
    seqs = unique(mutation_families(rng, 10, 80, 120, 0.1, alphabet))
    ss = dm.SeqSet(seqs, ctx)
    _same(dm.build_tree(ss, seed=42), ref.build_tree(seqs, seed=42))


def test_cfg0_full_vs_reference(dm, ctx, ref):
    data, offs = dm.synth(0)
    seqs = unique(dm.split(data, offs))
    ss = dm.SeqSet(seqs, ctx)
    _same(dm.build_tree(ss, seed=42), ref.build_tree(seqs, seed=42))


def test_cfg3_slice_vs_reference(dm, ctx, ref):
    data, offs = dm.synth(3, scale=0.1)  # 2,000 proteins
    seqs = unique(dm.split(data, offs))
    ss = dm.SeqSet(seqs, ctx)
    _same(dm.build_tree(ss, seed=42), ref.build_tree(seqs, seed=42))


@pytest.mark.parametrize("cache", ["1", "0", "10", "12"])
@pytest.mark.parametrize("bg", ["1", "0"])
def test_distance_cache_vs_reference(dm, ctx, ref, cache, bg, monkeypatch):
    """The build's table of pairs already computed (DistCache): on by default
    (a share of the tree's cells answered without a launch), off
    (DM_TREE_CACHE=0), and forced to 2^10 / 2^12 slots (inserts stop at a
    5/8 load, lookups walk long probe chains). The tree is the reference's
    in every mode, with the small subtrees in the background or not."""
    monkeypatch.setenv("DM_TREE_CACHE", cache)
    monkeypatch.setenv("DM_TREE_BG", bg)
    rng = random.Random(91)
    seqs = unique(mutation_families(rng, 12, 70, 90, 0.12))
    ss = dm.SeqSet(seqs, ctx)
    nodes, order, st = dm.build_tree(ss, seed=42, stats=True)
    _same((nodes, order), ref.build_tree(seqs, seed=42))
    if cache == "0":
        assert st["cells_reused"] == 0
    else:
        assert st["cells_reused"] > 0
    if cache == "1":
        # the reuse the structure guarantees: every big node's center is one
        # of its median candidates, so its sweep's distances to them are known
        assert st["cells_reused"] > 0.05 * (st["cells"] + st["cells_reused"])
