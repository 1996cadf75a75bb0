"""CPU: pin the oracle before trusting it.

The plain-C restatement (oracle/divmsa_oracle.c) is checked against
  * the reference's own known-answer literals (test_distance.cpp:11-28,
    test_pairwise.cpp:13-180, test_cluster_tree.cpp:123-207,
    test_msa_merge.cpp:79-176), restated here;
  * golden vectors produced by the unmodified reference
    (tests/golden/make_golden.py -> tests/golden/*.json);
  * the compiled reference itself (oracle/_ref), when it is present.
"""
import json
import os
import random

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_mt19937_64_known_answer(orc):
    # C++11 [rand.predef]: the 10000th output of a default-seeded mt19937_64
    assert orc.mt64(5489, 10000)[-1] == 9981545732273789042


def test_sample_distinct_properties(orc):
    for seed in range(20):
        s = orc.sample_distinct(seed, 1000, 100)
        assert len(s) == 100 and s == sorted(set(s)) and all(0 <= x < 1000 for x in s)
    assert orc.sample_distinct(1, 5, 10) == [0, 1, 2, 3, 4]


@pytest.mark.parametrize("a,b,d", [
    ("KITTEN", "SITTING", 3), ("", "", 0), ("A", "", 1), ("", "ACGT", 4), ("ACGT", "ACGT", 0), ("A", "C", 1),
    ("AC", "CA", 2), ("ABCXDEF", "ABCYDEF", 1), ("AAAA", "AAA", 1), ("XXXABC", "ABC", 3), ("ABC", "ABCXXX", 3)])
def test_levenshtein_literals(orc, a, b, d):
    assert orc.levenshtein(a, b) == d


def test_levenshtein_golden(orc):
    for a, b, d in load("lev.json"):
        assert orc.levenshtein(a, b) == d


def lev_rec(a, b):
    # test_support.hpp:24-50: memoized recursion from the definition
    from functools import lru_cache

    @lru_cache(maxsize=None)
    def f(i, j):
        if i == 0:
            return j
        if j == 0:
            return i
        return min(f(i - 1, j) + 1, f(i, j - 1) + 1, f(i - 1, j - 1) + (a[i - 1] != b[j - 1]))
    return f(len(a), len(b))


def test_levenshtein_vs_definition(orc):
    rng = random.Random(7)
    for _ in range(200):
        a = "".join(rng.choice("ACGT") for _ in range(rng.randrange(13)))
        b = "".join(rng.choice("ACGT") for _ in range(rng.randrange(13)))
        assert orc.levenshtein(a, b) == lev_rec(a, b)


def test_nw_literals(orc):
    t = orc.table("nt")
    r = orc.nw_align("ACGT", "AGT", t, -10, -1)
    assert (r["score"], r["aligned_a"], r["aligned_b"], r["gaps_into_b"]) == (-8, "ACGT", "A-GT", [1])
    assert orc.nw_align("A", "C", t, -10, -1)["score"] == -1
    r = orc.nw_align("AA", "A", t, -10, -1)
    assert (r["score"], r["aligned_b"], r["gaps_into_b"]) == (-10, "-A", [0])
    r = orc.nw_align("A-G", "AG", t, -10, -1)
    assert (r["score"], r["aligned_a"], r["aligned_b"], r["gaps_into_b"]) == (-9, "A-G", "A-G", [1])
    assert orc.nw_align("A-G", "A-G", t, -10, -1)["score"] == 2
    r = orc.nw_align("ACGT", "AGT", t, 0, -1)  # flat
    assert (r["score"], r["aligned_b"]) == (2, "A-GT")


def score_moves(a, b, moves, table, osur, ext):
    # test_support.hpp:57-82
    s, i, j, prev = 0, 0, 0, "M"
    for mv in moves:
        if mv == "M":
            s += int(table[ord(a[i]) * 128 + ord(b[j])])
            i += 1
            j += 1
        else:
            if mv != prev:
                s += osur
            s += ext
            if mv == "X":
                i += 1
            else:
                j += 1
        prev = mv
    return s


def enumerate_best(a, b, table, osur, ext):
    # test_support.hpp:86-113: exhaustive monotone paths
    best = [None]

    def walk(i, j, moves):
        if i == len(a) and j == len(b):
            v = score_moves(a, b, moves, table, osur, ext)
            best[0] = v if best[0] is None else max(best[0], v)
            return
        if i < len(a) and j < len(b):
            walk(i + 1, j + 1, moves + "M")
        if i < len(a):
            walk(i + 1, j, moves + "X")
        if j < len(b):
            walk(i, j + 1, moves + "Y")
    walk(0, 0, "")
    return best[0]


def test_nw_optimal_by_enumeration(orc):
    # test_pairwise.cpp:189-217 (seed 11) / acceptance #2
    rng = random.Random(11)
    t = orc.table("nt")
    for _ in range(60):
        a = "".join(rng.choice("ACGT") for _ in range(1 + rng.randrange(5)))
        b = "".join(rng.choice("ACGT") for _ in range(1 + rng.randrange(5)))
        for osur, ext in ((-10, -1), (-3, -2), (0, -1)):
            r = orc.nw_align(a, b, t, osur, ext)
            assert r["score"] == enumerate_best(a, b, t, osur, ext)
            moves = "".join("Y" if x == "-" else ("X" if y == "-" else "M")
                            for x, y in zip(r["aligned_a"], r["aligned_b"]))
            assert score_moves(a, b, moves, t, osur, ext) == r["score"]
            assert r["aligned_a"].replace("-", "") == a and r["aligned_b"].replace("-", "") == b


def test_nw_golden(orc):
    for c in load("nw.json"):
        t = orc.table(c["kind"], c["ge"])
        r = orc.nw_align(c["a"], c["b"], t, 0 if c["flat"] else c["go"], c["ge"])
        for k in ("score", "aligned_a", "aligned_b", "gaps_into_a", "gaps_into_b"):
            assert r[k] == c[k], (c["a"], c["b"], k)


def test_tree_literals(orc):
    nodes, order = orc.build_tree(["AAAA", "AAAT", "TTTT"])
    assert tuple(nodes[0][[2, 3, 4, 5]]) == (1, 3, 2, 0)
    nodes, order = orc.build_tree(["ACGT", "AGT"])
    assert tuple(nodes[0][[2, 4, 5]]) == (0, 1, 0)
    assert orc.geometric_median(["AAAA", "AAAT", "TTTT"], [0, 1, 2], 42) == 1
    assert orc.geometric_median(["AAAA", "TTTT"], [1, 0], 42) == 0
    with pytest.raises(RuntimeError, match="de-duplicated"):
        orc.build_tree(["ACGT", "ACGT", "TTTT"])


def test_tree_golden(orc):
    for c in load("tree.json"):
        nodes, order = orc.build_tree(c["seqs"], seed=c["seed"], cap=c["cap"])
        assert nodes.tolist() == c["nodes"]
        assert order.tolist() == c["order"]


def test_insert_gap_columns_literals(orc):
    assert orc.insert_gap_columns(["AC", "GT"], [1]) == ["A-C", "G-T"]
    assert orc.insert_gap_columns(["AB"], [0, 0, 2]) == ["--AB-"]
    with pytest.raises(ValueError):
        orc.insert_gap_columns(["AB"], [3])


def test_msa_golden(orc):
    for c in load("msa_small.json"):
        nodes, order = orc.build_tree(c["seqs"], seed=c["seed"])
        assert order.tolist() == c["order"]
        rows, w = orc.align_all(c["seqs"], nodes, order, orc.table(c["kind"]), -10, -1)
        assert w == c["width"] and rows == c["rows"]


def test_restatement_vs_compiled_reference(orc, ref):
    rng = random.Random(3)
    seqs = list(dict.fromkeys("".join(rng.choice("ACGT") for _ in range(rng.randint(5, 60))) for _ in range(150)))
    n1, o1 = orc.build_tree(seqs, seed=9)
    n2, o2 = ref.build_tree(seqs, seed=9)
    assert np.array_equal(n1, n2) and np.array_equal(o1, o2)
    rows, w = orc.align_all(seqs, n1, o1, orc.table("nt"), -10, -1)
    r = ref.msa(seqs, seed=9)
    assert rows == r["rows"] and w == r["width"]


def test_reference_metrics_pins(ref):
    """The compiled reference's metrics (the oracle of tests/test_metrics_gpu.py)
    against test_metrics.cpp:74-128."""
    assert ref.gap_percent(["AC-", "A-C"]) == pytest.approx(100.0 / 3)
    assert ref.gap_percent(["--", "--"]) == 100.0
    assert ref.p_score("AC-T", "AG-T") == pytest.approx(1.0 / 3)
    assert ref.p_score("A---", "-CCC") == 1.0
    assert ref.distortion_pair("AC--", "--GT", "AC", "GT") == pytest.approx(2.0)
    with pytest.raises(ValueError, match="identical"):
        ref.distortion_pair("ACGT", "ACGT", "ACGT", "ACGT")
    r = ref.evaluate(["AC-T", "AG-T"], [0, 1], ["ACT", "AGT"], 100, 100, 42)
    assert (r["width"], r["sample_size"], r["pair_count"], r["seed"]) == (4, 2, 1, 42)
    assert r["p_avg"] == pytest.approx(1.0 / 3) and r["distortion"] == pytest.approx(1.0)
    with pytest.raises(ValueError, match="empty alignment"):
        ref.evaluate([], [], [])
