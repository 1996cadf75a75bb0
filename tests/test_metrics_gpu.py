"""Parity of the GPU quality metrics (divmsa::evaluate).

Pins restate /root/reference/proj/tests/test_metrics.cpp:74-200 and
acceptance.cpp:247-320; every report is compared field by field (doubles
bit-exactly) with the compiled reference's divmsa::evaluate."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("width", "stretch", "gap_percent", "distortion", "p_min", "p_avg", "p_max", "sample_size",
          "pair_count", "seed", "zero_distance_pairs")


def same_report(got, want):
    for f in FIELDS:
        assert got[f] == want[f], (f, got[f], want[f])


def rand_str(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


def test_helper_pins(dm, ctx):
    # test_metrics.cpp:74-110
    assert dm.gap_percent(["AC-", "A-C"], ctx) == pytest.approx(100.0 / 3)
    assert dm.gap_percent(["ACGT"], ctx) == 0.0
    assert dm.gap_percent(["--", "--"], ctx) == 100.0
    with pytest.raises(ValueError, match="empty alignment"):
        dm.gap_percent([], ctx)
    assert dm.p_score("AC-T", "AG-T", ctx) == pytest.approx(1.0 / 3)
    assert dm.p_score("A---", "-CCC", ctx) == 1.0
    assert dm.p_score("ACGT", "ACGT", ctx) == 0.0
    assert dm.p_score("AAAA", "CCCC", ctx) == 1.0
    with pytest.raises(ValueError, match="equal-length"):
        dm.p_score("AC", "A", ctx)
    assert dm.distortion_pair("ACGT", "A-GT", "ACGT", "AGT", ctx) == 1.0
    assert dm.distortion_pair("AC--", "--GT", "AC", "GT", ctx) == pytest.approx(2.0)
    with pytest.raises(ValueError, match="identical"):
        dm.distortion_pair("ACGT", "ACGT", "ACGT", "ACGT", ctx)
    assert dm.hamming_aligned("AC-T", "AG-A", ctx) == 2


def test_helpers_match_reference_on_long_rows(dm, ctx, ref):
    rng = random.Random(77)
    for n in (1, 15, 16, 17, 31, 32, 33, 100, 511, 512, 513, 4000):
        a = rand_str(rng, n, "ACGT--")
        b = rand_str(rng, n, "ACGT--")
        assert dm.p_score(a, b, ctx) == ref.p_score(a, b)
        assert dm.hamming_aligned(a, b, ctx) == ref.hamming_aligned(a, b)
        rows = [rand_str(rng, n, "AC-") for _ in range(rng.randint(1, 9))]
        assert dm.gap_percent(rows, ctx) == ref.gap_percent(rows)


def test_evaluate_two_rows(dm, ctx):
    # test_metrics.cpp:112-128
    m = dm.Msa(rows=["AC-T", "AG-T"], row_to_sequence=np.array([0, 1], dtype=np.uint32), width=4)
    r = dm.evaluate(m, ["ACT", "AGT"], 100, 100, 42, ctx)
    assert r["width"] == 4 and r["sample_size"] == 2 and r["pair_count"] == 1 and r["seed"] == 42
    assert r["stretch"] == pytest.approx(4.0 / 3)
    assert r["p_min"] == r["p_avg"] == r["p_max"] == pytest.approx(1.0 / 3)
    assert r["distortion"] == pytest.approx(1.0)
    assert r["zero_distance_pairs"] == 0


def test_evaluate_caps(dm, ctx, ref):
    # test_metrics.cpp:170-191: row and pair caps
    rng = random.Random(111)
    rows = [rand_str(rng, 10) for _ in range(20)]
    m = dm.Msa(rows=rows, row_to_sequence=np.arange(20, dtype=np.uint32), width=10)
    r = dm.evaluate(m, rows, 5, 3, 42, ctx)
    assert r["sample_size"] == 5 and r["pair_count"] == 3
    same_report(r, ref.evaluate(rows, np.arange(20), rows, 5, 3, 42))
    tiny = dm.evaluate(m, rows, 1, 100, 42, ctx)
    assert tiny["sample_size"] == 1 and tiny["pair_count"] == 0 and tiny["p_avg"] == 0.0
    assert tiny["distortion"] == 0.0
    none = dm.evaluate(m, rows, 100, 0, 42, ctx)
    assert none["sample_size"] == 20 and none["pair_count"] == 0


def test_evaluate_errors(dm, ctx):
    with pytest.raises(ValueError, match="cannot evaluate an empty alignment"):
        dm.evaluate(dm.Msa(rows=[], row_to_sequence=np.zeros(0, dtype=np.uint32), width=0), [], ctx=ctx)
    with pytest.raises(ValueError, match="gap_percent of an empty alignment"):
        dm.evaluate(dm.Msa(rows=[""], row_to_sequence=np.zeros(1, dtype=np.uint32), width=0), [""], ctx=ctx)


@pytest.mark.parametrize("seed", [1, 9, 42])
def test_evaluate_random_msas_vs_reference(dm, ctx, ref, seed):
    """GPU MSAs of random families (duplicated raws included), several
    sample sizes / budgets: every field identical to the reference."""
    rng = random.Random(seed)
    base = rand_str(rng, rng.randint(30, 300))
    seqs = []
    for _ in range(rng.randint(20, 90)):
        s = list(base)
        for _ in range(rng.randint(0, 30)):
            p = rng.randrange(len(s))
            if rng.random() < 0.6:
                s[p] = rng.choice("ACGT")
            elif rng.random() < 0.5 and len(s) > 5:
                del s[p]
            else:
                s.insert(p, rng.choice("ACGT"))
        seqs.append("".join(s))
    seqs = list(dict.fromkeys(seqs))
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide())
    # raws indexed by row_to_sequence; duplicate a few raws so zero-distance pairs occur
    raws = list(seqs)
    rts = np.array(m.row_to_sequence, dtype=np.uint32)
    for k in range(0, len(rts), 7):
        raws.append(raws[int(rts[k])])
        rts[k] = len(raws) - 1
    mm = dm.Msa(rows=m.rows, row_to_sequence=rts, width=m.width)
    for ss, pb in ((10000, 100000), (len(seqs) // 2, 50), (7, 1000000)):
        same_report(dm.evaluate(mm, raws, ss, pb, seed, ctx), ref.evaluate(m.rows, rts, raws, ss, pb, seed))


def test_evaluate_cfg0_vs_reference(dm, ctx, ref):
    """cfg0 full MSA (1,000 rows): default sample (all rows), 100,000 of the
    499,500 pairs sampled."""
    data, offs = dm.synth(0, 1.0)
    seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide())
    got = dm.evaluate(m, seqs, ctx=ctx)
    want = ref.evaluate(m.rows, m.row_to_sequence, seqs)
    same_report(got, want)
    assert got["pair_count"] == 100000
