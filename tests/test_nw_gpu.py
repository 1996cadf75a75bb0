"""Parity of the GPU pairwise aligner (K5/K6) with nw_align.

Pins restate /root/reference/proj/tests/test_pairwise.cpp:13-233 and
acceptance.cpp:130-159; random sweeps compare score, aligned strings and gap
lists with the C restatement and the compiled reference."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu



@pytest.fixture(autouse=True, params=["ring", "seq", "clu2", "clu8"])
def nw_kernel(request, monkeypatch):
    """Every test runs on every forward kernel: the multi-warp ring kernel
    (nw_fwd.cuh), the one-warp-per-alignment throughput kernel (nw_seq.cuh,
    256-scaled tags, query profiles, short last bands; batches of >= 16
    alignments per SM) and the cluster kernel (nw_clu.cuh, 128-row bands
    across 2 or 8 CTAs with distributed-shared-memory rings and global wrap
    rows; batches too small to fill the GPU one alignment per CTA)."""
    monkeypatch.setenv("DM_NW_SEQ", "1" if request.param == "seq" else "0")
    monkeypatch.setenv("DM_NW_CLU", {"clu2": "2", "clu8": "8"}.get(request.param, "0"))
    return request.param

def rand_str(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


def as_tuple(r):
    if isinstance(r, dict):
        return (r["score"], r["aligned_a"], r["aligned_b"], list(r["gaps_into_a"]), list(r["gaps_into_b"]))
    return (r.score, r.aligned_a, r.aligned_b, list(r.gaps_into_a), list(r.gaps_into_b))


def test_scheme_values(dm):
    s = dm.ScoringScheme.nucleotide()
    assert (s.score("A", "A"), s.score("A", "R"), s.score("A", "Y"), s.score("U", "T"), s.score("N", "C")) == (1, 1, -1, 1, 1)
    assert s.score("-", "A") == s.gap_extend() and s.score("-", "-") == 0
    assert s.has("-") and s.has("W") and not s.has("E")
    assert (s.gap_open(), s.gap_extend(), s.open_surcharge()) == (-10, -1, -10)
    assert dm.ScoringScheme.nucleotide(-10, -1, "flat").open_surcharge() == 0
    p = dm.ScoringScheme.protein()
    assert (p.score("A", "A"), p.score("W", "W"), p.score("A", "R"), p.score("R", "A")) == (4, 11, -1, -1)
    assert (p.score("E", "Z"), p.score("*", "*"), p.score("W", "*"), p.score("-", "W")) == (4, 1, -4, -1)


def test_scheme_tables_match_reference(dm, ref):
    for kind, ctor in (("nt", dm.ScoringScheme.nucleotide), ("aa", dm.ScoringScheme.protein)):
        for go, ge, mode in ((-10, -1, "affine"), (-3, -2, "flat")):
            t, osur = ref.scheme_table(kind, go, ge, mode == "flat")
            s = ctor(go, ge, mode)
            assert np.array_equal(s.table, t) and s.open_surcharge() == osur


def test_scheme_validation(dm):
    m2 = [1, -1, -1, 1]
    dm.ScoringScheme.custom("AC", m2, -5, -1)
    for args in (("", [], -5, -1), ("ACG", m2, -5, -1), ("AC", m2, 5, -1), ("AC", m2, -5, 1), ("AC", m2, -1, -5),
                 ("A-", m2, -5, -1), ("AA", m2, -5, -1)):
        with pytest.raises(ValueError):
            dm.ScoringScheme.custom(*args)
    with pytest.raises(ValueError, match="not symmetric"):
        dm.ScoringScheme.custom("AC", [1, -1, -2, 1], -5, -1)


def test_alignment_pins(dm, ctx):
    r = dm.nw_align("ACGT", "AGT", ctx=ctx)
    assert (r.score, r.aligned_a, r.aligned_b, r.gaps_into_a, r.gaps_into_b) == (-8, "ACGT", "A-GT", [], [1])
    r = dm.nw_align("A", "C", ctx=ctx)
    assert (r.score, r.aligned_a, r.aligned_b) == (-1, "A", "C")
    r = dm.nw_align("AA", "A", ctx=ctx)  # tie: leading gap
    assert (r.score, r.aligned_a, r.aligned_b, r.gaps_into_b) == (-10, "AA", "-A", [0])
    r = dm.nw_align("A-G", "AG", ctx=ctx)  # pre-existing gaps are ordinary symbols
    assert (r.score, r.aligned_a, r.aligned_b, r.gaps_into_a, r.gaps_into_b) == (-9, "A-G", "A-G", [], [1])
    r = dm.nw_align("A-G", "A-G", ctx=ctx)
    assert (r.score, r.gaps_into_a, r.gaps_into_b) == (2, [], [])
    r = dm.nw_align("ACGT", "AGT", gap_mode="flat", ctx=ctx)
    assert (r.score, r.aligned_b) == (2, "A-GT")
    assert "PairwiseResult" in repr(r)


def test_input_validation(dm, ctx):
    for a, b in (("", "A"), ("A", ""), ("AQ", "A")):
        with pytest.raises(ValueError):
            dm.nw_align(a, b, ctx=ctx)
    with pytest.raises(ValueError):
        dm.nw_align("AC", "A", alphabet="dna", ctx=ctx)
    with pytest.raises(ValueError):
        dm.nw_align("AC", "A", gap_mode="linear", ctx=ctx)


def test_small_random_vs_restatement(dm, ctx, orc):
    """test_pairwise.cpp:189-217 (seed 11): 200 pairs x 3 schemes, plus gapped inputs."""
    rng = random.Random(11)
    schemes = [(-10, -1, "affine"), (-3, -2, "affine"), (-10, -1, "flat")]
    for go, ge, mode in schemes:
        sc = dm.ScoringScheme.nucleotide(go, ge, mode)
        pairs = [(rand_str(rng, 1 + rng.randrange(6)), rand_str(rng, 1 + rng.randrange(6))) for _ in range(200)]
        pairs += [(rand_str(rng, 1 + rng.randrange(9), "ACGT-"), rand_str(rng, 1 + rng.randrange(9), "ACGTN-"))
                  for _ in range(200)]
        got = dm.nw_batch(pairs, sc, ctx)
        table = orc.table("nt", ge)
        for (a, b), r in zip(pairs, got):
            assert as_tuple(r) == as_tuple(orc.nw_align(a, b, table, sc.open_surcharge(), ge)), (a, b, mode)


def test_self_alignment_protein(dm, ctx):
    rng = random.Random(12)
    sc = dm.ScoringScheme.protein()
    for _ in range(20):
        s = rand_str(rng, 1 + rng.randrange(30), "ARNDCQEG")
        r = dm.nw_align(s, s, alphabet="aa", ctx=ctx)
        assert r.aligned_a == s and r.aligned_b == s and not r.gaps_into_a and not r.gaps_into_b
        assert r.score == sum(sc.score(c, c) for c in s)


@pytest.mark.parametrize("kind", ["nt", "aa"])
def test_pass_boundaries_vs_reference(dm, ctx, ref, kind):
    """Lengths straddling the 16-row lane and 512-row pass boundaries."""
    rng = random.Random(7 if kind == "nt" else 8)
    alpha = "ACGT" if kind == "nt" else "ARNDCQEGHILKMFPSTWYV"
    sc = dm.ScoringScheme.nucleotide() if kind == "nt" else dm.ScoringScheme.protein()
    pairs = []
    for la in (1, 2, 15, 16, 17, 31, 32, 33, 511, 512, 513, 1023, 1024, 1025, 1600):
        a = rand_str(rng, la, alpha + "-")
        b = list(a)
        for _ in range(max(1, la // 10)):
            p = rng.randrange(len(b) + 1)
            op = rng.randrange(3)
            if op == 0 and b:
                b[min(p, len(b) - 1)] = rng.choice(alpha)
            elif op == 1 and len(b) > 1:
                del b[min(p, len(b) - 1)]
            else:
                b.insert(p, rng.choice(alpha))
        pairs.append((a, "".join(b) or "A"))
        pairs.append((rand_str(rng, max(1, la // 3), alpha), rand_str(rng, la + 5, alpha)))
    got = dm.nw_batch(pairs, sc, ctx)
    for (a, b), r in zip(pairs, got):
        assert as_tuple(r) == as_tuple(ref.nw_align(a, b, kind)), (len(a), len(b))


def test_flat_and_custom_vs_reference(dm, ctx, ref):
    rng = random.Random(99)
    syms = "ACGTX"
    mat = [[(5 if i == j else -3 - (i + j) % 3) for j in range(5)] for i in range(5)]
    flatm = [v for row in mat for v in row]
    pairs = [(rand_str(rng, rng.randint(1, 300), syms + "-"), rand_str(rng, rng.randint(1, 300), syms + "-"))
             for _ in range(60)]
    for mode in ("affine", "flat"):
        sc = dm.ScoringScheme.custom(syms, flatm, -7, -2, mode)
        got = dm.nw_batch(pairs, sc, ctx)
        for (a, b), r in zip(pairs, got):
            want = ref.nw_align(a, b, "custom", -7, -2, mode == "flat", symbols=syms, matrix=flatm)
            assert as_tuple(r) == as_tuple(want)


def test_wide_scores_use_int64_path(dm, ctx, ref):
    """|scores| near the int16 limit force the int64 kernel; still bit-exact."""
    rng = random.Random(5)
    syms = "ACGT"
    flatm = [30000 if i == j else -29000 for i in range(4) for j in range(4)]
    sc = dm.ScoringScheme.custom(syms, flatm, -32000, -20000)
    pairs = [(rand_str(rng, rng.randint(200, 900)), rand_str(rng, rng.randint(200, 900))) for _ in range(8)]
    got = dm.nw_batch(pairs, sc, ctx)
    for (a, b), r in zip(pairs, got):
        want = ref.nw_align(a, b, "custom", -32000, -20000, False, symbols=syms, matrix=flatm)
        assert as_tuple(r) == as_tuple(want)


def test_cfg1_nw_sample_vs_reference(dm, ctx, ref):
    """NW micro-benchmark inputs (cfg1 pairs) vs the reference."""
    data, offs = dm.synth(1, scale=0.0002)  # 200 pairs
    seqs = dm.split(data, offs)
    pairs = [(seqs[2 * i].decode(), seqs[2 * i + 1].decode()) for i in range(len(seqs) // 2)][:64]
    got, st = dm.nw_batch(pairs, dm.ScoringScheme.nucleotide(), ctx, stats=True)
    assert st["cells"] == sum(len(a) * len(b) for a, b in pairs)
    for (a, b), r in zip(pairs, got):
        assert as_tuple(r) == as_tuple(ref.nw_align(a, b))


@pytest.mark.timeout(600)
def test_more_bands_than_warps_vs_reference(dm, ctx, ref):
    """Alignments of 2..19 bands (512 rows each; more than 8 bands = several
    rounds of the 8-warp CTA, the round-to-round row going through global
    memory) and every warps-per-alignment group, including int64 scores."""
    rng = random.Random(12)
    pairs = []
    for la, lb in ((1000, 900), (1500, 1600), (2000, 1900), (4100, 600), (4700, 4800), (5200, 300),
                   (9000, 8800), (9700, 2500)):
        a = rand_str(rng, la)
        b = list(a[:lb]) + [rng.choice("ACGT") for _ in range(max(0, lb - la))]
        for _ in range(lb // 15):
            b[rng.randrange(len(b))] = rng.choice("ACGT")
        pairs.append((a, "".join(b)))
    got = dm.nw_batch(pairs, dm.ScoringScheme.nucleotide(), ctx)
    for (a, b), r in zip(pairs, got):
        assert as_tuple(r) == as_tuple(ref.nw_align(a, b)), (len(a), len(b))
    syms = "ACGT"
    flatm = [30000 if i == j else -29000 for i in range(4) for j in range(4)]
    sc = dm.ScoringScheme.custom(syms, flatm, -32000, -20000)
    big = [pairs[4], pairs[6]]
    for (a, b), r in zip(big, dm.nw_batch(big, sc, ctx)):
        want = ref.nw_align(a, b, "custom", -32000, -20000, False, symbols=syms, matrix=flatm)
        assert as_tuple(r) == as_tuple(want)


@pytest.mark.parametrize("kind", ["nt", "nt-iupac", "aa"])
def test_last_band_heights_vs_reference(dm, ctx, ref, kind, nw_kernel):
    """Rows around the last band's 128 / 256 / 512-row forms (4, 8, 16 rows per
    lane) and column alphabets with and without gaps (query profile for <= 8
    column symbols, table otherwise)."""
    rng = random.Random({"nt": 1, "nt-iupac": 2, "aa": 3}[kind])
    alpha = {"nt": "ACGT", "nt-iupac": "ACGTURYSWKMBDHVN", "aa": "ARNDCQEGHILKMFPSTWYV"}[kind]
    sc = dm.ScoringScheme.protein() if kind == "aa" else dm.ScoringScheme.nucleotide()
    pairs = []
    for la in (1, 4, 5, 127, 128, 129, 255, 256, 257, 383, 384, 385, 511, 512, 513, 640, 641, 768, 769,
               1023, 1024, 1025, 1153, 1300):
        a = rand_str(rng, la, alpha)
        b = list(a)
        for _ in range(max(1, la // 12)):
            p = rng.randrange(len(b))
            op = rng.randrange(4)
            if op == 0:
                b[p] = rng.choice(alpha)
            elif op == 1 and len(b) > 1:
                del b[p]
            elif op == 2:
                b.insert(p, rng.choice(alpha))
            else:
                b[p] = "-"
        pairs.append((a, "".join(b)))
        pairs.append(("".join(b), a[: max(1, la - 7)]))
    got = dm.nw_batch(pairs, sc, ctx)
    for (a, b), r in zip(pairs, got):
        assert as_tuple(r) == as_tuple(ref.nw_align(a, b, "aa" if kind == "aa" else "nt")), (len(a), len(b))


def test_trace_budget_chunks_vs_reference(dm, ctx, ref, monkeypatch, nw_kernel):
    """A small trace budget splits the batch into many chunks (forward +
    traceback per chunk, the trace buffer reused); results unchanged."""
    monkeypatch.setenv("DM_NW_TRACE_GB", "0.002")
    rng = random.Random(77)
    pairs = []
    for _ in range(40):
        la = rng.randint(200, 1400)
        a = rand_str(rng, la)
        b = list(a)
        for _ in range(la // 20):
            b[rng.randrange(len(b))] = rng.choice("ACGT")
        pairs.append((a, "".join(b[: max(1, la - rng.randint(0, 50))])))
    got = dm.nw_batch(pairs, dm.ScoringScheme.nucleotide(), ctx)
    for (a, b), r in zip(pairs, got):
        assert as_tuple(r) == as_tuple(ref.nw_align(a, b)), (len(a), len(b))
