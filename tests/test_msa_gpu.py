"""Parity of the GPU MSA builder (merge scheduler, K7/K8) and the pipeline.

Pins restate /root/reference/proj/tests/test_msa_merge.cpp:79-219,
tests/python/test_smoke.py:70-107 and acceptance.cpp:74-125; every MSA is
compared byte for byte with the compiled reference."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu



@pytest.fixture(autouse=True, params=["default", "seq", "ring"])
def nw_kernel(request, monkeypatch):
    """MSA parity with the merges on the library's own kernel choice per level
    (cluster / ring / throughput by batch size), on the throughput kernel
    only, and on the ring kernel only (see test_nw_gpu.py)."""
    if request.param == "seq":
        monkeypatch.setenv("DM_NW_SEQ", "1")
    elif request.param == "ring":
        monkeypatch.setenv("DM_NW_SEQ", "0")
        monkeypatch.setenv("DM_NW_CLU", "0")
    return request.param

def rand_str(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


def unique(seqs):
    out, seen = [], set()
    for s in seqs:
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


def families(rng, nfam, per, base, rate, alphabet="ACGT"):
    out = []
    for _ in range(nfam):
        anc = rand_str(rng, base, alphabet)
        for _ in range(per):
            s = list(anc)
            for _ in range(max(1, int(rate * base))):
                k, p = rng.randrange(3), rng.randrange(len(s))
                if k == 0:
                    s[p] = rng.choice(alphabet)
                elif k == 1 and len(s) > 4:
                    del s[p]
                else:
                    s.insert(p, rng.choice(alphabet))
            out.append("".join(s))
    return out


def test_insert_gap_columns_pins(dm, ctx):
    assert dm.insert_gap_columns(["AC", "GT"], [1], ctx) == ["A-C", "G-T"]
    assert dm.insert_gap_columns(["AC"], [], ctx) == ["AC"]
    assert dm.insert_gap_columns(["AB"], [0, 0, 2], ctx) == ["--AB-"]
    with pytest.raises(ValueError, match="width"):
        dm.insert_gap_columns(["AB"], [3], ctx)
    with pytest.raises(ValueError):
        dm.insert_gap_columns(["ABC"], [2, 1], ctx)


def test_insert_gap_columns_random(dm, ctx, orc):
    rng = random.Random(51)
    for _ in range(50):
        width, rows = 1 + rng.randrange(12), 1 + rng.randrange(4)
        block = [rand_str(rng, width, "ACGT-") for _ in range(rows)]
        pos = sorted(rng.randrange(width + 1) for _ in range(rng.randrange(6)))
        assert dm.insert_gap_columns(block, pos, ctx) == orc.insert_gap_columns(block, pos)


def _ref_msa(ref, seqs, kind="nt", **kw):
    return ref.msa(seqs, kind=kind, **kw)


def _check_same(m, r):
    assert m.width == r["width"]
    assert np.array_equal(m.row_to_sequence, r["row_seq"])
    bad = [i for i, (x, y) in enumerate(zip(m.rows, r["rows"])) if x != y]
    assert not bad, f"{len(bad)} rows differ, first {bad[0]}"


def test_merge_pins(dm, ctx):
    # test_msa_merge.cpp:146-176 via a whole (two-sequence) tree
    m = dm.msa(dm.SeqSet(["ACGT", "AGT"], ctx), dm.ScoringScheme.nucleotide())
    assert m.width == 4 and sorted(m.rows) == ["A-GT", "ACGT"]
    m = dm.msa(dm.SeqSet(["AC", "AG"], ctx), dm.ScoringScheme.nucleotide())
    assert m.width == 2 and sorted(m.rows) == ["AC", "AG"]


@pytest.mark.parametrize("it", range(6))
def test_random_vs_reference(dm, ctx, ref, it):
    # test_msa_merge.cpp:178-203 (seed 61) shapes
    rng = random.Random(61 + it)
    seqs = unique([rand_str(rng, rng.randint(4, 30)) for _ in range(3 + rng.randrange(25))])
    if len(seqs) < 2:
        return
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide())
    _check_same(m, _ref_msa(ref, seqs))
    for r, row in zip(m.row_to_sequence, m.rows):
        assert row.replace("-", "") == seqs[r]


def test_align_all_given_tree(dm, ctx, ref):
    rng = random.Random(71)
    seqs = unique(families(rng, 5, 20, 40, 0.2))
    r = _ref_msa(ref, seqs)
    ss = dm.SeqSet(seqs, ctx)
    m = dm.align_all(ss, r["nodes"], r["order"], dm.ScoringScheme.nucleotide())
    _check_same(m, r)


@pytest.mark.parametrize("mode", ["affine", "flat"])
def test_families_vs_reference(dm, ctx, ref, mode):
    rng = random.Random(1008)
    seqs = unique(families(rng, 30, 20, 70, 0.15))
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide(-10, -1, mode))
    _check_same(m, _ref_msa(ref, seqs, flat=(mode == "flat")))


def test_protein_vs_reference(dm, ctx, ref):
    rng = random.Random(3)
    seqs = unique(families(rng, 8, 40, 150, 0.1, "ARNDCQEGHILKMFPSTWYV"))
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.protein())
    _check_same(m, _ref_msa(ref, seqs, kind="aa"))


@pytest.mark.timeout(900)
def test_long_sequences_vs_reference(dm, ctx, ref, nw_kernel):
    """~3,800-residue families: merges of more than 4,096 rows (cluster kernel
    rounds with the row hand-off reused in place, ring-kernel wrap rows),
    traces of several hundred MB, byte-identical to the reference."""
    rng = random.Random(3800)
    seqs = unique(families(rng, 4, 10, 3800, 0.03))
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide())
    _check_same(m, _ref_msa(ref, seqs))
    assert m.width > 4096


def test_cfg0_full_vs_reference(dm, ctx, ref):
    data, offs = dm.synth(0)
    seqs = unique([s.decode() for s in dm.split(data, offs)])
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.nucleotide())
    _check_same(m, _ref_msa(ref, seqs))


def test_cfg3_slice_vs_reference(dm, ctx, ref):
    data, offs = dm.synth(3, scale=0.05)
    seqs = unique([s.decode() for s in dm.split(data, offs)])
    m = dm.msa(dm.SeqSet(seqs, ctx), dm.ScoringScheme.protein())
    _check_same(m, _ref_msa(ref, seqs, kind="aa"))


def test_align_pipeline_pins(dm, ctx):
    # tests/python/test_smoke.py:70-92
    seqs = ["ACGTACGT", "ACTTACGT", "ACGT", "ACGTACGT"]
    rows = dm.align(seqs, seed=7, ctx=ctx)
    assert len(rows) == 4 and len({len(r) for r in rows}) == 1
    assert all(r.replace("-", "") == s for r, s in zip(rows, seqs))
    assert rows[0] == rows[3]
    rows = dm.align(["MKVLAARNDE", "MKVLAARNDW", "MKVARNDE"], ctx=ctx)
    assert [r.replace("-", "") for r in rows] == ["MKVLAARNDE", "MKVLAARNDW", "MKVARNDE"]


def test_align_pipeline_vs_reference(dm, ctx, ref):
    # acceptance.cpp:74-125 (seed 1001): random datasets, both alphabets, input order
    rng = random.Random(1001)
    for ds in range(12):
        protein = ds % 2 == 1
        seqs = [rand_str(rng, rng.randint(5, 120), "ARNDCQEGHILKMFPSTWYV" if protein else "ACGT")
                for _ in range(10 + rng.randrange(120))]
        seqs += seqs[:3]  # duplicates re-expand onto their representative's row
        got = dm.align(seqs, ctx=ctx)
        assert got == ref.align(seqs)


def test_align_errors(dm, ctx):
    with pytest.raises(RuntimeError, match="no sequences"):
        dm.align([], ctx=ctx)
    with pytest.raises(ValueError):
        dm.align(["ACGT"], gap_open=-1, gap_extend=-5, ctx=ctx)
    with pytest.raises(RuntimeError, match="outside the nucleotide alphabet"):
        dm.align(["ACGT", "ACGE"], alphabet="nt", ctx=ctx)
    with pytest.raises(RuntimeError, match="gap symbol"):
        dm.align(["ACGT", "AC-T"], alphabet="nt", ctx=ctx)
    with pytest.raises(ValueError):
        dm.align(["ACGT"], gap_mode="linear", ctx=ctx)


def test_align_all_rejects_malformed_trees(dm, ctx):
    seqs = ["ACGT", "AGT", "ACCT", "TTGA"]
    ss = dm.SeqSet(seqs, ctx)
    nodes, order = dm.build_tree(ss)
    sc = dm.ScoringScheme.nucleotide()
    assert len(dm.align_all(ss, nodes, order, sc).rows) == 4
    bad = nodes.copy()
    bad[0, dm.NODE_FIELDS.index("left")] = 99
    with pytest.raises(ValueError, match="invalid cluster tree"):
        dm.align_all(ss, bad, order, sc)
    bad = nodes.copy()
    bad[1, dm.NODE_FIELDS.index("center")] = 17
    with pytest.raises(ValueError, match="invalid cluster tree"):
        dm.align_all(ss, bad, order, sc)
    with pytest.raises(ValueError, match="permutation"):
        dm.align_all(ss, nodes, [0, 0, 1, 2], sc)
    with pytest.raises(ValueError, match="2n-1"):
        dm.align_all(ss, nodes[:5], order, sc)


def test_align_all_progress_per_node(dm, ctx):
    """ProgressFn (msa_merge.cpp:121-129): one call per node, done = 1..N,
    total = N, leaves first; a throwing callback surfaces after the call."""
    import random
    rng = random.Random(5)
    seqs = list(dict.fromkeys("".join(rng.choice("ACGT") for _ in range(rng.randint(20, 60))) for _ in range(80)))
    ss = dm.SeqSet(seqs, ctx)
    nodes, order = dm.build_tree(ss, seed=3)
    seen = []
    m = dm.align_all(ss, nodes, order, dm.ScoringScheme.nucleotide(), progress=lambda d, t: seen.append((d, t)))
    assert [d for d, _ in seen] == list(range(1, len(nodes) + 1))
    assert {t for _, t in seen} == {len(nodes)}
    assert len(m.rows) == len(seqs)

    def boom(d, t):
        raise KeyError("stop")
    import pytest as _pt
    with _pt.raises(KeyError):
        dm.align_all(ss, nodes, order, dm.ScoringScheme.nucleotide(), progress=boom)
