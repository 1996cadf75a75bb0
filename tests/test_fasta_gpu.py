"""FASTA in / out around the aligner.

run_align / write_fasta outputs are compared byte for byte with the compiled
reference's divmsa::run_align / write_fasta, error messages verbatim
(seq_io.cpp:44-225, pipeline.cpp:160-187; pins from test_seq_io.cpp)."""
import random

import pytest

pytestmark = pytest.mark.gpu


def rand_str(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


def write(path, text):
    with open(path, "w", newline="") as f:
        f.write(text)
    return str(path)


def family_fasta(rng, n, base_len, alphabet="ACGT", dup_every=0, lower=False, crlf=False, wrap=60):
    base = rand_str(rng, base_len, alphabet)
    recs, seen = [], []
    for i in range(n):
        if dup_every and i % dup_every == dup_every - 1 and seen:
            s = rng.choice(seen)
        else:
            s = list(base)
            for _ in range(rng.randint(0, max(1, base_len // 10))):
                p = rng.randrange(len(s))
                if rng.random() < 0.6:
                    s[p] = rng.choice(alphabet)
                elif len(s) > 5 and rng.random() < 0.5:
                    del s[p]
                else:
                    s.insert(p, rng.choice(alphabet))
            s = "".join(s)
            seen.append(s)
        desc = "" if i % 3 else f"desc {i} \tx"
        body = s.lower() if lower and i % 2 else s
        lines = [body[k:k + wrap] for k in range(0, len(body), wrap)] or [""]
        nl = "\r\n" if crlf else "\n"
        recs.append(f">r{i}{' ' + desc if desc else ''}{nl}" + nl.join(lines) + nl + ("" if i % 4 else nl))
    return "".join(recs)


def both(dm, ctx, ref, tmp_path, text, **kw):
    src = write(tmp_path / "in.fa", text)
    dm.run_align(src, tmp_path / "gpu.fa", ctx=ctx, **kw)
    rkw = dict(kw)
    if "gap_mode" in rkw:
        rkw["flat"] = rkw.pop("gap_mode") == "flat"
    ref.run_align(src, str(tmp_path / "ref.fa"), **rkw)
    return open(tmp_path / "gpu.fa", "rb").read(), open(tmp_path / "ref.fa", "rb").read()


@pytest.mark.parametrize("order", ["tree", "input"])
@pytest.mark.parametrize("seed", [3, 4])
def test_run_align_matches_reference(dm, ctx, ref, tmp_path, order, seed):
    rng = random.Random(seed)
    text = family_fasta(rng, rng.randint(20, 70), rng.randint(40, 400), dup_every=5, lower=True, crlf=seed == 4)
    g, r = both(dm, ctx, ref, tmp_path, text, order=order, seed=seed)
    assert g == r
    assert not (tmp_path / "gpu.fa.partial").exists()


def test_run_align_protein_and_alphabets(dm, ctx, ref, tmp_path):
    rng = random.Random(21)
    text = family_fasta(rng, 30, 150, alphabet="ARNDCQEGHILKMFPSTWYV", dup_every=7)
    for alphabet in ("auto", "aa"):
        g, r = both(dm, ctx, ref, tmp_path, text, alphabet=alphabet)
        assert g == r
    g, r = both(dm, ctx, ref, tmp_path, family_fasta(rng, 12, 90), alphabet="nt", gap_mode="flat")
    assert g == r
    g, r = both(dm, ctx, ref, tmp_path, family_fasta(rng, 12, 90), gap_open=-3, gap_extend=-2)
    assert g == r


def test_run_align_cfg0(dm, ctx, ref, tmp_path):
    """cfg0 (1,000 records of ~300 nt, 80+ columns wrapped) end to end."""
    data, offs = dm.synth(0, 1.0)
    seqs = dm.split(data, offs)
    text = "".join(f">s{i} cfg0\n{s.decode()}\n" for i, s in enumerate(seqs))
    g, r = both(dm, ctx, ref, tmp_path, text)
    assert g == r and len(g) > 300000


@pytest.mark.parametrize("text,alphabet", [
    ("", "auto"),
    ("\n\n", "auto"),
    ("ACGT\n>a\nACGT\n", "auto"),
    (">\nACGT\n", "auto"),
    ("> a\nACGT\n", "auto"),
    (">a\n>b\nACGT\n", "auto"),
    (">a\nACGT\n>b\n", "auto"),
    (">a\nAC-GT\n", "auto"),
    (">a\nACGQ\n", "nt"),
    (">a\nACGT\n>b\nACJT\n", "aa"),
    (">a\nACGT\n>b\nAC*T\n", "auto"),
])
def test_parse_errors_match_reference(dm, ctx, ref, tmp_path, text, alphabet):
    """Same outcome as the reference: the same exception and message, or (when
    the reference accepts the input) the same output bytes."""
    src = write(tmp_path / "bad.fa", text)
    try:
        ref.run_align(src, str(tmp_path / "r.fa"), alphabet=alphabet)
    except (RuntimeError, ValueError) as want:
        with pytest.raises(type(want)) as got:
            dm.run_align(src, tmp_path / "g.fa", alphabet=alphabet, ctx=ctx)
        assert str(got.value) == str(want)
        assert not (tmp_path / "g.fa").exists() and not (tmp_path / "g.fa.partial").exists()
        return
    dm.run_align(src, tmp_path / "g.fa", alphabet=alphabet, ctx=ctx)
    assert open(tmp_path / "g.fa", "rb").read() == open(tmp_path / "r.fa", "rb").read()


def test_missing_input(dm, ctx, tmp_path):
    with pytest.raises(RuntimeError, match="cannot open .* for reading"):
        dm.run_align(tmp_path / "nope.fa", tmp_path / "o.fa", ctx=ctx)


def test_write_fasta_matches_reference(dm, ctx, ref, tmp_path):
    rng = random.Random(5)
    recs = [("id%d" % i, "" if i % 2 else "some description", rand_str(rng, n, "ACGT-"))
            for i, n in enumerate([0, 1, 79, 80, 81, 159, 160, 161, 1000, 2620])]
    dm.write_fasta(recs, tmp_path / "g.fa", ctx=ctx)
    ref.write_fasta(recs, str(tmp_path / "r.fa"))
    assert open(tmp_path / "g.fa", "rb").read() == open(tmp_path / "r.fa", "rb").read()


def test_parse_fasta_round_trip(dm, tmp_path):
    src = write(tmp_path / "p.fa", ">x  two  words \r\nac gt\n\nAC\n>y\nA-C\n")
    assert dm.parse_fasta(src, allow_gaps=True) == [("x", "two  words ", "ACGTAC"), ("y", "", "A-C")]
    with pytest.raises(RuntimeError, match="gap symbol"):
        dm.parse_fasta(src)


def test_run_align_dumps_match_reference(dm, ctx, ref, tmp_path):
    """RunConfig dump_tree_path / dump_dedup_path: the tree NDJSON
    (cluster_tree.cpp:253-280, nlohmann key order and escaping) and the
    duplicates TSV (seq_io.cpp:227-249) byte-identical to the reference."""
    rng = random.Random(8)
    text = family_fasta(rng, 60, 120, dup_every=4)
    text += '>we"ird\\id\tx\nACGTACGTAAC\n>ctl\x01id\nACGTTCGTAAC\n'
    src = write(tmp_path / "in.fa", text)
    dm.run_align(src, tmp_path / "g.fa", dump_tree=tmp_path / "g.tree", dump_dedup=tmp_path / "g.tsv", ctx=ctx)
    ref.run_align(src, str(tmp_path / "r.fa"), dump_tree=str(tmp_path / "r.tree"), dump_dedup=str(tmp_path / "r.tsv"))
    for ext in ("fa", "tree", "tsv"):
        assert open(tmp_path / f"g.{ext}", "rb").read() == open(tmp_path / f"r.{ext}", "rb").read(), ext
    assert open(tmp_path / "g.tsv").read().count("\n") > 5


def test_dump_tree_api(dm, ctx, tmp_path):
    import json
    seqs = ["ACGTACGT", "ACGTTCGT", "TTTTACGA", "ACGAACGT", "GGGTACGT"]
    nodes, order = dm.build_tree(dm.SeqSet(seqs, ctx))
    dm.dump_tree(nodes, [f"s{i}" for i in range(len(seqs))], tmp_path / "t.ndjson")
    lines = [json.loads(x) for x in open(tmp_path / "t.ndjson")]
    assert len(lines) == 2 * len(seqs) - 1
    assert lines[0]["parent"] is None and lines[0]["cardinality"] == len(seqs) and lines[0]["node"] == 0
    assert list(lines[0]) == ["cardinality", "center", "depth", "node", "parent", "radius"]
