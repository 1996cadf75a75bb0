"""Parity of the GPU distance engine (K1) with the CPU oracle.

Pins restate /root/reference/proj/tests/test_distance.cpp:11-28 and
acceptance.cpp:163-189; random sweeps compare every distance bit-exactly with
the C restatement and the compiled reference."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand_str(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


@pytest.mark.parametrize("a,b,d", [
    ("KITTEN", "SITTING", 3), ("", "", 0), ("A", "", 1), ("", "ACGT", 4), ("ACGT", "ACGT", 0),
    ("A", "C", 1), ("AC", "CA", 2),
    # trims must never change the value (test_distance.cpp:21-28)
    ("ABCXDEF", "ABCYDEF", 1), ("AAAA", "AAA", 1), ("XXXABC", "ABC", 3), ("ABC", "ABCXXX", 3),
    ("AAAA", "AAAA", 0),
])
def test_known_pairs(dm, ctx, a, b, d):
    assert dm.levenshtein(a, b, ctx) == d


def test_recursive_definition_small(dm, ctx, orc):
    # test_distance.cpp:30-42 / acceptance #3: short random pairs, both orders
    rng = random.Random(1003)
    seqs, ia, ib = [], [], []
    for _ in range(500):
        a, b = rand_str(rng, rng.randrange(13)), rand_str(rng, rng.randrange(13))
        ia.append(len(seqs)); seqs.append(a)
        ib.append(len(seqs)); seqs.append(b)
    ss = dm.SeqSet(seqs, ctx)
    fwd = dm.lev_pairs(ss, ia, ib)
    rev = dm.lev_pairs(ss, ib, ia)
    want = [orc.levenshtein(seqs[x], seqs[y]) for x, y in zip(ia, ib)]
    assert list(fwd) == want
    assert list(rev) == want


@pytest.mark.parametrize("alphabet", ["ACGT", "ACGTURYSWKMBDHVN", "ARNDCQEGHILKMFPSTWYV",
                                      "".join(chr(c) for c in range(33, 127))])
def test_block_boundaries(dm, ctx, orc, alphabet):
    """Lengths straddling 32/64/128/.../4096 rows exercise every (G, R) bucket."""
    rng = random.Random(len(alphabet))
    edges = [1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129, 191, 192, 255, 256, 257, 511, 512, 513,
             700, 1023, 1024, 1025, 1500, 2047, 2048, 2049, 3000, 4095, 4096, 4097]
    seqs, ia, ib = [], [], []
    for la in edges:
        for _ in range(3):
            lb = max(0, la + rng.randint(-40, 40))
            a = rand_str(rng, la, alphabet)
            # related pair: mutate a
            b = list(a[:lb]) + [rng.choice(alphabet) for _ in range(max(0, lb - la))]
            for k in range(max(1, lb // 20)):
                if b:
                    b[rng.randrange(len(b))] = rng.choice(alphabet)
            ia.append(len(seqs)); seqs.append(a)
            ib.append(len(seqs)); seqs.append("".join(b))
    ss = dm.SeqSet(seqs, ctx)
    got = dm.lev_pairs(ss, ia, ib)
    want = [orc.levenshtein(seqs[x], seqs[y]) for x, y in zip(ia, ib)]
    assert list(got) == want


def test_unrelated_long(dm, ctx, ref):
    rng = random.Random(5)
    seqs = [rand_str(rng, rng.randint(1, 2600)) for _ in range(120)]
    ia = list(range(0, 120, 2))
    ib = list(range(1, 120, 2))
    ss = dm.SeqSet(seqs, ctx)
    assert np.array_equal(dm.lev_pairs(ss, ia, ib), ref.lev_pairs(seqs, ia, ib))


def test_cfg1_sample_vs_reference(dm, ctx, ref):
    """cfg1-shaped pairs (L in [500,1500], 5% sub + 1% indel) vs the compiled reference."""
    data, offs = dm.synth(1, scale=0.003)  # 3000 pairs
    seqs = dm.split(data, offs)
    ss = dm.SeqSet(data=data, offsets=offs, ctx=ctx)
    n = len(seqs) // 2
    ia = np.arange(n) * 2
    ib = ia + 1
    got, st = dm.lev_pairs(ss, ia, ib, stats=True)
    want = ref.lev_pairs(seqs, ia, ib)
    assert np.array_equal(got, want)
    assert st["cells"] == sum(len(seqs[a]) * len(seqs[b]) for a, b in zip(ia, ib))


def test_one_to_many(dm, ctx, ref):
    data, offs = dm.synth(0, scale=0.3)
    seqs = dm.split(data, offs)
    ss = dm.SeqSet(data=data, offsets=offs, ctx=ctx)
    members = np.arange(len(seqs))
    got = dm.lev_one_to_many(ss, 7, members)
    want = ref.lev_pairs(seqs, np.full(len(seqs), 7), members)
    assert np.array_equal(got, want)
    assert got[7] == 0


def test_batch_sizes_and_grouping(dm, ctx, orc):
    """Tiny batches use wide groups (G up to 32); results must not depend on it."""
    rng = random.Random(9)
    seqs = [rand_str(rng, rng.randint(900, 1700)) for _ in range(6)]
    ss = dm.SeqSet(seqs, ctx)
    want = {(x, y): orc.levenshtein(seqs[x], seqs[y]) for x in range(6) for y in range(6)}
    for k in (1, 2, 5, 36):
        pairs = list(want)[:k]
        got = dm.lev_pairs(ss, [p[0] for p in pairs], [p[1] for p in pairs])
        assert list(got) == [want[p] for p in pairs]


def _cfg1_golden():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "lev_cfg1.json")) as f:
        return json.load(f)


def _sha(d):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(d, dtype="<u4").tobytes()).hexdigest()


def _first_bad_block(d, g):
    import hashlib
    blk = g["block"]
    for k, h in enumerate(g["block_sha256"]):
        if hashlib.sha256(np.ascontiguousarray(d[k * blk:(k + 1) * blk], dtype="<u4").tobytes()).hexdigest() != h:
            return k
    return None


@pytest.fixture(scope="module")
def cfg1(dm):
    data, offs = dm.synth(1, scale=1.0)
    return data, offs


def test_cfg1_full_pinned_to_reference(dm, ctx, cfg1):
    """All 10^6 cfg1 pairs == the compiled reference's levenshtein
    (distance.cpp:9-48), by SHA-256 of the uint32 vector (tests/golden/
    lev_cfg1.json, made by make_golden.py --only cfg1@1.0 from oracle/_ref),
    device-resident, in both orientations."""
    g = _cfg1_golden()
    data, offs = cfg1
    ss = dm.SeqSet(data=data, offsets=offs, ctx=ctx)
    n = (len(offs) - 1) // 2
    assert n == g["pairs"]
    ia = np.arange(n, dtype=np.uint32) * 2
    ib = ia + 1
    d = dm.lev_pairs(ss, ia, ib)
    assert d[:16].tolist() == g["first16"]
    assert _sha(d) == g["sha256"], f"first differing 65,536-pair block: {_first_bad_block(d, g)}"
    assert int(d.astype(np.uint64).sum()) == g["sum"]
    assert _sha(dm.lev_pairs(ss, ib, ia)) == g["sha256"]


@pytest.mark.parametrize("mode", ["pageable", "pinned-frac0", "pinned-frac0.3", "pinned-frac1", "nopack"])
def test_cfg1_full_streamed_pinned_to_reference(dm, ctx, cfg1, monkeypatch, mode):
    """The same 10^6 pairs from host memory through dm_lev_pairs_packed:
    pageable and pinned buffers, every speculative raw share, packing off."""
    g = _cfg1_golden()
    data, offs = cfg1
    if mode.startswith("pinned"):
        import torch
        buf = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
        monkeypatch.setenv("DM_STREAM_RAW_FRAC", mode.split("frac")[1])
    else:
        buf = data
        if mode == "nopack":
            monkeypatch.setenv("DM_STREAM_PACK", "0")
    d = dm.lev_pairs_packed(buf, offs, ctx)
    assert _sha(d) == g["sha256"], f"first differing 65,536-pair block: {_first_bad_block(d, g)}"


@pytest.mark.parametrize("alphabet", ["ACGT", "ARNDCQEGHILKMFPSTWYV", "".join(chr(c) for c in range(33, 127))])
@pytest.mark.parametrize("gpar", ["0", "1", "3"])
def test_every_bucket_forced_lanes(dm, ctx, ref, monkeypatch, alphabet, gpar):
    """Small batches normally widen groups to 32 lanes; DM_LEV_GPAR forces
    the minimum lanes per pair so every (G, W) kernel runs: patterns of
    1..48 words (W = 17..24 kernels for <= 4 symbols, 6..10 for 5 planes)."""
    monkeypatch.setenv("DM_LEV_GPAR", gpar)
    rng = random.Random(len(alphabet) * 7 + int(gpar))
    seqs, ia, ib = [], [], []
    for B in list(range(1, 25)) + list(range(33, 49)) + [64, 96, 128, 192, 256, 384, 768]:
        for delta in (-17, 0):
            la = max(1, 32 * B + delta)
            a = rand_str(rng, la, alphabet)
            b = list(a)
            for _ in range(max(1, la // 15)):
                b[rng.randrange(len(b))] = rng.choice(alphabet)
            b = "".join(b[:max(1, la - rng.randint(0, 40))]) + rand_str(rng, rng.randint(0, 40), alphabet)
            ia.append(len(seqs)); seqs.append(a)
            ib.append(len(seqs)); seqs.append(b)
    ss = dm.SeqSet(seqs, ctx)
    assert np.array_equal(dm.lev_pairs(ss, ia, ib), ref.lev_pairs(seqs, ia, ib))


def test_packed_streaming_matches(dm, ctx, orc, monkeypatch):
    """dm_lev_pairs_packed (host buffer, overlapped chunks) == resident batch."""
    monkeypatch.setenv("DM_STREAM_CHUNK_BYTES", "200000")  # force ~25 chunks
    data, offs = dm.synth(1, scale=0.004)  # 4000 pairs
    got = dm.lev_pairs_packed(data, offs, ctx)
    ss = dm.SeqSet(data=data, offsets=offs, ctx=ctx)
    n = (len(offs) - 1) // 2
    ia = np.arange(n) * 2
    assert np.array_equal(got, dm.lev_pairs(ss, ia, ia + 1))
    for i in (0, 1, n // 2, n - 1):
        assert got[i] == orc.levenshtein(data[offs[2 * i]:offs[2 * i + 1]], data[offs[2 * i + 1]:offs[2 * i + 2]])
    import torch
    pinned = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    assert np.array_equal(dm.lev_pairs_packed(pinned, offs, ctx), got)


@pytest.mark.parametrize("chunk", ["1", "3000", "50000"])
def test_packed_streaming_mixed_chunks(dm, ctx, orc, monkeypatch, chunk):
    """Chunks with different alphabets (2/5/8 bit-planes), empty sequences and
    one-pair chunks; each chunk is recoded on its own."""
    monkeypatch.setenv("DM_STREAM_CHUNK_BYTES", chunk)
    rng = random.Random(int(chunk))
    alphabets = ["ACGT", "ARNDCQEGHILKMFPSTWYV", "".join(chr(c) for c in range(33, 127))]
    seqs = []
    for k in range(300):
        alpha = alphabets[(k // 40) % 3]
        for _ in range(2):
            n = 0 if rng.random() < 0.05 else rng.randint(1, 700)
            seqs.append(rand_str(rng, n, alpha))
    data = "".join(seqs).encode()
    offs = np.zeros(len(seqs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(x) for x in seqs])
    got = dm.lev_pairs_packed(data, offs, ctx)
    want = [orc.levenshtein(seqs[2 * i], seqs[2 * i + 1]) for i in range(300)]
    assert list(got) == want
    # a second call on the same context reuses the planner slots
    assert list(dm.lev_pairs_packed(data, offs, ctx)) == want


def test_context_shared_by_threads(dm, ctx, orc):
    """The reference's functions are reentrant (called from parallel_for
    bodies); one context used by 8 host threads at once gives
    the same answers (ctypes drops the GIL, so the calls overlap in C)."""
    from concurrent.futures import ThreadPoolExecutor
    rng = random.Random(99)
    pairs = [(rand_str(rng, rng.randint(0, 300)), rand_str(rng, rng.randint(0, 300))) for _ in range(64)]
    want = [orc.levenshtein(a, b) for a, b in pairs]

    def work(k):
        a, b = pairs[k]
        d = dm.levenshtein(a, b, ctx)
        ss = dm.SeqSet([a, b, a], ctx)
        d2 = int(dm.lev_pairs(ss, [0, 1], [1, 2])[0])
        r = dm.nw_align(a + "A", b + "C", ctx=ctx)
        return d, d2, r.score

    with ThreadPoolExecutor(8) as ex:
        got = list(ex.map(work, range(len(pairs))))
    assert [g[0] for g in got] == want and [g[1] for g in got] == want
    assert all(g[2] == dm.nw_align(a + "A", b + "C", ctx=ctx).score for g, (a, b) in zip(got, pairs))


@pytest.mark.parametrize("chunk", ["100000", "5000000"])
def test_packed_upload_matches_raw_upload(dm, ctx, orc, monkeypatch, chunk):
    """2-bit upload of A/C/G/T chunks (all chunks packed, or a mix with
    speculative raw chunks) == raw upload, bit for bit; a chunk with any
    other byte (here 'N', lower case) goes up raw, or, sent speculatively,
    fails the device check and is recomputed. h2d_bytes shows which
    happened."""
    monkeypatch.setenv("DM_STREAM_CHUNK_BYTES", chunk)
    data, offs = dm.synth(1, scale=0.005)  # 5000 pairs, ~10 MB
    n = (len(offs) - 1) // 2
    monkeypatch.setenv("DM_STREAM_RAW_FRAC", "0")
    full, sf = dm.lev_pairs_packed(data, offs, ctx, stats=True)
    monkeypatch.setenv("DM_STREAM_RAW_FRAC", "0.5")
    split, sp = dm.lev_pairs_packed(data, offs, ctx, stats=True)
    monkeypatch.setenv("DM_STREAM_PACK", "0")
    raw, sr = dm.lev_pairs_packed(data, offs, ctx, stats=True)
    monkeypatch.delenv("DM_STREAM_PACK")
    monkeypatch.setenv("DM_STREAM_RAW_FRAC", "0")
    assert np.array_equal(split, raw) and np.array_equal(full, raw)
    # the host plan of packed chunks (bucket histogram, cells) == the device planner's
    assert (sf["cells"], sf["cells_executed"]) == (sr["cells"], sr["cells_executed"])
    monkeypatch.setenv("DM_STREAM_HOSTPLAN", "0")
    dev_planned, sdp = dm.lev_pairs_packed(data, offs, ctx, stats=True)
    monkeypatch.delenv("DM_STREAM_HOSTPLAN")
    assert np.array_equal(dev_planned, raw)
    assert (sdp["cells"], sdp["cells_executed"], sdp["launches"]) == (sr["cells"], sr["cells_executed"], sr["launches"])
    assert sf["launches"] < sr["launches"]  # no planner kernels on host-planned chunks
    assert sr["h2d_bytes"] >= len(data) + 8 * (len(offs) - 1)
    assert sf["h2d_bytes"] < 0.3 * len(data) + 8 * len(offs) + 64 * 1000
    assert sf["h2d_bytes"] < sp["h2d_bytes"] < sr["h2d_bytes"]
    assert sp["d2h_bytes"] == 4 * n
    # dirty bytes in the middle and near the end: those chunks go up raw
    dirty = bytearray(data)
    for p in (len(dirty) // 2, len(dirty) - 3):
        dirty[p] = ord("N")
    dirty[int(offs[10])] = ord("a")
    dirty = bytes(dirty)
    got, sd = dm.lev_pairs_packed(dirty, offs, ctx, stats=True)
    assert sf["h2d_bytes"] < sd["h2d_bytes"] < sr["h2d_bytes"] or chunk == "5000000"
    for i in list(range(0, 40)) + list(range(n // 2 - 30, n // 2 + 30)) + list(range(n - 20, n)):
        a = dirty[offs[2 * i]:offs[2 * i + 1]]
        b = dirty[offs[2 * i + 1]:offs[2 * i + 2]]
        assert got[i] == orc.levenshtein(a, b), i
    assert np.array_equal(got[np.r_[100:n // 2 - 100]], raw[100:n // 2 - 100])
    # every chunk speculative: the dirty ones fail the device check and are redone
    monkeypatch.setenv("DM_STREAM_RAW_FRAC", "1")
    spec = dm.lev_pairs_packed(dirty, offs, ctx)
    assert np.array_equal(spec, got)


@pytest.mark.parametrize("frac", ["0", "0.5", "1"])
@pytest.mark.parametrize("alphabet", ["ACGT", "GT", "ACGTN"])
@pytest.mark.parametrize("n", [1, 15, 16, 17, 63, 64, 65, 1000, 5000])
def test_packed_upload_odd_lengths(dm, ctx, orc, monkeypatch, n, alphabet, frac):
    """Chunk residue counts around the verifier's 16-byte groups, chunks
    missing some of A/C/G/T or holding an N, packed / speculative / mixed."""
    monkeypatch.setenv("DM_STREAM_CHUNK_BYTES", "1")  # one pair per chunk
    monkeypatch.setenv("DM_STREAM_RAW_FRAC", frac)
    rng = random.Random(n)
    seqs = []
    for k in range(6):
        la = max(0, n + k - 3)
        seqs += [rand_str(rng, la, alphabet), rand_str(rng, max(0, n - k), alphabet)]
    data = "".join(seqs).encode()
    offs = np.zeros(len(seqs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(x) for x in seqs])
    got = dm.lev_pairs_packed(data, offs, ctx)
    assert list(got) == [orc.levenshtein(seqs[2 * i], seqs[2 * i + 1]) for i in range(6)]


@pytest.mark.parametrize("frac", ["0", "1"])
@pytest.mark.parametrize("gpar", ["0", "2", "5"])
def test_host_planned_chunks_every_bucket(dm, ctx, ref, monkeypatch, frac, gpar):
    """Host-planned streamed chunks (patterns from 2-bit codes or from the raw
    A/C/G/T bytes at any alignment, texts likewise) over every (G, W)
    bucket: patterns of 1..48 words and up to 768 words, odd lengths, empty
    sequences; one chunk longer than one warp's rows (multi-pass) falls back
    to the device-planned path. Pinned buffer, so frac=1 sends every chunk
    raw; compared with the compiled reference."""
    import torch
    monkeypatch.setenv("DM_LEV_GPAR", gpar)
    monkeypatch.setenv("DM_STREAM_RAW_FRAC", frac)
    monkeypatch.setenv("DM_STREAM_CHUNK_BYTES", "60000")
    rng = random.Random(int(gpar) * 10 + len(frac))
    seqs = []
    words = list(range(1, 25)) + list(range(33, 49)) + [64, 96, 128, 192, 256, 384, 768]
    for B in words:
        for delta in (-17, -1, 0, 3):
            la = max(1, 32 * B + delta)
            a = rand_str(rng, la, "ACGT")
            b = list(a)
            for _ in range(max(1, la // 12)):
                b[rng.randrange(len(b))] = rng.choice("ACGT")
            b = "".join(b[:max(1, la - rng.randint(0, 50))]) + rand_str(rng, rng.randint(0, 50), "ACGT")
            seqs += [a, b] if rng.random() < 0.5 else [b, a]
    seqs += ["", "ACGT", "", ""]
    seqs += [rand_str(rng, 25000, "ACGT"), rand_str(rng, 26000, "ACGT")]  # > 24,576 rows: multi-pass
    data = "".join(seqs).encode()
    offs = np.zeros(len(seqs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(x) for x in seqs])
    pinned = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    got = dm.lev_pairs_packed(pinned, offs, ctx)
    n = len(seqs) // 2
    want = ref.lev_pairs(seqs, list(range(0, 2 * n, 2)), list(range(1, 2 * n, 2)))
    assert np.array_equal(got, want)
