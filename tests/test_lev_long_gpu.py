"""Patterns longer than one warp's rows: the multi-pass distance path.

The reference's two-row DP (/root/reference/proj/src/distance.cpp:30-47) has
no length limit. One warp holds 32 lanes x WMax words = 24,576 rows (<= 4
symbols), 10,240 (<= 32 symbols) or 6,144 (byte alphabets); longer patterns
run in passes of that many rows, the horizontal delta of every text column
carried between passes in global memory (lev.cu, LONG kernels). Every case
here is compared with the compiled reference (oracle/_ref)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DNA = "ACGT"
AA = "ARNDCQEGHILKMFPSTWYV"
BYTES = "".join(chr(c) for c in range(33, 127))  # 94 symbols -> 8 bit-planes


def mutate(rng, a, alphabet, rate, target_len):
    b = list(a)
    for _ in range(int(len(b) * rate)):
        k = rng.random()
        pos = rng.randrange(max(1, len(b)))
        if k < 0.6 and b:
            b[pos] = rng.choice(alphabet)
        elif k < 0.8 and b:
            del b[pos]
        else:
            b.insert(pos, rng.choice(alphabet))
    while len(b) < target_len:
        b.append(rng.choice(alphabet))
    return "".join(b[:target_len])


def pairs_for(rng, alphabet, lengths, rate=0.05):
    seqs, ia, ib = [], [], []
    for la, lb in lengths:
        a = "".join(rng.choice(alphabet) for _ in range(la))
        b = mutate(rng, a, alphabet, rate, lb) if rate else "".join(rng.choice(alphabet) for _ in range(lb))
        ia.append(len(seqs)); seqs.append(a)
        ib.append(len(seqs)); seqs.append(b)
    return seqs, ia, ib


CASES = {
    # (alphabet, [(len a, len b), ...]); one warp's rows: 24,576 / 10,240 / 6,144
    "dna": (DNA, [(24576, 24600), (24577, 24577), (24577, 30000), (49152, 49152), (49153, 49300), (60000, 59000),
                  (30000, 24577), (900, 1200), (5000, 4800)]),
    "protein": (AA, [(10240, 10240), (10241, 10300), (20481, 20481), (35000, 34000), (300, 400), (2000, 2100)]),
    "bytes": (BYTES, [(6144, 6144), (6145, 6200), (12289, 12289), (13000, 12500), (100, 90)]),
}


@pytest.mark.parametrize("kind", sorted(CASES))
@pytest.mark.parametrize("related", [True, False])
def test_long_pairs_vs_reference(dm, ctx, ref, kind, related):
    alphabet, lengths = CASES[kind]
    rng = random.Random(hash((kind, related)) & 0xffff)
    seqs, ia, ib = pairs_for(rng, alphabet, lengths, rate=0.05 if related else 0.0)
    ss = dm.SeqSet(seqs, ctx)
    want = ref.lev_pairs(seqs, ia, ib)
    got, st = dm.lev_pairs(ss, ia, ib, stats=True)
    assert np.array_equal(got, want), [(len(seqs[a]), len(seqs[b]), int(g), int(w))
                                       for a, b, g, w in zip(ia, ib, got, want) if g != w]
    # both orientations (the planner makes the shorter string the pattern)
    assert np.array_equal(dm.lev_pairs(ss, ib, ia), want)
    assert st["cells"] == sum(len(seqs[a]) * len(seqs[b]) for a, b in zip(ia, ib))


def test_long_single_pair_api(dm, ctx, ref):
    rng = random.Random(77)
    a = "".join(rng.choice(DNA) for _ in range(40000))
    b = mutate(rng, a, DNA, 0.03, 39000)
    assert dm.levenshtein(a, b, ctx) == ref.levenshtein(a, b)
    assert dm.levenshtein(a, "", ctx) == 40000
    assert dm.levenshtein(a, a, ctx) == 0


def test_long_many_jobs_mixed_passes(dm, ctx, ref):
    """Many long jobs of different pass counts in one launch series, among short ones."""
    rng = random.Random(11)
    lengths = [(rng.randint(24000, 52000), 0) for _ in range(24)] + [(rng.randint(50, 3000), 0) for _ in range(200)]
    lengths = [(la, max(1, la + rng.randint(-500, 500))) for la, _ in lengths]
    seqs, ia, ib = pairs_for(rng, DNA, lengths, rate=0.08)
    ss = dm.SeqSet(seqs, ctx)
    assert np.array_equal(dm.lev_pairs(ss, ia, ib), ref.lev_pairs(seqs, ia, ib))


def test_long_one_to_many_and_packed(dm, ctx, ref):
    rng = random.Random(21)
    root = "".join(rng.choice(DNA) for _ in range(26000))
    seqs = [root] + [mutate(rng, root, DNA, 0.02 * (k + 1), 26000 + 37 * k) for k in range(6)]
    seqs += ["".join(rng.choice(DNA) for _ in range(rng.randint(100, 900))) for _ in range(5)]
    ss = dm.SeqSet(seqs, ctx)
    members = np.arange(len(seqs))
    want = ref.lev_pairs(seqs, np.zeros(len(seqs), dtype=np.uint32), members)
    assert np.array_equal(dm.lev_one_to_many(ss, 0, members), want)
    # host-buffer streamed path: pairs (2i, 2i+1) of one packed buffer
    flat = []
    for k in range(1, len(seqs)):
        flat += [seqs[0], seqs[k]]
    data = "".join(flat).encode()
    offs = np.concatenate([[0], np.cumsum([len(x) for x in flat])]).astype(np.uint64)
    assert np.array_equal(dm.lev_pairs_packed(data, offs, ctx), want[1:])


def test_long_guide_tree_vs_reference(dm, ctx, ref):
    """build_tree over sequences longer than one warp's rows (viral-genome sized)."""
    rng = random.Random(31)
    root = "".join(rng.choice(DNA) for _ in range(25500))
    seqs = []
    for k in range(9):
        s = mutate(rng, root, DNA, 0.01 + 0.01 * (k % 4), 25000 + rng.randint(0, 1500))
        seqs.append(s)
    seqs = list(dict.fromkeys(seqs))
    ss = dm.SeqSet(seqs, ctx)
    nodes, order = dm.build_tree(ss, seed=7)
    rnodes, rorder = ref.build_tree(seqs, seed=7)
    assert np.array_equal(nodes, rnodes)
    assert np.array_equal(order, rorder)
