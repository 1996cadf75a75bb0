"""The sharded (multi-GPU) code path, exercised on one GPU with a simulated
world: every distance batch and every merge level is split into w
contiguous ranges computed in turn and exchanged through the same
gather/scatter and zeroed-buffer reductions NCCL performs across ranks.
Results must be identical to the unsharded run and to the reference."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def unique(seqs):
    return list(dict.fromkeys(seqs))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_tree_and_msa_identical(dm, ctx, world):
    from paper_2601_15458_b200.dist import simulate_world
    data, offs = dm.synth(0, scale=0.4)
    seqs = unique(s.decode() for s in dm.split(data, offs))
    sc = dm.ScoringScheme.nucleotide()
    base = dm.msa(dm.SeqSet(seqs, ctx), sc, seed=42)
    c2 = dm.Context(0)
    simulate_world(c2, world)
    got = dm.msa(dm.SeqSet(seqs, c2), sc, seed=42)
    assert np.array_equal(got.nodes, base.nodes) and np.array_equal(got.order, base.order)
    assert got.width == base.width and got.rows == base.rows


def test_sharded_matches_reference_large_nodes(dm, ref):
    """Sampled medians (|C| > 100) and sweeps across shards vs the reference."""
    from paper_2601_15458_b200.dist import simulate_world
    rng = random.Random(8)
    anc = "".join(rng.choice("ACGT") for _ in range(200))
    seqs = []
    for _ in range(700):
        s = list(anc)
        for _ in range(20):
            s[rng.randrange(len(s))] = rng.choice("ACGT")
        seqs.append("".join(s))
    seqs = unique(seqs)
    c2 = dm.Context(0)
    simulate_world(c2, 4)
    m = dm.msa(dm.SeqSet(seqs, c2), dm.ScoringScheme.nucleotide(), seed=42)
    r = ref.msa(seqs, seed=42)
    assert np.array_equal(m.nodes, r["nodes"]) and np.array_equal(m.order, r["order"])
    assert m.rows == r["rows"]


def test_attach_single_rank(dm):
    from paper_2601_15458_b200.dist import attach, nccl_unique_id
    c = dm.Context(0)
    attach(c, 0, 1, nccl_unique_id())  # world 1: no communicator, plain path
    assert dm.levenshtein("KITTEN", "SITTING", c) == 3


@pytest.mark.parametrize("world", [2, 8])
def test_run_align_gpu_count_independent(dm, ctx, tmp_path, world):
    """test_pipeline.cpp:236-255 (byte-identical FASTA at 1/2/8 threads),
    here across simulated GPU counts, with duplicates and tree order."""
    from paper_2601_15458_b200.dist import simulate_world
    data, offs = dm.synth(0, scale=0.3)
    seqs = [s.decode() for s in dm.split(data, offs)]
    seqs += seqs[:25]  # duplicates re-expanded on every rank
    src = tmp_path / "in.fa"
    src.write_text("".join(f">s{i}\n{s}\n" for i, s in enumerate(seqs)))
    dm.run_align(src, tmp_path / "w1.fa", dump_tree=tmp_path / "w1.tree", ctx=ctx)
    c2 = dm.Context(0)
    simulate_world(c2, world)
    dm.run_align(src, tmp_path / "wk.fa", dump_tree=tmp_path / "wk.tree", ctx=c2)
    assert (tmp_path / "w1.fa").read_bytes() == (tmp_path / "wk.fa").read_bytes()
    assert (tmp_path / "w1.tree").read_bytes() == (tmp_path / "wk.tree").read_bytes()


def test_repeat_determinism_2000(dm, ctx):
    """acceptance.cpp:361-409 (#8): 2,000 sequences aligned twice -> identical."""
    rng = random.Random(1008)
    anc = [("".join(rng.choice("ACGT") for _ in range(150))) for _ in range(10)]
    seqs = []
    for k in range(2000):
        s = list(anc[k % 10])
        for _ in range(12):
            s[rng.randrange(len(s))] = rng.choice("ACGT")
        seqs.append("".join(s))
    seqs = unique(seqs)
    a = dm.align(seqs, ctx=ctx)
    b = dm.align(seqs, ctx=ctx)
    assert a == b
