"""The reference's own C++ code on the GPU drop-in.

tests/cpp/Makefile (run by build() where /root/reference exists) compiles
the reference's unmodified sources -- its unit tests (tests/test_*.cpp), its
acceptance suite (tests/acceptance.cpp) and its file pipeline (pipeline.cpp,
seq_io.cpp, alphabet.cpp, parallel.cpp) -- against include/dropin/divmsa/
(distance.hpp, pairwise.hpp, cluster_tree.hpp, msa_merge.hpp, metrics.hpp
replaced; the reference's distance.cpp, pairwise.cpp, cluster_tree.cpp,
msa_merge.cpp and metrics.cpp are not compiled) and links libdmb200.so. The
binaries travel to the GPU box; here they run there."""
import os
import random
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def _bin(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.fail(f"{p} missing: run __graft_entry__.build() where /root/reference exists")
    return p


@pytest.mark.parametrize("name", ["divmsa_tests_b200", "divmsa_acceptance_b200", "run_align_b200", "test_shim"])
def test_dropin_binaries_call_the_library(name):
    """CPU check: every binary takes the hot path from libdmb200 (undefined
    dm_* symbols resolved by the .so), and none carries the reference's
    replaced implementations."""
    p = _bin(name)
    ldd = subprocess.run(["ldd", p], capture_output=True, text=True).stdout
    assert "libdmb200.so" in ldd
    und = subprocess.run(["nm", "-D", "--undefined-only", p], capture_output=True, text=True).stdout
    nm = subprocess.run(["nm", "-C", p], capture_output=True, text=True).stdout
    assert "dm_ctx_create" in und
    if name != "test_shim":
        assert "dm_build_tree" in und and "dm_align_all_progress" in und
    if name in ("divmsa_tests_b200", "divmsa_acceptance_b200"):
        assert "dm_nw_align" in und and "dm_levenshtein" in und
    # the reference's replaced translation units are absent: no BLOSUM62
    # table of pairwise.cpp, no out-of-line ClusterTree::leaf_count of
    # cluster_tree.cpp (the drop-in's is inline)
    assert "kBlosum62" not in nm
    assert " T divmsa::ClusterTree::leaf_count() const" not in nm


@pytest.mark.gpu
def test_reference_unit_tests_on_gpu_dropin():
    """All 71 of the reference's doctest cases (test_distance, test_seq_io,
    test_pairwise, test_cluster_tree, test_msa_merge, test_metrics,
    test_pipeline) pass on the GPU drop-in."""
    out = subprocess.run([_bin("divmsa_tests_b200")], capture_output=True, text=True, timeout=1200)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-6000:] + out.stderr[-2000:]
    assert "[FAIL]" not in out.stdout
    assert out.stdout.count("[PASS]") >= 71


@pytest.mark.gpu
def test_reference_acceptance_suite_on_gpu_dropin(tmp_path):
    env = dict(os.environ, TMPDIR=str(tmp_path))
    out = subprocess.run([_bin("divmsa_acceptance_b200")], capture_output=True, text=True, timeout=1500, env=env)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all acceptance checks passed" in out.stdout


@pytest.mark.gpu
def test_cpp_shim_pins():
    out = subprocess.run([_bin("test_shim")], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


def _family_fasta(rng, n, base_len, alphabet, dup_every):
    base = "".join(rng.choice(alphabet) for _ in range(base_len))
    recs, seen = [], []
    for i in range(n):
        if dup_every and i % dup_every == dup_every - 1 and seen:
            s = rng.choice(seen)
        else:
            s = list(base)
            for _ in range(rng.randint(1, max(2, base_len // 8))):
                p = rng.randrange(len(s))
                if rng.random() < 0.6:
                    s[p] = rng.choice(alphabet)
                elif len(s) > 5 and rng.random() < 0.5:
                    del s[p]
                else:
                    s.insert(p, rng.choice(alphabet))
            s = "".join(s)
            seen.append(s)
        desc = "" if i % 3 else f"desc {i}"
        body = "\n".join(s[k:k + 70] for k in range(0, len(s), 70))
        recs.append(f">r{i}{' ' + desc if desc else ''}\n{body}\n")
    return "".join(recs)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,order", [("nt", "tree"), ("aa", "input"), ("nt", "input")])
def test_reference_run_align_on_dropin_matches_reference(tmp_path, ref, kind, order):
    """The reference's run_align compiled against the drop-in writes the same
    bytes (aligned FASTA, tree NDJSON, dedup TSV) as the reference itself."""
    rng = random.Random(hash((kind, order)) & 0xffff)
    alphabet = "ACGT" if kind == "nt" else "ARNDCQEGHILKMFPSTWYV"
    src = tmp_path / "in.fa"
    src.write_text(_family_fasta(rng, 300, 220, alphabet, dup_every=7))
    out = tmp_path / "b200.fa"
    r = subprocess.run([_bin("run_align_b200"), str(src), str(out), "--order", order, "--dump-tree",
                        str(tmp_path / "b200.tree"), "--dump-dedup", str(tmp_path / "b200.tsv")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    ref.run_align(str(src), str(tmp_path / "ref.fa"), order=order,
                  dump_tree=str(tmp_path / "ref.tree"), dump_dedup=str(tmp_path / "ref.tsv"))
    for ext in ("fa", "tree", "tsv"):
        assert (tmp_path / f"b200.{ext}").read_bytes() == (tmp_path / f"ref.{ext}").read_bytes(), ext
