"""CPU: the C ABI library loads, exports every symbol include/dm_b200.h
declares, and its host-only entry points behave (no GPU compute here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(dm):
    from paper_2601_15458_b200._lib import LIB_PATH, SIGNATURES
    L = C.CDLL(LIB_PATH)
    decl = declared_symbols()
    assert len(decl) >= 40
    missing = [s for s in decl if not hasattr(L, s)]
    assert not missing, missing
    unbound = [s for s in decl if s not in SIGNATURES]
    assert not unbound, unbound


def test_library_is_sm100a(dm):
    import subprocess
    from paper_2601_15458_b200._lib import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly(dm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(dm.DmError):
        dm.Context(0)


def test_scheme_tables_host_side(dm, orc):
    s = dm.ScoringScheme.nucleotide()
    assert np.array_equal(s.table, orc.table("nt"))
    assert s.open_surcharge() == -10
    p = dm.ScoringScheme.protein(-11, -2, "flat")
    assert np.array_equal(p.table, orc.table("aa", -2)) and p.open_surcharge() == 0
    with pytest.raises(ValueError, match="not symmetric"):
        dm.ScoringScheme.custom("AC", [1, -1, -2, 1], -5, -1)
    with pytest.raises(ValueError):
        dm.ScoringScheme.custom("AC", [1, -1, -1, 1], -1, -5)


def test_scheme_tables_match_reference(dm, ref):
    for kind, ctor in (("nt", dm.ScoringScheme.nucleotide), ("aa", dm.ScoringScheme.protein)):
        t, osur = ref.scheme_table(kind, -7, -3, False)
        s = ctor(-7, -3)
        assert np.array_equal(s.table, t) and s.open_surcharge() == osur


def test_synth_shapes_and_determinism(dm):
    d0, o0 = dm.synth(0, scale=0.2)
    d1, o1 = dm.synth(0, scale=0.2)
    assert d0 == d1 and np.array_equal(o0, o1)
    assert len(o0) - 1 == 200
    lens = np.diff(o0)
    assert 200 < lens.mean() < 400
    assert set(d0) <= set(b"ACGT")
    d, o = dm.synth(3, scale=0.01)
    assert set(d) <= set(b"ARNDCQEGHILKMFPSTWYV")
    d, o = dm.synth(1, scale=0.0005)
    lens = np.diff(o)
    assert len(lens) == 1000 and lens[0::2].min() >= 500 and lens[0::2].max() <= 1500


def _np_pack(b):
    codes = np.frombuffer(b, dtype=np.uint8)
    k = ((codes >> 1) ^ (codes >> 2)) & 3
    k = np.concatenate([k, np.zeros((-len(k)) % 4, dtype=np.uint8)]).reshape(-1, 4)
    return (k[:, 0] | (k[:, 1] << 2) | (k[:, 2] << 4) | (k[:, 3] << 6)).astype(np.uint8).tobytes()


def test_pack_nt_host(dm):
    """The streamed path's 2-bit packer (host only): codes A0 C1 G2 T3, any
    other byte rejected wherever it sits (SIMD body, 128-residue groups,
    scalar tail, across the 1 Mi-residue task boundary)."""
    from paper_2601_15458_b200._lib import lib
    rng = np.random.default_rng(4)
    for n in (0, 1, 3, 4, 5, 127, 128, 129, 1000, (1 << 20) - 1, (1 << 20) + 77, 3 * (1 << 20) + 5):
        src = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, n)].tobytes()
        dst = (C.c_uint8 * max(1, (n + 3) // 4))()
        assert lib().dm_pack_nt(src, n, dst) == 0
        assert bytes(dst)[:(n + 3) // 4] == _np_pack(src), n
        for pos in {0, n // 2, n - 1} if n else ():
            for badc in (b"N", b"a", b"-", b"\x00", b"\xc1", b"E"):
                bad = src[:pos] + badc + src[pos + 1:]
                assert lib().dm_pack_nt(bad, n, dst) != 0, (n, pos, badc)


def test_pack_nt_seqs_layout(dm):
    """Per-sequence 2-bit layout of the streamed upload (= the device code
    buffer of a <= 4-symbol set): 32 bytes per started 128-residue block,
    residue j at bits 2(j%16) of 32-bit word j/16, zero padding."""
    for lens in ([0, 1, 15, 16, 17, 31, 32, 127, 128, 129, 255, 256, 1000, 3]
                 + list(np.random.default_rng(7).integers(0, 3000, 9000)),
                 list(np.random.default_rng(8).integers(0, 40, 20000)) + [5, 0, 2]):
        _check_pack_seqs(lens)


def _check_pack_seqs(lens):
    from paper_2601_15458_b200._lib import lib
    rng = np.random.default_rng(len(lens))
    seqs = [np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, L)].tobytes() for L in lens]
    data = b"".join(seqs)
    offs = np.zeros(len(seqs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum(lens)
    want = []
    for s_ in seqs:
        words = 8 * ((len(s_) + 127) // 128)
        k = ((np.frombuffer(s_, dtype=np.uint8) >> 1) ^ (np.frombuffer(s_, dtype=np.uint8) >> 2)) & 3
        k = np.concatenate([k, np.zeros(16 * words - len(k), dtype=np.uint8)]).astype(np.uint32).reshape(words, 16)
        want.append((k << (2 * np.arange(16, dtype=np.uint32))).sum(axis=1).astype("<u4").tobytes())
    want = b"".join(want)
    raw = np.zeros(len(data) // 4 + 32 * len(seqs) + 128, dtype=np.uint8)
    dst = raw[(-raw.ctypes.data) % 32:]  # 32-byte aligned view
    nb = C.c_uint64()
    u64p = C.POINTER(C.c_uint64)
    assert lib().dm_pack_nt_seqs(data, offs.ctypes.data_as(u64p), len(seqs), dst.ctypes.data, C.byref(nb)) == 0
    assert nb.value == len(want) and dst[:nb.value].tobytes() == want
    for pos in (len(data) - 1, len(data) // 2, 0):  # buffer end (tail through the buffer), middle, start
        bad = bytearray(data)
        bad[pos] = ord("N")
        assert lib().dm_pack_nt_seqs(bytes(bad), offs.ctypes.data_as(u64p), len(seqs), dst.ctypes.data,
                                     C.byref(nb)) != 0
    assert lib().dm_pack_nt_seqs(data, offs.ctypes.data_as(u64p), len(seqs), dst[1:].ctypes.data, C.byref(nb)) != 0


def test_oracle_synth_is_the_product_generator():
    """bench.py --impl reference takes its inputs from oracle/_build/libsynth.so
    (so it never loads libdmb200.so); they must be the product's dm.synth inputs."""
    import numpy as np

    import oracle
    import paper_2601_15458_b200 as dm
    for cfg, scale in ((0, 1.0), (1, 0.001), (3, 0.01), (4, 0.01)):
        a, b = oracle.synth(cfg, scale), dm.synth(cfg, scale)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
