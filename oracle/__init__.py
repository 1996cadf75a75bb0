"""TEST INFRASTRUCTURE ONLY — CPU checkers for the GPU hot path.

Two oracles, both CPU-only:
  * ``Restatement`` — ctypes binding of divmsa_oracle.c, a plain-C
    restatement of the reference algorithm (oracle/_build/liboracle.so);
  * ``Reference``   — ctypes binding of the UNMODIFIED reference C++ library
    compiled from /root/reference/proj/src by oracle/Makefile
    (oracle/_ref/libdivmsa_ref.so; travels to the GPU box prebuilt).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product
(paper_2601_15458_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libdivmsa_ref.so")

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_i16p = C.POINTER(C.c_int16)

NODE_FIELDS = ("begin", "end", "center", "radius", "pole_l", "pole_r", "left", "right", "parent", "depth")


def _bytes(s) -> bytes:
    return s.encode() if isinstance(s, str) else bytes(s)


def _seq_arrays(seqs: Sequence):
    bs = [_bytes(s) for s in seqs]
    arr = (C.c_char_p * len(bs))(*bs)
    lens = np.array([len(b) for b in bs], dtype=np.uint32)
    return bs, arr, lens


class OrcNode(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in NODE_FIELDS[:6]] + [(f, C.c_int32) for f in NODE_FIELDS[6:9]] + [
        ("depth", C.c_uint32)]


class Restatement:
    """Plain-C restatement (divmsa_oracle.c)."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: make -C oracle restatement")
        L = C.CDLL(path)
        L.orc_levenshtein.restype = C.c_uint32
        L.orc_levenshtein.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64]
        L.orc_combine_seed.restype = C.c_uint64
        L.orc_combine_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_hash_members.restype = C.c_uint64
        L.orc_hash_members.argtypes = [_u32p, C.c_size_t]
        L.orc_build_tree.restype = C.c_int
        L.orc_build_tree.argtypes = [C.POINTER(C.c_char_p), _u32p, C.c_size_t, C.c_uint64, C.c_size_t,
                                     C.POINTER(OrcNode), C.POINTER(C.c_size_t), _u32p]
        L.orc_geometric_median.restype = C.c_int
        L.orc_geometric_median.argtypes = [_u32p, C.c_size_t, C.POINTER(C.c_char_p), _u32p, C.c_uint64,
                                           C.c_size_t, _u32p]
        L.orc_nucleotide_table.argtypes = [C.c_int, _i16p]
        L.orc_protein_table.argtypes = [C.c_int, _i16p]
        L.orc_nw_align.restype = C.c_int
        L.orc_nw_align.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, _i16p, C.c_int, C.c_int,
                                   _i64p, C.c_char_p, C.c_char_p, C.POINTER(C.c_size_t), _u32p,
                                   C.POINTER(C.c_size_t), _u32p, C.POINTER(C.c_size_t)]
        L.orc_insert_gap_columns.restype = C.c_int
        L.orc_insert_gap_columns.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, _u32p, C.c_size_t,
                                             C.c_char_p]
        L.orc_align_all.restype = C.c_int
        L.orc_align_all.argtypes = [C.POINTER(OrcNode), C.c_size_t, _u32p, C.POINTER(C.c_char_p), _u32p,
                                    C.c_size_t, _i16p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_size_t)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_mt64_next.restype = C.c_uint64
        L.orc_mt64_next.argtypes = [C.c_void_p]
        L.orc_sample_distinct.restype = C.c_uint64
        L.orc_sample_distinct.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, _u64p]
        self.L = L

    def levenshtein(self, a, b) -> int:
        a, b = _bytes(a), _bytes(b)
        return int(self.L.orc_levenshtein(a, len(a), b, len(b)))

    def mt64(self, seed: int, count: int) -> List[int]:
        g = C.create_string_buffer(312 * 8 + 16)
        self.L.orc_mt64_seed(g, seed)
        return [int(self.L.orc_mt64_next(g)) for _ in range(count)]

    def sample_distinct(self, seed: int, n: int, k: int) -> List[int]:
        g = C.create_string_buffer(312 * 8 + 16)
        self.L.orc_mt64_seed(g, seed)
        out = np.zeros(max(min(n, k), 1), dtype=np.uint64)
        c = self.L.orc_sample_distinct(g, n, k, out.ctypes.data_as(_u64p))
        return [int(x) for x in out[:c]]

    def table(self, kind: str = "nt", gap_extend: int = -1) -> np.ndarray:
        t = np.zeros(128 * 128, dtype=np.int16)
        (self.L.orc_nucleotide_table if kind == "nt" else self.L.orc_protein_table)(gap_extend,
                                                                                       t.ctypes.data_as(_i16p))
        return t

    def nw_align(self, a, b, table: np.ndarray, open_surcharge: int, gap_extend: int):
        a, b = _bytes(a), _bytes(b)
        if not a or not b:
            raise ValueError("nw_align requires non-empty inputs")
        oa = C.create_string_buffer(len(a) + len(b) + 1)
        ob = C.create_string_buffer(len(a) + len(b) + 1)
        ga = np.zeros(len(b) + 1, dtype=np.uint32)
        gb = np.zeros(len(a) + 1, dtype=np.uint32)
        sc = C.c_int64()
        ln, na, nb = C.c_size_t(), C.c_size_t(), C.c_size_t()
        table = np.ascontiguousarray(table, dtype=np.int16)
        self.L.orc_nw_align(a, len(a), b, len(b), table.ctypes.data_as(_i16p), open_surcharge, gap_extend,
                            C.byref(sc), oa, ob, C.byref(ln), ga.ctypes.data_as(_u32p), C.byref(na),
                            gb.ctypes.data_as(_u32p), C.byref(nb))
        return dict(score=sc.value, aligned_a=oa.raw[:ln.value].decode(), aligned_b=ob.raw[:ln.value].decode(),
                    gaps_into_a=[int(x) for x in ga[:na.value]], gaps_into_b=[int(x) for x in gb[:nb.value]])

    def build_tree(self, seqs, seed: int = 42, cap: int = 100):
        bs, arr, lens = _seq_arrays(seqs)
        n = len(bs)
        nodes = (OrcNode * max(2 * n - 1, 1))()
        order = np.zeros(max(n, 1), dtype=np.uint32)
        nn = C.c_size_t()
        rc = self.L.orc_build_tree(arr, lens.ctypes.data_as(_u32p), n, seed, cap, nodes, C.byref(nn),
                                   order.ctypes.data_as(_u32p))
        if rc == 1:
            raise RuntimeError("cannot build a cluster tree from zero sequences")
        if rc == 2:
            raise RuntimeError("cluster contains identical sequences; input was not de-duplicated")
        rows = np.array([[getattr(nodes[i], f) for f in NODE_FIELDS] for i in range(nn.value)], dtype=np.int64)
        return rows, order[:n].copy()

    def geometric_median(self, seqs, members, seed: int, cap: int = 100) -> int:
        bs, arr, lens = _seq_arrays(seqs)
        m = np.ascontiguousarray(members, dtype=np.uint32)
        out = C.c_uint32()
        rc = self.L.orc_geometric_median(m.ctypes.data_as(_u32p), len(m), arr, lens.ctypes.data_as(_u32p),
                                         seed, cap, C.byref(out))
        if rc:
            raise ValueError("geometric_median of an empty member set")
        return int(out.value)

    def insert_gap_columns(self, rows: List[str], positions) -> List[str]:
        width = len(rows[0]) if rows else 0
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        out = C.create_string_buffer(len(rows) * (width + len(pos)) + 1)
        rc = self.L.orc_insert_gap_columns("".join(rows).encode(), len(rows), width, pos.ctypes.data_as(_u32p),
                                           len(pos), out)
        if rc == 1:
            raise ValueError("gap position exceeds alignment width")
        if rc == 2:
            raise ValueError("gap positions must be sorted ascending")
        w = width + len(pos)
        return [out.raw[r * w:(r + 1) * w].decode() for r in range(len(rows))]

    def align_all(self, seqs, nodes: np.ndarray, order: np.ndarray, table, open_surcharge: int,
                  gap_extend: int) -> Tuple[List[str], int]:
        bs, arr, lens = _seq_arrays(seqs)
        on = (OrcNode * len(nodes))()
        for i, row in enumerate(nodes):
            for f, v in zip(NODE_FIELDS, row):
                setattr(on[i], f, int(v))
        p = C.c_void_p()
        w = C.c_size_t()
        table = np.ascontiguousarray(table, dtype=np.int16)
        order = np.ascontiguousarray(order, dtype=np.uint32)
        self.L.orc_align_all(on, len(nodes), order.ctypes.data_as(_u32p), arr, lens.ctypes.data_as(_u32p),
                             len(bs), table.ctypes.data_as(_i16p), open_surcharge, gap_extend, C.byref(p),
                             C.byref(w))
        raw = C.string_at(p, len(bs) * w.value)
        self.L.orc_free(p)
        W = w.value
        return [raw[r * W:(r + 1) * W].decode() for r in range(len(bs))], W


class RefMetrics(C.Structure):
    """ref_metrics in oracle/ref_capi.cpp (divmsa::MetricsReport fields)."""
    _fields_ = [("width", C.c_uint64)] + [(f, C.c_double) for f in (
        "stretch", "gap_percent", "distortion", "p_min", "p_avg", "p_max")] + [(f, C.c_uint64) for f in (
            "sample_size", "pair_count", "seed", "zero_distance_pairs")] + [("time_s", C.c_double)]


class Reference:
    """The unmodified reference library (oracle/_ref/libdivmsa_ref.so)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: make -C oracle ref (needs /root/reference)")
        L = C.CDLL(path)
        P = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_levenshtein.restype = C.c_uint32
        L.ref_levenshtein.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_lev_pairs.restype = C.c_int
        L.ref_lev_pairs.argtypes = [C.POINTER(C.c_char_p), _u32p, C.c_uint64, _u32p, _u32p, C.c_uint64, C.c_int,
                                    _u32p]
        L.ref_nw_align.restype = C.c_int
        L.ref_nw_align.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.c_int, C.c_char_p,
                                   C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.POINTER(P)]
        L.ref_scheme_table.restype = C.c_int
        L.ref_scheme_table.argtypes = [C.c_int, C.c_char_p, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, _i16p,
                                       C.POINTER(C.c_int)]
        for f, r in (("score", C.c_int64), ("len", C.c_uint64), ("a", C.c_void_p), ("b", C.c_void_p),
                     ("ngaps_a", C.c_uint64), ("ngaps_b", C.c_uint64), ("gaps_a", C.c_void_p),
                     ("gaps_b", C.c_void_p)):
            fn = getattr(L, "ref_pw_" + f)
            fn.restype = r
            fn.argtypes = [P]
        L.ref_pw_free.argtypes = [P]
        L.ref_build_tree.restype = C.c_int
        L.ref_build_tree.argtypes = [C.POINTER(C.c_char_p), _u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                     _i64p, _u64p, _u32p]
        L.ref_geometric_median.restype = C.c_int
        L.ref_geometric_median.argtypes = [C.POINTER(C.c_char_p), _u32p, C.c_uint64, _u32p, C.c_uint64,
                                           C.c_uint64, C.c_uint64, C.c_int, _u32p]
        L.ref_msa.restype = C.c_int
        L.ref_msa.argtypes = [C.POINTER(C.c_char_p), _u32p, C.c_uint64, C.c_int, C.c_char_p,
                              C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.POINTER(P)]
        for f, r in (("width", C.c_uint64), ("rows", C.c_uint64), ("data", C.c_void_p), ("row_seq", C.c_void_p),
                     ("tree_s", C.c_double), ("align_s", C.c_double), ("nnodes", C.c_uint64)):
            fn = getattr(L, "ref_msa_" + f)
            fn.restype = r
            fn.argtypes = [P]
        L.ref_msa_nodes.argtypes = [P, _i64p, _u32p]
        L.ref_msa_free.argtypes = [P]
        L.ref_align.restype = C.c_int
        L.ref_align.argtypes = [C.POINTER(C.c_char_p), _u32p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_uint64, C.c_int, C.POINTER(C.c_void_p), _u64p]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_insert_gap_columns.restype = C.c_int
        L.ref_insert_gap_columns.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, _u32p, C.c_uint64, C.c_char_p]
        L.ref_evaluate.restype = C.c_int
        L.ref_evaluate.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, _u32p, C.POINTER(C.c_char_p), _u32p,
                                   C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(RefMetrics)]
        L.ref_gap_percent.restype = C.c_int
        L.ref_gap_percent.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_p_score.restype = C.c_int
        L.ref_p_score.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_hamming_aligned.restype = C.c_int
        L.ref_hamming_aligned.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, _u32p]
        L.ref_run_align.restype = C.c_int
        L.ref_run_align.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                    C.c_int, C.c_int, C.c_char_p, C.c_char_p]
        L.ref_write_fasta.restype = C.c_int
        L.ref_write_fasta.argtypes = [C.c_char_p, C.c_char_p, _u64p, C.c_char_p, _u64p, C.c_char_p, _u64p,
                                      C.c_uint64]
        L.ref_distortion_pair.restype = C.c_int
        L.ref_distortion_pair.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                          C.c_char_p, C.c_uint64, C.POINTER(C.c_double)]
        self.L = L

    def _check(self, rc):
        if rc == 0:
            return
        msg = (self.L.ref_last_error() or b"").decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def levenshtein(self, a, b) -> int:
        a, b = _bytes(a), _bytes(b)
        return int(self.L.ref_levenshtein(a, len(a), b, len(b)))

    def lev_pairs(self, seqs, ia, ib, threads: int = 0) -> np.ndarray:
        bs, arr, lens = _seq_arrays(seqs)
        ia = np.ascontiguousarray(ia, dtype=np.uint32)
        ib = np.ascontiguousarray(ib, dtype=np.uint32)
        out = np.zeros(len(ia), dtype=np.uint32)
        threads = threads or os.cpu_count() or 1
        self._check(self.L.ref_lev_pairs(arr, lens.ctypes.data_as(_u32p), len(bs), ia.ctypes.data_as(_u32p),
                                         ib.ctypes.data_as(_u32p), len(ia), threads, out.ctypes.data_as(_u32p)))
        return out

    @staticmethod
    def _scheme_args(kind, symbols, matrix):
        k = {"nt": 0, "aa": 1, "custom": 2}[kind]
        if k == 2:
            m = (C.c_int * len(matrix))(*matrix)
            return k, _bytes(symbols), m
        return k, None, None

    def scheme_table(self, kind="nt", gap_open=-10, gap_extend=-1, flat=False, symbols=None, matrix=None):
        k, sy, m = self._scheme_args(kind, symbols, matrix)
        t = np.zeros(128 * 128, dtype=np.int16)
        osur = C.c_int()
        self._check(self.L.ref_scheme_table(k, sy, m, gap_open, gap_extend, int(flat), t.ctypes.data_as(_i16p),
                                            C.byref(osur)))
        return t, osur.value

    def nw_align(self, a, b, kind="nt", gap_open=-10, gap_extend=-1, flat=False, symbols=None, matrix=None):
        a, b = _bytes(a), _bytes(b)
        k, sy, m = self._scheme_args(kind, symbols, matrix)
        h = C.c_void_p()
        self._check(self.L.ref_nw_align(a, len(a), b, len(b), k, sy, m, gap_open, gap_extend, int(flat),
                                        C.byref(h)))
        L = self.L
        n = L.ref_pw_len(h)
        res = dict(score=L.ref_pw_score(h), aligned_a=C.string_at(L.ref_pw_a(h), n).decode(),
                   aligned_b=C.string_at(L.ref_pw_b(h), n).decode(),
                   gaps_into_a=list(np.ctypeslib.as_array(C.cast(L.ref_pw_gaps_a(h), _u32p),
                                                          shape=(L.ref_pw_ngaps_a(h),)).astype(int))
                   if L.ref_pw_ngaps_a(h) else [],
                   gaps_into_b=list(np.ctypeslib.as_array(C.cast(L.ref_pw_gaps_b(h), _u32p),
                                                          shape=(L.ref_pw_ngaps_b(h),)).astype(int))
                   if L.ref_pw_ngaps_b(h) else [])
        L.ref_pw_free(h)
        res["gaps_into_a"] = [int(x) for x in res["gaps_into_a"]]
        res["gaps_into_b"] = [int(x) for x in res["gaps_into_b"]]
        return res

    def build_tree(self, seqs, seed: int = 42, cap: int = 100, threads: int = 0):
        bs, arr, lens = _seq_arrays(seqs)
        n = len(bs)
        nodes = np.zeros((max(2 * n - 1, 1), 10), dtype=np.int64)
        order = np.zeros(max(n, 1), dtype=np.uint32)
        nn = C.c_uint64()
        threads = threads or os.cpu_count() or 1
        self._check(self.L.ref_build_tree(arr, lens.ctypes.data_as(_u32p), n, seed, cap, threads,
                                          nodes.ctypes.data_as(_i64p), C.byref(nn), order.ctypes.data_as(_u32p)))
        return nodes[:nn.value].copy(), order[:n].copy()

    def geometric_median(self, seqs, members, seed: int, cap: int = 100, threads: int = 0) -> int:
        bs, arr, lens = _seq_arrays(seqs)
        m = np.ascontiguousarray(members, dtype=np.uint32)
        out = C.c_uint32()
        self._check(self.L.ref_geometric_median(arr, lens.ctypes.data_as(_u32p), len(bs), m.ctypes.data_as(_u32p),
                                                len(m), seed, cap, threads or os.cpu_count() or 1, C.byref(out)))
        return int(out.value)

    def msa(self, seqs, kind="nt", gap_open=-10, gap_extend=-1, flat=False, seed=42, threads=0, symbols=None,
            matrix=None):
        """build_tree + align_all; returns dict(rows, width, row_seq, nodes, order, tree_s, align_s)."""
        bs, arr, lens = _seq_arrays(seqs)
        k, sy, m = self._scheme_args(kind, symbols, matrix)
        h = C.c_void_p()
        self._check(self.L.ref_msa(arr, lens.ctypes.data_as(_u32p), len(bs), k, sy, m, gap_open, gap_extend,
                                   int(flat), seed, threads or os.cpu_count() or 1, C.byref(h)))
        L = self.L
        W, R = L.ref_msa_width(h), L.ref_msa_rows(h)
        raw = C.string_at(L.ref_msa_data(h), W * R)
        rows = [raw[r * W:(r + 1) * W].decode() for r in range(R)]
        row_seq = np.ctypeslib.as_array(C.cast(L.ref_msa_row_seq(h), _u32p), shape=(R,)).copy()
        nn = L.ref_msa_nnodes(h)
        nodes = np.zeros((nn, 10), dtype=np.int64)
        order = np.zeros(len(bs), dtype=np.uint32)
        L.ref_msa_nodes(h, nodes.ctypes.data_as(_i64p), order.ctypes.data_as(_u32p))
        out = dict(rows=rows, width=W, row_seq=row_seq, nodes=nodes, order=order, tree_s=L.ref_msa_tree_s(h),
                   align_s=L.ref_msa_align_s(h))
        L.ref_msa_free(h)
        return out

    def align(self, seqs, alphabet="auto", gap_open=-10, gap_extend=-1, gap_mode="affine", seed=42, threads=0):
        bs, arr, lens = _seq_arrays(seqs)
        a = {"auto": 0, "nt": 1, "aa": 2}[alphabet]
        p = C.c_void_p()
        w = C.c_uint64()
        self._check(self.L.ref_align(arr, lens.ctypes.data_as(_u32p), len(bs), a, gap_open, gap_extend,
                                     int(gap_mode == "flat"), seed, threads, C.byref(p), C.byref(w)))
        raw = C.string_at(p, len(bs) * w.value)
        self.L.ref_free(p)
        W = w.value
        return [raw[r * W:(r + 1) * W].decode() for r in range(len(bs))]

    def evaluate(self, rows: List[str], row_to_sequence, raws, sample_size: int = 10000,
                 pair_budget: int = 100000, seed: int = 42, threads: int = 0) -> dict:
        """divmsa::evaluate (metrics.cpp:84-169) on an Msa given as rows."""
        width = len(rows[0]) if rows else 0
        block = "".join(rows).encode()
        rts = np.ascontiguousarray(row_to_sequence, dtype=np.uint32)
        bs, arr, lens = _seq_arrays(raws)
        out = RefMetrics()
        self._check(self.L.ref_evaluate(block, len(rows), width, rts.ctypes.data_as(_u32p), arr,
                                        lens.ctypes.data_as(_u32p), len(bs), sample_size, pair_budget, seed,
                                        threads or os.cpu_count() or 1, C.byref(out)))
        return {f: getattr(out, f) for f, _ in RefMetrics._fields_}

    def run_align(self, input_path: str, output_path: str, alphabet: str = "auto", gap_open: int = -10,
                  gap_extend: int = -1, flat: bool = False, seed: int = 42, order: str = "tree",
                  threads: int = 0, dump_tree: str | None = None, dump_dedup: str | None = None) -> None:
        """divmsa::run_align (pipeline.cpp:160-187): FASTA in, aligned FASTA out."""
        a = {"auto": 0, "nt": 1, "aa": 2}[alphabet]
        self._check(self.L.ref_run_align(input_path.encode(), output_path.encode(), a, gap_open, gap_extend,
                                         int(flat), seed, int(order == "input"), threads or os.cpu_count() or 1,
                                         dump_tree.encode() if dump_tree else None,
                                         dump_dedup.encode() if dump_dedup else None))

    def write_fasta(self, records, path: str) -> None:
        """divmsa::write_fasta over [(id, description, residues), ...]."""
        cols = []
        for f in range(3):
            bs = [_bytes(r[f]) for r in records]
            off = np.zeros(len(bs) + 1, dtype=np.uint64)
            off[1:] = np.cumsum([len(b) for b in bs]) if bs else []
            cols.append((b"".join(bs), off))
        self._check(self.L.ref_write_fasta(path.encode(), cols[0][0], cols[0][1].ctypes.data_as(_u64p), cols[1][0],
                                           cols[1][1].ctypes.data_as(_u64p), cols[2][0],
                                           cols[2][1].ctypes.data_as(_u64p), len(records)))

    def gap_percent(self, rows: List[str]) -> float:
        width = len(rows[0]) if rows else 0
        v = C.c_double()
        self._check(self.L.ref_gap_percent("".join(rows).encode(), len(rows), width, C.byref(v)))
        return v.value

    def p_score(self, a, b) -> float:
        a, b = _bytes(a), _bytes(b)
        v = C.c_double()
        self._check(self.L.ref_p_score(a, len(a), b, len(b), C.byref(v)))
        return v.value

    def hamming_aligned(self, a, b) -> int:
        a, b = _bytes(a), _bytes(b)
        v = C.c_uint32()
        self._check(self.L.ref_hamming_aligned(a, len(a), b, len(b), C.byref(v)))
        return v.value

    def distortion_pair(self, a, b, ra, rb) -> float:
        a, b, ra, rb = _bytes(a), _bytes(b), _bytes(ra), _bytes(rb)
        v = C.c_double()
        self._check(self.L.ref_distortion_pair(a, len(a), b, len(b), ra, len(ra), rb, len(rb), C.byref(v)))
        return v.value

    def insert_gap_columns(self, rows: List[str], positions) -> List[str]:
        width = len(rows[0]) if rows else 0
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        out = C.create_string_buffer(len(rows) * (width + len(pos)) + 1)
        self._check(self.L.ref_insert_gap_columns("".join(rows).encode(), len(rows), width,
                                                  pos.ctypes.data_as(_u32p), len(pos), out))
        w = width + len(pos)
        return [out.raw[r * w:(r + 1) * w].decode() for r in range(len(rows))]


_cache = {}


SYNTH_SO = os.path.join(HERE, "_build", "libsynth.so")
_synth_lib = None


def synth(cfg: int, scale: float = 1.0, seed: int = 0):
    """The seeded synthetic inputs of BASELINE config `cfg` from
    oracle/_build/libsynth.so (the generator source compiled on its own), so
    a CPU-only process gets the same inputs as the product's dm.synth without
    loading the product library. Returns (data: bytes, offsets: uint64[n+1])."""
    global _synth_lib
    if _synth_lib is None:
        L = C.CDLL(SYNTH_SO)
        L.dm_synth.restype = C.c_int
        L.dm_synth.argtypes = [C.c_int, C.c_double, C.c_uint64, C.POINTER(C.c_char_p), C.POINTER(_u64p),
                               C.POINTER(C.c_uint64)]
        _synth_lib = L
    libc = C.CDLL(None)
    data = C.c_char_p()
    offs = _u64p()
    n = C.c_uint64()
    if _synth_lib.dm_synth(cfg, float(scale), int(seed), C.byref(data), C.byref(offs), C.byref(n)) != 0:
        raise ValueError("dm_synth failed")
    try:
        o = np.ctypeslib.as_array(offs, shape=(n.value + 1,)).copy()
        buf = C.string_at(data, int(o[-1]))
    finally:
        libc.free(C.cast(data, C.c_void_p))
        libc.free(C.cast(offs, C.c_void_p))
    return buf, o


def restatement() -> Restatement:
    if "r" not in _cache:
        _cache["r"] = Restatement()
    return _cache["r"]


def reference() -> Reference:
    if "ref" not in _cache:
        _cache["ref"] = Reference()
    return _cache["ref"]


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)
