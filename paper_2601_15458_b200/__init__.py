"""B200-native MuSAlS hot path (arXiv 2601.15458).

Python face of libdmb200.so. It mirrors the reference's Python module
``divmsa`` (proj/python/py_module.cpp:73-190): ``levenshtein``, ``nw_align``,
``PairwiseResult``, ``align``; plus the batched and tree-level entry points
the reference keeps in C++ (``build_tree``, ``align_all``,
``geometric_median``, ``insert_gap_columns``). Every call goes through the C
ABI in include/dm_b200.h; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from ._lib import DmError, check, dm_metrics, dm_node, dm_stats, lib

__version__ = "0.1.0"

__all__ = [
    "Context", "SeqSet", "PairwiseResult", "DmError", "levenshtein", "lev_pairs", "lev_one_to_many",
    "geometric_median", "build_tree", "synth", "default_context", "__version__",
]


class Context:
    """One CUDA device + stream + scratch arena (dm_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().dm_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def sync(self):
        check(lib().dm_ctx_sync(self._h))

    def close(self):
        if self._h:
            lib().dm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _pack(seqs: Sequence) -> tuple:
    """Concatenate str/bytes sequences -> (bytes, uint64 offsets)."""
    bs = [s.encode() if isinstance(s, str) else bytes(s) for s in seqs]
    offs = np.zeros(len(bs) + 1, dtype=np.uint64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs], dtype=np.uint64)
    return b"".join(bs), offs


class SeqSet:
    """Device-resident sequences (dm_seqset): raw bytes + bit-plane profiles."""

    def __init__(self, seqs=None, ctx: Context | None = None, *, data: bytes | None = None,
                 offsets: np.ndarray | None = None):
        self.ctx = ctx or default_context()
        if data is None:
            data, offsets = _pack(seqs)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = len(offsets) - 1
        h = C.c_void_p()
        check(lib().dm_seqset_create(self.ctx.handle, data, offsets.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     n, C.byref(h)))
        self._h = h
        self.n = n
        self.lengths = np.diff(offsets).astype(np.int64)

    @property
    def handle(self):
        return self._h

    @property
    def planes(self) -> int:
        return lib().dm_seqset_planes(self._h)

    def __len__(self):
        return self.n

    def close(self):
        if self._h:
            lib().dm_seqset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a: np.ndarray, t=C.c_uint32):
    return a.ctypes.data_as(C.POINTER(t))


def levenshtein(a, b, ctx: Context | None = None) -> int:
    """divmsa.levenshtein (distance.hpp:11) on the GPU."""
    ctx = ctx or default_context()
    a = a.encode() if isinstance(a, str) else bytes(a)
    b = b.encode() if isinstance(b, str) else bytes(b)
    st = C.c_int(0)
    d = lib().dm_levenshtein(ctx.handle, a, len(a), b, len(b), C.byref(st))
    check(st.value)
    return int(d)


def lev_pairs(seqset: SeqSet, ia, ib, stats: bool = False):
    """out[i] = levenshtein(seq ia[i], seq ib[i]); batched (cluster_tree.cpp:36 batching)."""
    ia, ib = _u32(ia), _u32(ib)
    if ia.shape != ib.shape:
        raise ValueError("ia and ib must have the same length")
    out = np.empty(len(ia), dtype=np.uint32)
    s = dm_stats()
    check(lib().dm_lev_pairs(seqset.ctx.handle, seqset.handle, _ptr(ia), _ptr(ib), len(ia), _ptr(out),
                             C.byref(s)))
    return (out, s.as_dict()) if stats else out


def lev_pairs_packed(data, offsets, ctx: Context | None = None, stats: bool = False):
    """End-to-end batch from host memory: pair i = (sequence 2i, 2i+1) of
    (data, offsets); transfers overlap the kernels (dm_lev_pairs_packed).
    `data` may be bytes or an object exposing a host pointer (e.g. a pinned
    torch uint8 tensor, via .data_ptr())."""
    ctx = ctx or default_context()
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    npairs = (len(offsets) - 1) // 2
    out = np.empty(npairs, dtype=np.uint32)
    ptr = C.c_void_p(data.data_ptr()) if hasattr(data, "data_ptr") else C.cast(C.c_char_p(data), C.c_void_p)
    s = dm_stats()
    check(lib().dm_lev_pairs_packed(ctx.handle, ptr, _ptr(offsets, C.c_uint64), npairs, _ptr(out), C.byref(s)))
    return (out, s.as_dict()) if stats else out


def lev_one_to_many(seqset: SeqSet, origin: int, members, stats: bool = False):
    """distance_scan (cluster_tree.cpp:31-41): distances from `origin` to each member."""
    members = _u32(members)
    out = np.empty(len(members), dtype=np.uint32)
    s = dm_stats()
    check(lib().dm_lev_one_to_many(seqset.ctx.handle, seqset.handle, int(origin), _ptr(members),
                                   len(members), _ptr(out), C.byref(s)))
    return (out, s.as_dict()) if stats else out


NODE_FIELDS = ("begin", "end", "center", "radius", "pole_l", "pole_r", "left", "right", "parent", "depth")
NO_SEQUENCE = 0xFFFFFFFF  # cluster_tree.hpp:15 kNoSequence


_SIGNED = [NODE_FIELDS.index(f) for f in ("left", "right", "parent")]


def nodes_to_array(nodes, count: int) -> np.ndarray:
    """dm_node[count] (ten 32-bit fields) -> int64 [count, 10] in NODE_FIELDS order."""
    if count == 0:
        return np.zeros((0, len(NODE_FIELDS)), dtype=np.int64)
    raw = np.ctypeslib.as_array(C.cast(nodes, C.POINTER(C.c_uint32)), shape=(count * len(NODE_FIELDS),))
    u = raw.reshape(count, len(NODE_FIELDS))
    out = u.astype(np.int64)
    out[:, _SIGNED] = u[:, _SIGNED].view(np.int32)
    return out


def array_to_nodes(arr: np.ndarray):
    a = np.asarray(arr, dtype=np.int64).reshape(-1, len(NODE_FIELDS))
    out = (dm_node * max(len(a), 1))()
    if len(a):
        u = np.ascontiguousarray(a.astype(np.uint32))  # keep alive across the copy
        C.memmove(out, u.ctypes.data, u.nbytes)
    return out


def build_tree(seqset: SeqSet, seed: int = 42, exact_cap: int = 100, stats: bool = False):
    """divmsa::build_tree (cluster_tree.hpp:66-67) on the GPU.

    Returns (nodes, order): nodes is an int64 array [2n-1, 10] with columns
    NODE_FIELDS in the reference's BFS numbering; order the uint32 permutation."""
    n = seqset.n
    nodes = (dm_node * max(2 * n - 1, 1))()
    order = np.zeros(max(n, 1), dtype=np.uint32)
    nn = C.c_uint64()
    s = dm_stats()
    check(lib().dm_build_tree(seqset.ctx.handle, seqset.handle, int(seed), int(exact_cap), nodes, C.byref(nn),
                              _ptr(order), C.byref(s)))
    res = (nodes_to_array(nodes, nn.value), order[:n].copy())
    return res + (s.as_dict(),) if stats else res


def geometric_median(seqset: SeqSet, members, seed: int, exact_cap: int = 100) -> int:
    """divmsa::geometric_median (cluster_tree.hpp:56-59) on the GPU."""
    members = _u32(members)
    out = C.c_uint32()
    check(lib().dm_geometric_median(seqset.ctx.handle, seqset.handle, _ptr(members), len(members), int(seed),
                                    int(exact_cap), C.byref(out)))
    return int(out.value)


class ScoringScheme:
    """divmsa::ScoringScheme (pairwise.hpp:22-52): 128x128 int16 table over
    chars, the gap symbol a first-class row, affine or flat gap mode."""

    def __init__(self, table: np.ndarray, has_symbol: np.ndarray, gap_open: int, gap_extend: int, mode: str,
                 symbols: str):
        self.table = np.ascontiguousarray(table, dtype=np.int16)
        self.has_symbol = np.ascontiguousarray(has_symbol, dtype=np.uint8)
        self._gap_open, self._gap_extend, self.mode, self.symbols = gap_open, gap_extend, mode, symbols

    @classmethod
    def nucleotide(cls, gap_open: int = -10, gap_extend: int = -1, mode: str = "affine"):
        """default_nucleotide_scheme (pairwise.cpp:122-137)."""
        return cls._default(0, gap_open, gap_extend, mode, "ACGTURYSWKMBDHVN")

    @classmethod
    def protein(cls, gap_open: int = -10, gap_extend: int = -1, mode: str = "affine"):
        """default_protein_scheme, BLOSUM62 (pairwise.cpp:139-142)."""
        return cls._default(1, gap_open, gap_extend, mode, "ARNDCQEGHILKMFPSTWYVBZX*")

    @classmethod
    def _default(cls, kind, gap_open, gap_extend, mode, symbols):
        t = np.zeros(128 * 128, dtype=np.int16)
        h = np.zeros(128, dtype=np.uint8)
        o = C.c_int()
        check(lib().dm_scheme_default(kind, gap_open, gap_extend, int(_flat(mode)), _ptr(t, C.c_int16),
                                      _ptr(h, C.c_uint8), C.byref(o)))
        return cls(t, h, gap_open, gap_extend, mode, symbols)

    @classmethod
    def custom(cls, symbols: str, matrix, gap_open: int, gap_extend: int, mode: str = "affine",
               gap_scores=None, gap_gap: int = 0):
        """ScoringScheme(symbols, matrix, gap_open, gap_extend, mode) (pairwise.cpp:59-108)."""
        m = np.ascontiguousarray(np.asarray(matrix, dtype=np.int32).ravel())
        gs = None if gap_scores is None else np.ascontiguousarray(gap_scores, dtype=np.int32)
        t = np.zeros(128 * 128, dtype=np.int16)
        h = np.zeros(128, dtype=np.uint8)
        o = C.c_int()
        check(lib().dm_scheme_custom(symbols.encode(), len(symbols), _ptr(m, C.c_int) if m.size else None,
                                     gap_open, gap_extend, int(_flat(mode)), None if gs is None else _ptr(gs, C.c_int),
                                     gap_gap, _ptr(t, C.c_int16), _ptr(h, C.c_uint8), C.byref(o)))
        return cls(t, h, gap_open, gap_extend, mode, symbols)

    def score(self, x: str, y: str) -> int:
        return int(self.table[ord(x) * 128 + ord(y)])

    def has(self, c: str) -> bool:
        return bool(self.has_symbol[ord(c)]) if ord(c) < 128 else False

    def gap_open(self) -> int:
        return self._gap_open

    def gap_extend(self) -> int:
        return self._gap_extend

    def open_surcharge(self) -> int:
        """gap_open in affine mode, 0 in flat mode (pairwise.hpp:36-38)."""
        return self._gap_open if self.mode == "affine" else 0


def _flat(mode: str) -> bool:
    if mode not in ("affine", "flat"):
        raise ValueError(f"unknown gap mode '{mode}' (expected affine or flat)")
    return mode == "flat"


def _scheme_for(alphabet: str, gap_open: int, gap_extend: int, gap_mode: str) -> ScoringScheme:
    """py_module.cpp scheme_for: alphabet 'nt' | 'aa'."""
    if alphabet == "nt":
        return ScoringScheme.nucleotide(gap_open, gap_extend, gap_mode)
    if alphabet == "aa":
        return ScoringScheme.protein(gap_open, gap_extend, gap_mode)
    raise ValueError(f"unknown alphabet '{alphabet}' (expected nt or aa)")


@dataclass
class PairwiseResult:
    """divmsa::PairwiseResult (pairwise.hpp:78-84)."""
    aligned_a: str
    aligned_b: str
    score: int
    gaps_into_a: List[int] = field(default_factory=list)
    gaps_into_b: List[int] = field(default_factory=list)

    def __repr__(self):
        return f"PairwiseResult(aligned_a='{self.aligned_a}', aligned_b='{self.aligned_b}', score={self.score})"


def _pw_results(h, count: int) -> List[PairwiseResult]:
    L = lib()
    out = []
    for k in range(count):
        n = L.dm_pw_len(h, k)
        a = C.create_string_buffer(n + 1)
        b = C.create_string_buffer(n + 1)
        L.dm_pw_aligned(h, k, a, b)
        ga = np.zeros(max(L.dm_pw_ngaps_a(h, k), 1), dtype=np.uint32)
        gb = np.zeros(max(L.dm_pw_ngaps_b(h, k), 1), dtype=np.uint32)
        L.dm_pw_gaps(h, k, _ptr(ga), _ptr(gb))
        out.append(PairwiseResult(a.raw[:n].decode("latin-1"), b.raw[:n].decode("latin-1"), int(L.dm_pw_score(h, k)),
                                  [int(x) for x in ga[:L.dm_pw_ngaps_a(h, k)]],
                                  [int(x) for x in gb[:L.dm_pw_ngaps_b(h, k)]]))
    return out


def nw_align(a, b, alphabet="nt", gap_open: int = -10, gap_extend: int = -1, gap_mode: str = "affine",
             scheme: ScoringScheme | None = None, ctx: Context | None = None) -> PairwiseResult:
    """divmsa.nw_align (py_module.cpp:105-118 -> pairwise.cpp:301) on the GPU."""
    ctx = ctx or default_context()
    sc = scheme or _scheme_for(alphabet, gap_open, gap_extend, gap_mode)
    a = a.encode() if isinstance(a, str) else bytes(a)
    b = b.encode() if isinstance(b, str) else bytes(b)
    h = C.c_void_p()
    check(lib().dm_nw_align(ctx.handle, a, len(a), b, len(b), _ptr(sc.table, C.c_int16),
                            _ptr(sc.has_symbol, C.c_uint8), sc.open_surcharge(), sc.gap_extend(), C.byref(h)))
    try:
        return _pw_results(h, 1)[0]
    finally:
        lib().dm_pw_free(h)


def nw_batch(pairs, scheme: ScoringScheme, ctx: Context | None = None, stats: bool = False):
    """Batched nw_align over [(a, b), ...] (one device launch pair)."""
    ctx = ctx or default_context()
    A, ao = _pack([p[0] for p in pairs])
    B, bo = _pack([p[1] for p in pairs])
    h = C.c_void_p()
    s = dm_stats()
    check(lib().dm_nw_batch(ctx.handle, A, _ptr(ao, C.c_uint64), B, _ptr(bo, C.c_uint64), len(pairs),
                            _ptr(scheme.table, C.c_int16), _ptr(scheme.has_symbol, C.c_uint8), scheme.open_surcharge(),
                            scheme.gap_extend(), C.byref(h), C.byref(s)))
    try:
        res = _pw_results(h, len(pairs))
    finally:
        lib().dm_pw_free(h)
    return (res, s.as_dict()) if stats else res


def insert_gap_columns(rows: List[str], positions, ctx: Context | None = None) -> List[str]:
    """divmsa::insert_gap_columns (msa_merge.hpp:34-35) on the GPU."""
    ctx = ctx or default_context()
    width = len(rows[0]) if rows else 0
    pos = _u32(positions)
    nw = width + len(pos)
    out = C.create_string_buffer(max(len(rows) * nw, 1))
    check(lib().dm_insert_gap_columns(ctx.handle, "".join(rows).encode(), len(rows), width, _ptr(pos), len(pos), out))
    return [out.raw[r * nw:(r + 1) * nw].decode("latin-1") for r in range(len(rows))]


@dataclass
class Msa:
    """divmsa::Msa (msa_merge.hpp:18-26): rows in tree order."""
    rows: List[str]
    row_to_sequence: np.ndarray
    width: int
    nodes: np.ndarray = None
    order: np.ndarray = None
    stats: dict = None

    def row_of(self, sequence: int) -> int:
        hit = np.nonzero(self.row_to_sequence == sequence)[0]
        if len(hit) == 0:
            raise ValueError(f"center row for sequence {sequence} not found in alignment")
        return int(hit[0])


def _msa_from(h) -> Msa:
    L = lib()
    W, R = L.dm_msa_width(h), L.dm_msa_rows(h)
    buf = bytearray(max(W * R, 1))
    L.dm_msa_copy_rows(h, (C.c_char * len(buf)).from_buffer(buf))
    rs = np.zeros(max(R, 1), dtype=np.uint32)
    L.dm_msa_copy_row_seq(h, _ptr(rs))
    nn = L.dm_msa_nnodes(h)
    nodes = (dm_node * max(nn, 1))()
    order = np.zeros(max(R, 1), dtype=np.uint32)
    L.dm_msa_copy_tree(h, nodes, _ptr(order))
    text = buf.decode("latin-1") if W * R else ""  # one decode, then str slices
    return Msa([text[r * W:(r + 1) * W] for r in range(R)], rs[:R].copy(), int(W),
               nodes_to_array(nodes, nn), order[:R].copy())


def align_all(seqset: SeqSet, nodes: np.ndarray, order, scheme: ScoringScheme, stats: bool = False,
              progress=None) -> Msa:
    """divmsa::align_all (msa_merge.hpp:47-49) on the GPU: per-level merge scheduler.
    progress(done, total) is called once per node as it completes (ProgressFn)."""
    from ._lib import PROGRESS_FN
    order = _u32(order)
    nd = array_to_nodes(nodes)
    h = C.c_void_p()
    s = dm_stats()
    errors = []

    def _cb(done, total, _user):
        try:
            progress(int(done), int(total))
        except BaseException as e:  # noqa: BLE001 -- re-raised after the call
            errors.append(e)

    cb = PROGRESS_FN(_cb) if progress else None
    check(lib().dm_align_all_progress(seqset.ctx.handle, seqset.handle, nd, len(nodes), _ptr(order),
                                      _ptr(scheme.table, C.c_int16), _ptr(scheme.has_symbol, C.c_uint8),
                                      scheme.open_surcharge(), scheme.gap_extend(),
                                      C.cast(cb, C.c_void_p) if cb else None, None, C.byref(h), C.byref(s)))
    if errors:
        lib().dm_msa_free(h)
        raise errors[0]
    try:
        m = _msa_from(h)
    finally:
        lib().dm_msa_free(h)
    m.stats = s.as_dict()
    return m


def msa(seqset: SeqSet, scheme: ScoringScheme, seed: int = 42, exact_cap: int = 100) -> Msa:
    """build_tree + align_all (pipeline.cpp:116-128), device-resident between the two."""
    h = C.c_void_p()
    s = dm_stats()
    check(lib().dm_msa(seqset.ctx.handle, seqset.handle, int(seed), int(exact_cap), _ptr(scheme.table, C.c_int16),
                       _ptr(scheme.has_symbol, C.c_uint8), scheme.open_surcharge(), scheme.gap_extend(), C.byref(h),
                       C.byref(s)))
    try:
        m = _msa_from(h)
    finally:
        lib().dm_msa_free(h)
    m.stats = s.as_dict()
    return m


def align(sequences: Sequence, alphabet: str = "auto", gap_open: int = -10, gap_extend: int = -1,
          gap_mode: str = "affine", seed: int = 42, threads: int = 0, scheme: ScoringScheme | None = None,
          order: str = "input", ctx: Context | None = None, summary: bool = False):
    """divmsa.align (py_module.cpp:120-155 -> align_sequences, pipeline.cpp:78-159).

    Returns gapped rows parallel to the input (RowOrder::Input). `threads` is
    accepted for API parity; the work runs on the GPU."""
    from ._lib import dm_align_summary
    ctx = ctx or default_context()
    amap = {"auto": 0, "nt": 1, "dna": None, "aa": 2}
    if alphabet not in ("auto", "nt", "aa"):
        raise ValueError(f"unknown alphabet '{alphabet}' (expected auto, nt or aa)")
    flat = _flat(gap_mode)
    data, offs = _pack(sequences)
    rows = C.c_void_p()
    width = C.c_uint64()
    summ = dm_align_summary()
    s = dm_stats()
    check(lib().dm_align_sequences(ctx.handle, data, _ptr(offs, C.c_uint64), len(offs) - 1, amap[alphabet], gap_open,
                                   gap_extend, int(flat), None if scheme is None else _ptr(scheme.table, C.c_int16),
                                   None if scheme is None else _ptr(scheme.has_symbol, C.c_uint8), int(seed),
                                   int(order == "input"), C.byref(rows), C.byref(width), C.byref(summ), C.byref(s)))
    try:
        W = width.value
        raw = C.string_at(rows, W * (len(offs) - 1))
    finally:
        lib().dm_free(rows)
    text = raw.decode("latin-1")
    out = [text[r * W:(r + 1) * W] for r in range(len(offs) - 1)]
    if summary:
        return out, {f: getattr(summ, f) for f, _ in summ._fields_}, s.as_dict()
    return out


# ---- quality metrics (divmsa/metrics.hpp; metrics.cpp, distance.cpp:50-57) --------------

def _rows_block(rows) -> tuple:
    rows = [r.encode() if isinstance(r, str) else bytes(r) for r in rows]
    width = len(rows[0]) if rows else 0
    if any(len(r) != width for r in rows):
        raise ValueError("alignment rows must have equal width")
    return b"".join(rows), len(rows), width


def evaluate(msa_: Msa, raws, sample_size: int = 10000, pair_budget: int = 100000, seed: int = 42,
             ctx: Context | None = None) -> dict:
    """divmsa::evaluate (metrics.hpp:53-56): width, stretch, gap_percent and
    the seeded pair sample's p-distance / distortion statistics. `raws` are
    the unaligned sequences indexed by msa_.row_to_sequence. Bit-identical
    to the reference; the pair work runs on the GPU."""
    ctx = ctx or default_context()
    block, nrows, width = _rows_block(msa_.rows)
    rts = np.ascontiguousarray(msa_.row_to_sequence, dtype=np.uint32)
    raw, offs = _pack(raws)
    out = dm_metrics()
    check(lib().dm_evaluate(ctx.handle, block, nrows, width, _ptr(rts), raw, _ptr(offs, C.c_uint64), len(offs) - 1,
                            int(sample_size), int(pair_budget), int(seed), C.byref(out)))
    return out.as_dict()


def gap_percent(msa_or_rows, ctx: Context | None = None) -> float:
    """divmsa::gap_percent (metrics.cpp:16-27)."""
    ctx = ctx or default_context()
    rows = msa_or_rows.rows if isinstance(msa_or_rows, Msa) else msa_or_rows
    block, nrows, width = _rows_block(rows)
    v = C.c_double()
    check(lib().dm_gap_percent(ctx.handle, block, nrows, width, C.byref(v)))
    return v.value


def _row_pair(a, b, ctx, what: str):
    a = a.encode() if isinstance(a, str) else bytes(a)
    b = b.encode() if isinstance(b, str) else bytes(b)
    if len(a) != len(b):
        raise ValueError(f"{what} requires equal-length rows")
    cons, mism, ham = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib().dm_row_pair_stats((ctx or default_context()).handle, a, len(a), b, len(b), C.byref(cons),
                                  C.byref(mism), C.byref(ham)))
    return cons.value, mism.value, ham.value


def p_score(a, b, ctx: Context | None = None) -> float:
    """divmsa::p_score (metrics.cpp:29-45): mismatches over shared residue columns, 1.0 when none."""
    cons, mism, _ = _row_pair(a, b, ctx, "p_score")
    return 1.0 if cons == 0 else mism / cons


def hamming_aligned(a, b, ctx: Context | None = None) -> int:
    """divmsa::hamming_aligned (distance.cpp:50-57)."""
    return _row_pair(a, b, ctx, "hamming_aligned")[2]


def distortion_pair(a_aligned, b_aligned, a_raw, b_raw, ctx: Context | None = None) -> float:
    """divmsa::distortion_pair (metrics.cpp:47-56): aligned hamming / raw levenshtein."""
    lev = levenshtein(a_raw, b_raw, ctx)
    if lev == 0:
        raise ValueError("distortion is undefined for identical sequences")
    return hamming_aligned(a_aligned, b_aligned, ctx) / lev


# ---- FASTA in / out (seq_io.hpp, pipeline.hpp:63-64) ---------------------------------------

def run_align(input_path, output_path, alphabet: str = "auto", gap_open: int = -10, gap_extend: int = -1,
              gap_mode: str = "affine", seed: int = 42, order: str = "tree", scheme: ScoringScheme | None = None,
              dump_tree=None, dump_dedup=None, ctx: Context | None = None, stats: bool = False):
    """divmsa::run_align (pipeline.cpp:160-187): parse the FASTA file, align
    (tree + merges on the GPU), write the aligned FASTA (assembled on the GPU)
    to output_path via a ".partial" sibling. Returns the AlignSummary fields."""
    from ._lib import dm_align_summary
    ctx = ctx or default_context()
    if alphabet not in ("auto", "nt", "aa"):
        raise ValueError(f"unknown alphabet '{alphabet}' (expected auto, nt or aa)")
    if order not in ("tree", "input"):
        raise ValueError("order must be 'tree' or 'input'")
    summ = dm_align_summary()
    s = dm_stats()
    check(lib().dm_run_align(ctx.handle, str(input_path).encode(), str(output_path).encode(),
                             {"auto": 0, "nt": 1, "aa": 2}[alphabet], gap_open, gap_extend, int(_flat(gap_mode)),
                             None if scheme is None else _ptr(scheme.table, C.c_int16),
                             None if scheme is None else _ptr(scheme.has_symbol, C.c_uint8), int(seed),
                             int(order == "input"), str(dump_tree).encode() if dump_tree else None,
                             str(dump_dedup).encode() if dump_dedup else None, C.byref(summ), C.byref(s)))
    out = {f: getattr(summ, f) for f, _ in summ._fields_}
    return (out, s.as_dict()) if stats else out


def dump_tree(nodes, ids, path) -> None:
    """divmsa::dump_tree (cluster_tree.cpp:253-280): NDJSON, one line per node
    (`nodes` as returned by build_tree, `ids` indexed by sequence)."""
    arr = nodes if isinstance(nodes, np.ndarray) else np.asarray(nodes)
    nn = len(arr)
    cn = array_to_nodes(arr)
    data, offs = _pack(ids)
    check(lib().dm_dump_tree(cn, nn, data, _ptr(offs, C.c_uint64), len(ids), str(path).encode()))


def write_fasta(records, path, ctx: Context | None = None) -> None:
    """divmsa::write_fasta (seq_io.cpp:188-225) over [(id, description, residues), ...]:
    80-column lines, text assembled on the GPU."""
    ctx = ctx or default_context()
    cols = [_pack([r[f] for r in records]) for f in range(3)]
    check(lib().dm_write_fasta(ctx.handle, str(path).encode(), cols[0][0], _ptr(cols[0][1], C.c_uint64), cols[1][0],
                               _ptr(cols[1][1], C.c_uint64), cols[2][0], _ptr(cols[2][1], C.c_uint64), len(records)))


def parse_fasta(path, alphabet: str | None = None, allow_gaps: bool = False) -> list:
    """divmsa::parse_fasta (seq_io.cpp:44-119): [(id, description, residues), ...]."""
    a = {None: 0, "nt": 1, "aa": 2}[alphabet]
    ptrs = [C.c_void_p() for _ in range(3)]
    offs = [C.POINTER(C.c_uint64)() for _ in range(3)]
    n = C.c_uint64()
    check(lib().dm_parse_fasta(str(path).encode(), a, int(allow_gaps), C.byref(ptrs[0]), C.byref(offs[0]),
                               C.byref(ptrs[1]), C.byref(offs[1]), C.byref(ptrs[2]), C.byref(offs[2]), C.byref(n)))
    try:
        cols = []
        for f in range(3):
            o = np.ctypeslib.as_array(offs[f], shape=(n.value + 1,)).copy()
            raw = C.string_at(ptrs[f], int(o[-1])) if o[-1] else b""
            cols.append([raw[int(o[k]):int(o[k + 1])].decode("latin-1") for k in range(n.value)])
    finally:
        for f in range(3):
            lib().dm_free(ptrs[f])
            lib().dm_free(C.cast(offs[f], C.c_void_p))
    return list(zip(*cols))


def synth(cfg: int, scale: float = 1.0, seed: int = 0):
    """Seeded synthetic inputs of BASELINE config `cfg`.

    Returns (data: bytes, offsets: np.uint64[n+1])."""
    data = C.c_char_p()
    offs = C.POINTER(C.c_uint64)()
    n = C.c_uint64()
    check(lib().dm_synth(cfg, float(scale), int(seed), C.byref(data), C.byref(offs), C.byref(n)))
    try:
        o = np.ctypeslib.as_array(offs, shape=(n.value + 1,)).copy()
        buf = C.string_at(data, int(o[-1]))
    finally:
        lib().dm_free(C.cast(data, C.c_void_p))
        lib().dm_free(C.cast(offs, C.c_void_p))
    return buf, o


def split(data: bytes, offsets: np.ndarray) -> List[bytes]:
    return [data[int(offsets[i]):int(offsets[i + 1])] for i in range(len(offsets) - 1)]
