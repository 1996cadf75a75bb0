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

from ._lib import DmError, check, dm_node, dm_stats, lib

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


def nodes_to_array(nodes, count: int) -> np.ndarray:
    return np.array([[getattr(nodes[i], f) for f in NODE_FIELDS] for i in range(count)], dtype=np.int64)


def array_to_nodes(arr: np.ndarray):
    out = (dm_node * len(arr))()
    for i, row in enumerate(np.asarray(arr, dtype=np.int64)):
        for f, v in zip(NODE_FIELDS, row):
            setattr(out[i], f, int(v))
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
