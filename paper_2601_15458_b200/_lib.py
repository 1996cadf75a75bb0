"""ctypes binding of libdmb200.so (the C ABI declared in include/dm_b200.h).

The product has no CPU fallback: if the shared library is missing, or no
B200 is visible when a compute call is made, these functions raise.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DM_LIB_PATH: load a differently-built copy (tuning experiments only)
LIB_PATH = os.environ.get("DM_LIB_PATH") or os.path.join(_HERE, "libdmb200.so")

DM_OK, DM_EINVAL, DM_ERUNTIME, DM_ECUDA, DM_ENOMEM = 0, 1, 2, 3, 4


class DmError(RuntimeError):
    """A CUDA / runtime failure inside libdmb200 (DM_ECUDA / DM_ENOMEM)."""


# dm_progress_fn (include/dm_b200.h): void (*)(uint64_t done, uint64_t total, void* user)
PROGRESS_FN = C.CFUNCTYPE(None, C.c_uint64, C.c_uint64, C.c_void_p)


class dm_node(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in ("begin", "end", "center", "radius", "pole_l", "pole_r")] + [
        (f, C.c_int32) for f in ("left", "right", "parent")] + [("depth", C.c_uint32)]


class dm_metrics(C.Structure):
    """divmsa::MetricsReport (metrics.hpp:13-35)."""
    _fields_ = [("width", C.c_uint64)] + [(f, C.c_double) for f in (
        "stretch", "gap_percent", "distortion", "p_min", "p_avg", "p_max")] + [(f, C.c_uint64) for f in (
            "sample_size", "pair_count", "seed", "zero_distance_pairs")] + [("time_s", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class dm_stats(C.Structure):
    _fields_ = [("kernel_ms", C.c_double), ("total_ms", C.c_double), ("cells", C.c_uint64),
                ("cells_executed", C.c_uint64), ("launches", C.c_uint64), ("tree_ms", C.c_double),
                ("align_ms", C.c_double), ("lev_calls", C.c_uint64), ("nw_calls", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("cells_reused", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class dm_align_summary(C.Structure):
    _fields_ = [("input_count", C.c_uint64), ("unique_count", C.c_uint64), ("duplicate_count", C.c_uint64),
                ("tree_depth", C.c_uint32), ("width", C.c_uint64), ("alphabet", C.c_int),
                ("elapsed_s", C.c_double)]


_P = C.c_void_p
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i16p = C.POINTER(C.c_int16)
_u8p = C.POINTER(C.c_uint8)

# name -> (restype, argtypes). Every symbol declared in include/dm_b200.h.
SIGNATURES = {
    "dm_last_error": (C.c_char_p, []),
    "dm_abi_version": (C.c_int, []),
    "dm_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "dm_ctx_destroy": (C.c_int, [_P]),
    "dm_ctx_sync": (C.c_int, [_P]),
    "dm_ctx_set_stream": (C.c_int, [_P, _P]),
    "dm_int32_peak": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double)]),
    "dm_nccl_unique_id": (C.c_int, [_u8p]),
    "dm_ctx_attach_nccl": (C.c_int, [_P, _u8p, C.c_int, C.c_int]),
    "dm_ctx_simulate_world": (C.c_int, [_P, C.c_int]),
    "dm_ctx_set_shard": (C.c_int, [_P, C.c_int, C.c_int]),
    "dm_seqset_create": (C.c_int, [_P, C.c_char_p, _u64p, C.c_uint32, C.POINTER(_P)]),
    "dm_seqset_destroy": (C.c_int, [_P]),
    "dm_seqset_count": (C.c_uint32, [_P]),
    "dm_seqset_planes": (C.c_int, [_P]),
    "dm_levenshtein": (C.c_uint32, [_P, C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.POINTER(C.c_int)]),
    "dm_lev_pairs": (C.c_int, [_P, _P, _u32p, _u32p, C.c_uint64, _u32p, C.POINTER(dm_stats)]),
    "dm_lev_pairs_device": (C.c_int, [_P, _P, _P, _P, C.c_uint64, _P, C.POINTER(dm_stats)]),
    "dm_lev_pairs_packed": (C.c_int, [_P, C.c_void_p, _u64p, C.c_uint64, _u32p, C.POINTER(dm_stats)]),
    "dm_pack_nt": (C.c_int, [C.c_char_p, C.c_uint64, C.c_void_p]),
    "dm_pack_nt_seqs": (C.c_int, [C.c_char_p, _u64p, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64)]),
    "dm_lev_one_to_many": (C.c_int, [_P, _P, C.c_uint32, _u32p, C.c_uint64, _u32p, C.POINTER(dm_stats)]),
    "dm_geometric_median": (C.c_int, [_P, _P, _u32p, C.c_uint64, C.c_uint64, C.c_uint64, _u32p]),
    "dm_build_tree": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64, C.POINTER(dm_node), _u64p, _u32p,
                                C.POINTER(dm_stats)]),
    "dm_nw_align": (C.c_int, [_P, C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, _i16p, _u8p, C.c_int,
                              C.c_int, C.POINTER(_P)]),
    "dm_nw_batch": (C.c_int, [_P, C.c_char_p, _u64p, C.c_char_p, _u64p, C.c_uint32, _i16p, _u8p, C.c_int,
                              C.c_int, C.POINTER(_P), C.POINTER(dm_stats)]),
    "dm_pw_score": (C.c_int64, [_P, C.c_uint32]),
    "dm_pw_len": (C.c_uint64, [_P, C.c_uint32]),
    "dm_pw_aligned": (C.c_int, [_P, C.c_uint32, C.c_char_p, C.c_char_p]),
    "dm_pw_ngaps_a": (C.c_uint64, [_P, C.c_uint32]),
    "dm_pw_ngaps_b": (C.c_uint64, [_P, C.c_uint32]),
    "dm_pw_gaps": (C.c_int, [_P, C.c_uint32, _u32p, _u32p]),
    "dm_pw_free": (None, [_P]),
    "dm_insert_gap_columns": (C.c_int, [_P, C.c_char_p, C.c_uint64, C.c_uint64, _u32p, C.c_uint64,
                                        C.c_char_p]),
    "dm_align_all": (C.c_int, [_P, _P, C.POINTER(dm_node), C.c_uint64, _u32p, _i16p, _u8p, C.c_int, C.c_int,
                               C.POINTER(_P), C.POINTER(dm_stats)]),
    "dm_align_all_progress": (C.c_int, [_P, _P, C.POINTER(dm_node), C.c_uint64, _u32p, _i16p, _u8p, C.c_int, C.c_int,
                                        C.c_void_p, C.c_void_p, C.POINTER(_P), C.POINTER(dm_stats)]),
    "dm_ctx_attach_host_comm": (C.c_int, [_P, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "dm_shard_bounds": (C.c_int, [_u64p, C.c_uint64, C.c_int, _u64p]),
    "dm_ctx_comm_stats": (C.c_int, [_P, _u64p]),
    "dm_assign_owners": (C.c_int, [_u64p, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]),
    "dm_format_tree": (C.c_int, [C.POINTER(dm_node), C.c_uint64, C.c_char_p, _u64p, C.c_uint64,
                                 C.POINTER(C.c_void_p), _u64p]),
    "dm_msa": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64, _i16p, _u8p, C.c_int, C.c_int, C.POINTER(_P),
                         C.POINTER(dm_stats)]),
    "dm_msa_width": (C.c_uint64, [_P]),
    "dm_msa_rows": (C.c_uint64, [_P]),
    "dm_msa_copy_rows": (C.c_int, [_P, C.c_char_p]),
    "dm_msa_copy_row_seq": (C.c_int, [_P, _u32p]),
    "dm_msa_nnodes": (C.c_uint64, [_P]),
    "dm_msa_copy_tree": (C.c_int, [_P, C.POINTER(dm_node), _u32p]),
    "dm_msa_free": (None, [_P]),
    "dm_scheme_default": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _i16p, _u8p, C.POINTER(C.c_int)]),
    "dm_scheme_custom": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_int), C.c_int, _i16p, _u8p, C.POINTER(C.c_int)]),
    "dm_align_sequences": (C.c_int, [_P, C.c_char_p, _u64p, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, _i16p,
                                     _u8p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p), _u64p, _P,
                                     C.POINTER(dm_stats)]),
    "dm_synth": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.POINTER(C.c_char_p), C.POINTER(_u64p), _u64p]),
    "dm_evaluate": (C.c_int, [_P, C.c_char_p, C.c_uint64, C.c_uint64, _u32p, C.c_char_p, _u64p, C.c_uint32,
                              C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(dm_metrics)]),
    "dm_gap_percent": (C.c_int, [_P, C.c_char_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]),
    "dm_row_pair_stats": (C.c_int, [_P, C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, _u32p, _u32p, _u32p]),
    "dm_run_align": (C.c_int, [_P, C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, _i16p, _u8p,
                               C.c_uint64, C.c_int, C.c_char_p, C.c_char_p, _P, C.POINTER(dm_stats)]),
    "dm_dump_tree": (C.c_int, [C.POINTER(dm_node), C.c_uint64, C.c_char_p, _u64p, C.c_uint64, C.c_char_p]),
    "dm_write_fasta": (C.c_int, [_P, C.c_char_p, C.c_char_p, _u64p, C.c_char_p, _u64p, C.c_char_p, _u64p,
                                 C.c_uint64]),
    "dm_parse_fasta": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_u64p),
                                 C.POINTER(C.c_void_p), C.POINTER(_u64p), C.POINTER(C.c_void_p), C.POINTER(_u64p),
                                 _u64p]),
    "dm_free": (None, [_P]),
}

_lib = None


def lib():
    """Load libdmb200.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the CUDA extension is required; there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:  # reported by tests/test_capi.py::test_exports
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    """Map a DM_* status onto the exception type the reference throws."""
    if rc == DM_OK:
        return
    msg = (lib().dm_last_error() or b"").decode(errors="replace")
    if rc == DM_EINVAL:
        raise ValueError(msg)  # std::invalid_argument (pybind11 maps it to ValueError)
    if rc == DM_ERUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    raise DmError(msg)
