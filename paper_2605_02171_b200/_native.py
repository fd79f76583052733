"""ctypes binding of libqvg.so (include/qvg.h).

Loading fails loudly when the CUDA library is missing — there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libqvg.so")

QVG_OK = 0
QVG_INVALID_ARGUMENT = 1
QVG_CUDA_ERROR = 2
QVG_OUT_OF_MEMORY = 3
QVG_CAPACITY_OVERFLOW = 4
QVG_NOT_IMPLEMENTED = 5
QVG_RUNTIME_ERROR = 6

SENTINEL = 0xFFFFFFFF

# every symbol include/qvg.h declares
EXPORTED_SYMBOLS = (
    "qvg_last_error", "qvg_abi_version", "qvg_index_create", "qvg_index_load",
    "qvg_index_save", "qvg_index_destroy", "qvg_index_info", "qvg_index_set_stream",
    "qvg_index_export", "qvg_search", "qvg_search_ex", "qvg_beam_search", "qvg_encode",
    "qvg_sm2_distance", "qvg_build", "qvg_brute_force_topk", "qvg_compatibility_probe",
    "qvg_strong_bit_rate", "qvg_encode_rows", "qvg_robust_prune",
)


class qvg_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "queries", "expansions", "tie_expansions", "dist_evals", "inpool_drops",
        "adjacency_slots", "cold_accesses", "tie_overflows", "max_tie_depth",
        "adjacency_bytes", "code_bytes", "rerank_bytes", "io_bytes")] + [
        (n, C.c_double) for n in ("encode_ms", "search_ms", "device_ms", "total_ms")] + [
        (n, C.c_uint32) for n in ("grid_blocks", "warps_per_block", "smem_per_block",
                                  "resident_warps_per_sm")]

    def to_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class qvg_search_opts(C.Structure):
    _fields_ = [("visited_slots", C.c_uint32), ("tie_capacity", C.c_uint32),
                ("exact_visited", C.c_uint32), ("entry_point", C.c_uint32),
                ("no_rerank", C.c_uint32), ("timing_only", C.c_uint32),
                ("rerank_depth", C.c_uint32), ("relaxed_expansions", C.c_uint32)]


class qvg_build_params(C.Structure):
    _fields_ = [("m", C.c_uint32), ("ef_c", C.c_uint32), ("alpha", C.c_float),
                ("passes", C.c_uint32), ("batch", C.c_uint32), ("seed", C.c_uint64),
                ("prune_candidates", C.c_uint32), ("reserved", C.c_uint32 * 3)]


class qvg_build_stats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("reprunes", C.c_uint64), ("batches", C.c_uint64),
                ("mean_degree", C.c_double), ("min_degree", C.c_uint32),
                ("max_degree", C.c_uint32)]


class qvg_probe_report(C.Structure):
    _fields_ = [("overlap_at_k", C.c_double), ("sample_size", C.c_uint64), ("k", C.c_uint32),
                ("go", C.c_uint32)]


class qvg_encoding_diagnostics(C.Structure):
    _fields_ = [("sample_size", C.c_uint64), ("p_s", C.c_double), ("nu2", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    global LIB_PATH
    LIB_PATH = os.environ.get("QVG_LIB", LIB_PATH)  # A/B of two builds (tools/)
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 query path has no CPU fallback. "
            "Build it with `python paper_2605_02171_b200/build.py`.")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    L.qvg_last_error.restype = C.c_char_p
    L.qvg_abi_version.restype = C.c_int
    L.qvg_index_create.argtypes = [vp, u64, u32, vp, u32, vp, u32, i32, C.POINTER(vp)]
    L.qvg_index_load.argtypes = [C.c_char_p, i32, C.POINTER(vp)]
    L.qvg_index_save.argtypes = [vp, C.c_char_p]
    L.qvg_index_destroy.argtypes = [vp]
    L.qvg_index_destroy.restype = None
    L.qvg_index_info.argtypes = [vp, C.POINTER(u64), C.POINTER(u32), C.POINTER(u32),
                                 C.POINTER(u32)]
    L.qvg_index_set_stream.argtypes = [vp, vp]
    L.qvg_index_export.argtypes = [vp, vp, vp, vp]
    L.qvg_search.argtypes = [vp, vp, u64, u32, u32, vp, vp, vp, vp, C.POINTER(qvg_stats)]
    L.qvg_search_ex.argtypes = [vp, vp, u64, u32, u32, C.POINTER(qvg_search_opts), vp, vp, vp,
                                vp, vp, vp, vp, vp, C.POINTER(qvg_stats)]
    L.qvg_beam_search.argtypes = [vp, vp, u64, u32, u32, vp, vp, vp, C.POINTER(qvg_stats)]
    L.qvg_encode.argtypes = [i32, vp, u64, u32, vp, vp, vp, vp]
    L.qvg_sm2_distance.argtypes = [vp, vp, vp, u64, vp]
    L.qvg_build.argtypes = [vp, u64, u32, C.POINTER(qvg_build_params), i32, C.POINTER(vp),
                            C.POINTER(qvg_build_stats)]
    L.qvg_brute_force_topk.argtypes = [i32, vp, u64, vp, u64, u32, u32, i32, i32, vp, vp, vp, vp]
    L.qvg_compatibility_probe.argtypes = [i32, vp, u64, u32, u64, u32, i32,
                                          C.POINTER(qvg_probe_report)]
    L.qvg_encode_rows.argtypes = [i32, vp, u64, u32, i32, vp, vp]
    L.qvg_robust_prune.argtypes = [vp, u64, vp, vp, vp, u32, C.c_float, vp, vp]
    L.qvg_strong_bit_rate.argtypes = [vp, vp, u64, u32, i32, C.POINTER(qvg_encoding_diagnostics)]
    for name in EXPORTED_SYMBOLS:
        f = getattr(L, name)
        if name not in ("qvg_last_error", "qvg_abi_version", "qvg_index_destroy"):
            f.restype = C.c_int
    _lib = L
    return L


def last_error() -> str:
    return lib().qvg_last_error().decode(errors="replace")


def ptr(a):
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")
