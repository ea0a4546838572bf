"""ctypes binding of the C ABI in include/bandmatch_gpu.h (libbmg.so, built in-tree).

The product has no CPU fallback: if the shared library is missing or no CUDA
device is present, the entry points raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["BMG_LIBBMG"]) if os.environ.get("BMG_LIBBMG") else PKG / "libbmg.so"
DIM = 128

STATUS_NAMES = {
    0: "Ok", 1: "InvalidArgument", 2: "HashMismatch", 3: "CapacityExceeded",
    4: "NotResident", 5: "CudaError", 6: "OutOfMemory", 7: "Unsupported", 8: "InvalidScene",
    9: "FormatError", 10: "TruncatedFile", 11: "TooFewDescriptors",
}


class BandmatchError(RuntimeError):
    """Mirror of bandmatch::Error (common.hpp:13-26): stable ``code`` + message."""

    def __init__(self, code: str, message: str):
        super().__init__(f"{code}: {message}")
        self.code = code


class HashParamsC(C.Structure):
    _fields_ = [("tables", C.c_int32), ("coarse_bits", C.c_int32), ("fine_bits", C.c_int32)]


class MatchParamsC(C.Structure):
    _fields_ = [("k_nearest", C.c_int32), ("ratio", C.c_double)]


class ConfigC(C.Structure):
    _fields_ = [("device", C.c_int32), ("hash", HashParamsC), ("coarse_planes", C.c_void_p),
                ("fine_planes", C.c_void_p), ("function_seed", C.c_uint64),
                ("capacity_units", C.c_uint64)]


class CodeSetC(C.Structure):
    _fields_ = [("image_id", C.c_uint64), ("function_seed", C.c_uint64), ("params", HashParamsC),
                ("count", C.c_uint64), ("coarse", C.c_void_p), ("fine", C.c_void_p)]


class FeatureViewC(C.Structure):
    _fields_ = [("image_id", C.c_uint64), ("descriptors", C.c_void_p), ("count", C.c_uint64)]


class FeatureFileC(C.Structure):
    _fields_ = [("image_id", C.c_uint64), ("path", C.c_char_p), ("count", C.c_uint64)]


class ArenaStatsC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("capacity", "occupancy", "peak_occupancy", "uploads",
                                          "evictions", "units_uploaded", "resident_count")]


class PlanC(C.Structure):
    _fields_ = [("n_iterations", C.c_uint64), ("rows_per_iteration", C.c_void_p),
                ("n_rows", C.c_uint64), ("row_needed_offsets", C.c_void_p),
                ("needed_ids", C.c_void_p), ("row_pair_offsets", C.c_void_p),
                ("pairs", C.c_void_p), ("row_evict_offsets", C.c_void_p),
                ("evict_ids", C.c_void_p)]


PAIR_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_int32), C.c_uint64)
UPLOAD_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64)
EVICT_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64)


class ExecOptionsC(C.Structure):
    _fields_ = [("match", MatchParamsC), ("on_pair", PAIR_CB), ("on_pair_user", C.c_void_p),
                ("on_upload", UPLOAD_HOOK), ("on_evict", EVICT_HOOK), ("hook_user", C.c_void_p),
                ("flags", C.c_uint32)]

EXEC_RETAIN = 1
EXEC_MEAN_CHAIN = 2
EXEC_SERIAL = 4
EXEC_REPROJECT = 8


EXPORTED = [
    "bmg_status_name", "bmg_last_error", "bmg_abi_version", "bmg_seed_for",
    "bmg_make_hash_functions", "bmg_create", "bmg_destroy", "bmg_synchronize", "bmg_upload",
    "bmg_evict", "bmg_is_resident", "bmg_arena_stats_get", "bmg_row", "bmg_row_mean", "bmg_codes",
    "bmg_match", "bmg_compute_codes", "bmg_match_pair", "bmg_execute_plan",
    "bmg_result_pair_count", "bmg_result_match_count", "bmg_result_copy", "bmg_result_metrics",
    "bmg_result_iteration_count", "bmg_result_iteration", "bmg_result_free", "bmg_launch_count",
    "bmg_set_profiling", "bmg_kernel_time", "bmg_fixup_counts", "bmg_exact_walk_count", "bmg_synthetic_counts",
    "bmg_generate_synthetic", "bmg_result_device_ms", "bmg_row_mean_info", "bmg_result_view",
    "bmg_result_write_matches", "bmg_read_features_header", "bmg_read_features",
    "bmg_write_matches_binary", "bmg_generate_synthetic_subset", "bmg_set_test_flags",
    "bmg_result_row_timing", "bmg_execute_plan_files", "bmg_sao_filter",
    "bmg_delaunay_knn", "bmg_encode_vlad", "bmg_train_codebook",
]

_lib = None


def load(path: Path = LIB_PATH):
    """Load libbmg.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not path.exists():
        raise BandmatchError("Unsupported", f"{path} is missing: run __graft_entry__.build() "
                             "(the B200 matcher has no CPU fallback)")
    L = C.CDLL(str(path))
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int32
    sig = {
        "bmg_status_name": (C.c_char_p, [C.c_int]),
        "bmg_last_error": (C.c_char_p, []),
        "bmg_abi_version": (C.c_int, []),
        "bmg_seed_for": (u64, [u64, C.c_char_p]),
        "bmg_make_hash_functions": (C.c_int, [u64, C.POINTER(HashParamsC), vp, vp]),
        "bmg_create": (C.c_int, [C.POINTER(ConfigC), C.POINTER(vp)]),
        "bmg_destroy": (C.c_int, [vp]),
        "bmg_synchronize": (C.c_int, [vp]),
        "bmg_upload": (C.c_int, [vp, u64, vp, u64]),
        "bmg_evict": (C.c_int, [vp, u64]),
        "bmg_is_resident": (C.c_int, [vp, u64]),
        "bmg_arena_stats_get": (C.c_int, [vp, C.POINTER(ArenaStatsC)]),
        "bmg_row": (C.c_int, [vp, vp, u64, vp]),
        "bmg_row_mean": (C.c_int, [vp, vp]),
        "bmg_codes": (C.c_int, [vp, u64, vp, vp]),
        "bmg_match": (C.c_int, [vp, vp, vp, u64, C.POINTER(MatchParamsC), vp, vp, u64]),
        "bmg_compute_codes": (C.c_int, [vp, vp, u64, vp, vp, vp]),
        "bmg_match_pair": (C.c_int, [vp, vp, C.POINTER(CodeSetC), vp, C.POINTER(CodeSetC),
                                     C.POINTER(MatchParamsC), vp, C.POINTER(u64)]),
        "bmg_execute_plan": (C.c_int, [vp, C.POINTER(PlanC), vp, u64, C.POINTER(ExecOptionsC),
                                       C.POINTER(vp)]),
        "bmg_result_pair_count": (u64, [vp]),
        "bmg_result_match_count": (u64, [vp]),
        "bmg_result_copy": (C.c_int, [vp, vp, vp, vp]),
        "bmg_result_view": (C.c_int, [vp, C.POINTER(C.POINTER(u64)), C.POINTER(C.POINTER(u64)),
                                      C.POINTER(C.POINTER(i32))]),
        "bmg_result_metrics": (C.c_int, [vp, vp, C.POINTER(C.c_double)]),
        "bmg_result_iteration_count": (u64, [vp]),
        "bmg_result_iteration": (C.c_int, [vp, u64, vp]),
        "bmg_result_free": (None, [vp]),
        "bmg_result_write_matches": (C.c_int, [vp, C.c_char_p]),
        "bmg_read_features_header": (C.c_int, [C.c_char_p, C.POINTER(u64), C.POINTER(u64)]),
        "bmg_read_features": (C.c_int, [C.c_char_p, u64, vp, vp, C.c_int, C.POINTER(u64), C.POINTER(u64)]),
        "bmg_write_matches_binary": (C.c_int, [C.c_char_p, u64, vp, vp, vp, vp]),
        "bmg_result_device_ms": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "bmg_launch_count": (u64, [vp]),
        "bmg_set_profiling": (C.c_int, [vp, C.c_int]),
        "bmg_kernel_time": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_double), C.POINTER(u64)]),
        "bmg_fixup_counts": (C.c_int, [vp, C.POINTER(u64), C.POINTER(u64)]),
        "bmg_exact_walk_count": (C.c_int, [vp, C.POINTER(u64)]),
        "bmg_row_mean_info": (C.c_int, [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_int)]),
        "bmg_set_test_flags": (C.c_int, [vp, C.c_uint32]),
        "bmg_result_row_timing": (C.c_int, [vp, u64, vp]),
        "bmg_execute_plan_files": (C.c_int, [vp, C.POINTER(PlanC), vp, u64, C.POINTER(ExecOptionsC),
                                             C.POINTER(vp)]),
        "bmg_sao_filter": (C.c_int, [vp, u64, vp, u64, vp, u64, C.c_int, C.c_double, vp, vp,
                                     C.POINTER(C.c_uint32)]),
        "bmg_delaunay_knn": (C.c_int, [vp, u64, C.c_int, vp, C.POINTER(C.c_int)]),
        "bmg_encode_vlad": (C.c_int, [vp, vp, C.c_int, vp, u64, vp, vp]),
        "bmg_train_codebook": (C.c_int, [vp, vp, u64, C.c_int, C.c_int, u64, vp, vp, C.POINTER(C.c_int)]),
        "bmg_synthetic_counts": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, vp]),
        "bmg_generate_synthetic": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                             u64, vp, vp]),
        "bmg_generate_synthetic_subset": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double,
                                                    C.c_double, u64, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        L = load()
        raise BandmatchError(STATUS_NAMES.get(rc, "Unknown"), L.bmg_last_error().decode())


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data
