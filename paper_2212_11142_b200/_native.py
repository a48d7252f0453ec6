"""ctypes binding of libbx_sm100.so (include/bx_sm100.h).

This is the only module that touches the shared library.  Loading fails loudly: there is no CPU
fallback for any entry point.  Status codes map onto the exception types the reference raises at
the same call sites.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libbx_sm100.so"

BX_OK, BX_ERR_ARG, BX_ERR_CUDA, BX_ERR_NOT_PD, BX_ERR_STATE, BX_ERR_UNSUPPORTED, BX_ERR_NO_TREES = range(7)
BX_REAL, BX_INTEGER, BX_ORDINAL, BX_CATEGORICAL, BX_PERMUTATION = range(5)
BX_KENDALL, BX_SPEARMAN, BX_HAMMING, BX_NAIVE = range(4)
METRIC_CODES = {"kendall": BX_KENDALL, "spearman": BX_SPEARMAN, "hamming": BX_HAMMING, "naive": BX_NAIVE}
KIND_CODES = {"real": BX_REAL, "integer": BX_INTEGER, "ordinal": BX_ORDINAL,
              "categorical": BX_CATEGORICAL, "permutation": BX_PERMUTATION}
BX_MAX_PARAMS = 64
BX_MAX_ROW_WORDS = 64
BX_MAX_K = 32
BX_SCORE_RF_PAIRWISE = 1
BX_SCORE_NO_SUMMARY = 2

EXPORTED = (
    "bx_create", "bx_destroy", "bx_last_error", "bx_abi_version", "bx_device_sm_count",
    "bx_set_space", "bx_set_gp", "bx_set_forest", "bx_clear_forest", "bx_set_evaluated",
    "bx_set_cot", "bx_clear_cot", "bx_set_constraints", "bx_score", "bx_score_host",
    "bx_gp_predict", "bx_rf_predict", "bx_neighbor_slots", "bx_neighbors", "bx_climb", "bx_rf_fit", "bx_cot_contains",
    "bx_constraints_eval", "bx_lml_batched", "bx_pairwise_sq", "bx_last_timing", "bx_probe_fp64", "bx_probe_int8",
    "bx_lml_core", "bx_generate", "bx_score_generated", "bx_gp_kernel", "bx_gp_distance_ksteps", "bx_gp_embedding_dims", "bx_pcg64_permutations", "bx_pcg64_choice", "bx_pcg64_forest_draws", "bx_unique_rows", "bx_lml_core_host", "bx_gp_factor", "bx_set_option", "bx_packed_row_words", "bx_pack_rows", "bx_unpack_rows",
)
BX_SCORE_TIMING = 4
BX_SCORE_TIMING_POSTERIOR = 8
BX_SCORE_PACKED = 16
BX_OPT_LML_NARROW = 1


class ParamDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("word", C.c_int32), ("size", C.c_int32), ("metric", C.c_int32),
                ("coord", C.c_int32), ("rank", C.c_int32), ("feat", C.c_int32), ("is_log", C.c_int32),
                ("lo", C.c_double), ("hi", C.c_double), ("step", C.c_double), ("raw_mx", C.c_double)]


class Cand(C.Structure):
    _fields_ = [("value", C.c_double), ("prob", C.c_double), ("index", C.c_int64),
                ("row", C.c_uint32 * BX_MAX_ROW_WORDS)]


class ScoreSummary(C.Structure):
    _fields_ = [("n_scored", C.c_int64), ("n_finite", C.c_int64), ("k", C.c_int32),
                ("n_top", C.c_int32), ("top", Cand * BX_MAX_K), ("best", Cand),
                ("best_prob", Cand)]


class NativeError(RuntimeError):
    """A libbx_sm100 call failed; `.code` is the bx_status."""

    def __init__(self, code: int, message: str):
        super().__init__(f"bx error {code}: {message}")
        self.code = code


_lib = None

_p = C.c_void_p
_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "bx_create": (_p, [C.c_int]),
    "bx_destroy": (None, [_p]),
    "bx_last_error": (C.c_char_p, [_p]),
    "bx_abi_version": (C.c_int, []),
    "bx_device_sm_count": (C.c_int, [_p]),
    "bx_gp_kernel": (C.c_int, [_p]),
    "bx_gp_distance_ksteps": (C.c_int, [_p]),
    "bx_gp_embedding_dims": (C.c_int, [_p]),
    "bx_pcg64_permutations": (C.c_int, [_p, _p, _p, _i64, _i32, _p]),
    "bx_pcg64_choice": (C.c_int, [_p, _p, _p, _i64, _i32, _i32, _p]),
    "bx_pcg64_forest_draws": (C.c_int, [_p, _i32, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _p]),
    "bx_unique_rows": (_i64, [_p, _i64, _i32, _p]),
    "bx_lml_core_host": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _i32, _f64, _f64, _i32, _p, _p, _p, _p]),
    "bx_gp_factor": (C.c_int, [_p, _p, _i32, _p, _f64, _f64, _p, _p, _p, _p]),
    "bx_set_option": (C.c_int, [_p, _i32, _i32]),
    "bx_packed_row_words": (C.c_int, [_p]),
    "bx_pack_rows": (C.c_int, [_p, _p, _i64, _p]),
    "bx_unpack_rows": (C.c_int, [_p, _p, _i64, _p]),
    "bx_set_space": (C.c_int, [_p, _p, _i32, _i32, _p, _i32, _p, _i32, _i32]),
    "bx_set_gp": (C.c_int, [_p, _p, _i32, _p, _p, _f64, _p, _f64, _f64, _p]),
    "bx_set_forest": (C.c_int, [_p, _p, _p, _p, _p, _p, _i32, _p, _i32, _i32, _f64]),
    "bx_clear_forest": (C.c_int, [_p]),
    "bx_set_evaluated": (C.c_int, [_p, _p, _i32]),
    "bx_set_cot": (C.c_int, [_p, _i32, _p, _p, _p, _p, _i32, _p, _p, _p, _p]),
    "bx_clear_cot": (C.c_int, [_p]),
    "bx_set_constraints": (C.c_int, [_p, _i32, _p, _p, _i32, _p, _i32, _p, _p, _p, _p, _i32]),
    "bx_score": (C.c_int, [_p, _p, _i64, _i64, _f64, _f64, _i32, _i32, _p, _p, _p, _p]),
    "bx_score_host": (C.c_int, [_p, _p, _i64, _i64, _f64, _f64, _i32, _i32, _p, _p]),
    "bx_gp_predict": (C.c_int, [_p, _p, _i64, _p, _p, _p]),
    "bx_rf_predict": (C.c_int, [_p, _p, _i64, _i32, _p, _p]),
    "bx_neighbor_slots": (C.c_int, [_p]),
    "bx_neighbors": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _p]),
    "bx_climb": (C.c_int, [_p, _p, _p, _p, _i32, _i32, _f64, _f64, _i32, _p, _p, _p]),
    "bx_rf_fit": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _i32, _i32, _i32, _i32,
                            _p, _p, _p, _p, _p, _p, _p, _p]),
    "bx_cot_contains": (C.c_int, [_p, _p, _i64, _p, _p]),
    "bx_constraints_eval": (C.c_int, [_p, _p, _i64, _p, _p]),
    "bx_lml_batched": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _i32, _p, _p]),
    "bx_pairwise_sq": (C.c_int, [_p, _p, _i32, _p, _i32, _p, _p]),
    "bx_last_timing": (C.c_int, [_p, _p, _p, _p]),
    "bx_probe_fp64": (C.c_int, [C.c_int, _p, _p]),
    "bx_probe_int8": (C.c_int, [C.c_int, _p, _p]),
    "bx_lml_core": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _i32, _f64, _f64, _i32, _i32, _p, _p, _p, _p]),
    "bx_generate": (C.c_int, [_p, C.c_uint64, _i64, _i64, _i32, _p, _p]),
    "bx_score_generated": (C.c_int, [_p, C.c_uint64, _i64, _i64, _i32, _f64, _f64, _i32, _p, _p]),
}


def lib():
    """The loaded library (raises if it is missing: build it with __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (there is no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(h, code: int):
    if code != BX_OK:
        msg = lib().bx_last_error(h)
        raise NativeError(code, msg.decode() if msg else "")
