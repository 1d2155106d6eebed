"""ctypes binding of libhcomp.so (include/hcomp.h).

The CUDA library is the only compute path of this package: if it is missing
or no GPU is present, operations raise instead of falling back to any CPU
code.  The library is built in-tree by `python -m paper_2408_17063_b200.build`
(or `__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .params import BackendMismatch, LevelExhausted, MissingRotationKey

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HCOMP_LIB") or os.path.join(_HERE, "libhcomp.so")  # max_level <= 3
LIB5_PATH = os.environ.get("HCOMP_LIB5") or os.path.join(_HERE, "libhcomp_l4.so")  # max_level 4
LIBDEEP_PATH = os.environ.get("HCOMP_LIBDEEP") or os.path.join(_HERE, "libhcomp_deep.so")  # max_level 5..22

HC_OK = 0
HC_ERR_ARG = 1
HC_ERR_LEVEL = 2
HC_ERR_KEY = 3
HC_ERR_MISMATCH = 4
HC_ERR_CUDA = 5
HC_ERR_STATE = 6


class HcompError(RuntimeError):
    """CUDA / state failure inside libhcomp (no reference analogue)."""


_libs: dict = {}  # path -> CDLL
_last = None  # the library of the most recent lib() call (its hc_last_error)

# (name, restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_SIGS = [
    ("hc_last_error", ctypes.c_char_p, []),
    ("hc_ctx_create", _I, [_I, _I, _P, _U64, _I, _I, ctypes.POINTER(_P)]),
    ("hc_ctx_destroy", None, [_P]),
    ("hc_ctx_digits", _I, [_P, _P]),
    ("hc_load_ksk", _I, [_P, _U32, _P]),
    ("hc_clear_keys", _I, [_P]),
    ("hc_load_ksk_slice", _I, [_P, _U32, _P, _I, _I]),
    ("hc_plan", _I, [_P, _I64, _I, _I]),
    ("hc_plan_masked", _I, [_P, ctypes.c_int64, _I, _I, _P]),
    ("hc_plan_range", _I, [_P, _I64, _I, _I, _I64, _I64]),
    ("hc_plan_shared", _I, [_P, _P, _I]),
    ("hc_plan_info", _I, [_P, _P]),
    ("hc_comp", _I, [_P, _P, _P, _I, _P]),
    ("hc_comp_packed", _I, [_P, _P, _I64, _P]),
    ("hc_comp_mixed", _I, [_P, _P, _I, _P, _I, _I, _P]),
    ("hc_answer_db", _I, [_P, _I, _P]),
    ("hc_answer", _I, [_P, _P, _I, _I, _P]),
    ("hc_mixed_launch", _I, [_P, _P]),
    ("hc_plain_row", _I, []),
    ("hc_comp_async", _I, [_P, _P, _P, _I, _P, _P]),
    ("hc_comp_upload_async", _I, [_P, _P, _P, _I, _P]),
    ("hc_comp_set_inputs", _I, [_P, _P, _P, _I]),
    ("hc_comp_set_inputs_range", _I, [_P, _P, _P, _I, _I, _P]),
    ("hc_comp_set_inputs_device", _I, [_P, _P, _P, _I, _P]),
    ("hc_comp_launch", _I, [_P, _P]),
    ("hc_comp_get_output", _I, [_P, _P]),
    ("hc_comp_get_output_async", _I, [_P, _P, _P]),
    ("hc_partial_words", _I64, [_P]),
    ("hc_comp_partial", _I, [_P, _I64, _I64, _P, _P]),
    ("hc_comp_finish", _I, [_P, _P, _P]),
    ("hc_ntt", _I, [_P, _P, _I, _P, _I]),
    ("hc_pointwise", _I, [_P, _P, _P, _P, _I, _P, _I]),
    ("hc_mul_plain", _I, [_P, _P, _I, _P, _P]),
    ("hc_decrypt", _I, [_P, _P, _I, _P, _P]),
    ("hc_rotate", _I, [_P, _P, _I, _U32, _P]),
    ("hc_comp_profile", _I, [_P, _P, _I, _P, _P, _P]),
    ("hc_comp_profile_ex", _I, [_P, _P, _I, _P, _P, _P, _P]),
    ("hc_bf_peak", _I, [_P, ctypes.POINTER(ctypes.c_double)]),
    ("hc_bench_xform", _I, [_P, _I, _I, _I, ctypes.POINTER(ctypes.c_double)]),
    ("hc_imad_peak", _I, [_P, _P]),
    ("hc_set_cluster_threshold", _I, [_I]),
    ("hc_set_lane_blocks", _I, [_I]),
    ("hc_set_ksfused", _I, [_I]),
    ("hc_set_vt2_jobs", _I, [_I]),
    ("hc_max_active_clusters", _I, [_P, _P]),
    ("hc_trace_reset", _I, []),
    ("hc_trace_read", _I, [_P]),
    ("hc_trace_read_tail", _I, [_P]),
    ("hc_rng_create", _I, [_P, _I, _P]),
    ("hc_rng_destroy", None, [_P]),
    ("hc_rng_getrandbits", _I, [_P, _I, _P]),
    ("hc_rng_ternary", _I, [_P, _I, _P]),
    ("hc_rng_cbd", _I, [_P, _I, _I, _P]),
    ("hc_rng_uniform", _I, [_P, _I, _P, _I, _I, _P, _I, _P]),
    ("hc_galois_tables", _I, [_I, _U32, _P, _P]),
    ("hc_prim_root_2n", _U64, [_U64, _I]),
]
EXPORTS = [s[0] for s in _SIGS]


def lib(max_level: int = 3):
    """Load the CUDA library for chains up to max_level + 1 primes (raises if
    it has not been built).  Both builds export the same C ABI."""
    global _last
    path = LIB_PATH if max_level <= 3 else LIB5_PATH if max_level == 4 else LIBDEEP_PATH
    L = _libs.get(path)
    if L is None:
        if not os.path.exists(path):
            raise HcompError(
                f"{path} is missing: build it with `python -m paper_2408_17063_b200.build` "
                "(there is no CPU fallback for Comp)"
            )
        L = ctypes.CDLL(path)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _libs[path] = L
    _last = L
    return L


def ptr(a: np.ndarray):
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(ctypes.c_void_p)


def check(rc: int) -> None:
    """Map libhcomp status codes onto the reference's exceptions."""
    if rc == HC_OK:
        return
    msg = (_last or lib()).hc_last_error().decode(errors="replace")
    if rc == HC_ERR_ARG:
        raise ValueError(msg)
    if rc == HC_ERR_LEVEL:
        raise LevelExhausted(msg)
    if rc == HC_ERR_KEY:
        raise MissingRotationKey(msg)
    if rc == HC_ERR_MISMATCH:
        raise BackendMismatch(msg)
    raise HcompError(msg)
