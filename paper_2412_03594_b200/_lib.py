"""ctypes binding of libpsa.so (the C ABI in include/psa.h).

This is the only place the package touches the native library. There is no
fallback: if libpsa.so is missing or cannot be loaded, every compute entry
point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpsa.so")

PSA_OK, PSA_INVALID_ARGUMENT, PSA_UNSUPPORTED, PSA_CUDA_ERROR = 0, 1, 2, 3
DTYPE_F32, DTYPE_BF16, DTYPE_F16, DTYPE_F64 = 0, 1, 2, 3
FLAG_PARTIAL_OUT = 1
FLAG_CAUSAL = 2  # include/psa.h PSA_FLAG_CAUSAL (extension: causal prefill chunks)
ABI_VERSION = 3  # include/psa.h PSA_ABI_VERSION (checked at load)


class Problem(C.Structure):
    _fields_ = [
        ("num_groups", C.c_int32), ("num_requests", C.c_int32),
        ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
        ("head_dim", C.c_int32), ("value_dim", C.c_int32),
        ("dtype", C.c_int32), ("flags", C.c_uint32),
        ("scale", C.c_double),
        ("cu_req", C.POINTER(C.c_int64)), ("cu_q", C.POINTER(C.c_int64)),
        ("cu_prefix", C.POINTER(C.c_int64)), ("cu_distinct", C.POINTER(C.c_int64)),
        ("q", C.c_void_p), ("k_prefix", C.c_void_p), ("v_prefix", C.c_void_p),
        ("k_distinct", C.c_void_p), ("v_distinct", C.c_void_p),
        ("out", C.c_void_p), ("lse", C.c_void_p), ("m_out", C.c_void_p), ("l_out", C.c_void_p),
        ("page_size", C.c_int32), ("reserved0", C.c_int32),
        ("prefix_pages", C.c_void_p), ("distinct_pages", C.c_void_p),
        ("prefix_cache_rows", C.c_int64), ("distinct_cache_rows", C.c_int64),
    ]


class PlanOpts(C.Structure):
    _fields_ = [
        ("num_sms", C.c_int32), ("ctas_per_sm", C.c_int32), ("tile_min_rows", C.c_int32),
        ("disable_tiles", C.c_int32), ("min_chunk_keys", C.c_int32),
        ("max_chunk_keys", C.c_int32), ("target_waves", C.c_int32), ("disable_vec_fast", C.c_int32),
        ("kernel_variant", C.c_int32),
    ]


class PlanView(C.Structure):
    _fields_ = [
        ("num_items", C.c_int32), ("num_units", C.c_int32), ("num_contribs", C.c_int32),
        ("item_words", C.c_int32), ("unit_words", C.c_int32), ("num_tile_items", C.c_int32),
        ("workspace_rows", C.c_int64),
        ("items", C.POINTER(C.c_int32)), ("units", C.POINTER(C.c_int32)),
        ("contribs", C.POINTER(C.c_int32)),
    ]


# (name, restype, argtypes) — every symbol include/psa.h declares.
SIGNATURES = [
    ("psa_last_error", C.c_char_p, []),
    ("psa_abi_version", C.c_int32, []),
    ("psa_device_sms", C.c_int, [C.POINTER(C.c_int32)]),
    ("psa_plan_create", C.c_int, [C.POINTER(Problem), C.POINTER(PlanOpts), C.POINTER(C.c_void_p)]),
    ("psa_plan_view_get", C.c_int, [C.c_void_p, C.POINTER(PlanView)]),
    ("psa_plan_workspace_bytes", C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    ("psa_plan_upload", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("psa_plan_destroy", None, [C.c_void_p]),
    ("psa_run", C.c_int, [C.POINTER(Problem), C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("psa_workspace_bytes", C.c_int, [C.POINTER(Problem), C.POINTER(PlanOpts), C.POINTER(C.c_size_t)]),
    ("psa_prefix_shared_attention", C.c_int,
     [C.POINTER(Problem), C.POINTER(PlanOpts), C.c_void_p, C.c_size_t, C.c_void_p]),
    ("psa_workspace_error", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    ("psa_merge", C.c_int, [C.c_int64, C.c_int32, C.c_int32] + [C.c_void_p] * 9 + [C.c_void_p]),
    ("psa_finalize", C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p]),
    ("psa_count_nonfinite", C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    ("psa_debug_set_trace", C.c_int, [C.c_void_p, C.c_int64]),
    ("psa_shard_groups", C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32)]),
    ("psa_group_costs", C.c_int, [C.POINTER(Problem), C.POINTER(C.c_int64)]),
    ("psa_prefix_groups", C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_int64)]),
]

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def _bind(handle):
    for name, res, args in SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    got = handle.psa_abi_version()
    if got != ABI_VERSION:
        raise RuntimeError(f"libpsa.so ABI version {got}, this binding expects {ABI_VERSION}: "
                           "rebuild with `python -m paper_2412_03594_b200.build`")
    return handle


def lib():
    """Load libpsa.so (building it first when the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        alt = os.environ.get("PSA_LIB_PATH")  # diagnostics: A/B another build of the library
        if alt:
            _lib = _bind(C.CDLL(alt))
            return _lib
        if os.environ.get("PSA_NO_BUILD") != "1":
            try:
                from . import build as _build
                _build.build()
            except RuntimeError:
                if not os.path.exists(LIB_PATH):
                    raise
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libpsa.so not found at {LIB_PATH}; run "
                               "`python -m paper_2412_03594_b200.build` (no CPU fallback exists)")
        _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def last_error() -> str:
    msg = lib().psa_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status != PSA_OK:
        raise NativeError(status, (what + ": " if what else "") + last_error())
