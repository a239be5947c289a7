"""The C-ABI library loads (no GPU needed) and exports every symbol include/psa.h declares."""

import ctypes
import os
import re

from paper_2412_03594_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "psa.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(psa_[a-z_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    names = declared_symbols()
    for must in ("psa_plan_create", "psa_run", "psa_prefix_shared_attention", "psa_merge",
                 "psa_finalize", "psa_count_nonfinite", "psa_shard_groups", "psa_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in L.SIGNATURES}
    assert set(declared_symbols()) <= bound


def test_abi_version_and_error_channel():
    lib = L.lib()
    assert lib.psa_abi_version() == 1
    # a NULL problem is rejected with INVALID_ARGUMENT and a message, no CUDA needed
    h = ctypes.c_void_p()
    st = lib.psa_plan_create(None, None, ctypes.byref(h))
    assert st == L.PSA_INVALID_ARGUMENT
    assert "NULL" in L.last_error()


def test_struct_sizes_match_header_layout():
    # psa_problem: 8 int32 + double + 4 offset ptrs + 9 buffer ptrs = 32 + 8 + 104 on LP64
    # (cross-checked against gcc's sizeof of include/psa.h)
    assert ctypes.sizeof(L.Problem) == 144
    assert ctypes.sizeof(L.PlanOpts) == 32
    assert ctypes.sizeof(L.PlanView) == 56
