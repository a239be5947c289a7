"""The C-ABI library loads (no GPU needed) and exports every symbol include/psa.h declares."""

import ctypes
import pytest
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
    assert lib.psa_abi_version() == 3 == L.ABI_VERSION  # checked by _lib.lib() at load
    # a NULL problem is rejected with INVALID_ARGUMENT and a message, no CUDA needed
    h = ctypes.c_void_p()
    st = lib.psa_plan_create(None, None, ctypes.byref(h))
    assert st == L.PSA_INVALID_ARGUMENT
    assert "NULL" in L.last_error()


def test_struct_sizes_match_header_layout(tmp_path):
    # psa_problem: 8 int32 + double + 4 offset ptrs + 9 buffer ptrs = 32 + 8 + 104 on LP64
    assert ctypes.sizeof(L.Problem) == 184
    assert ctypes.sizeof(L.PlanOpts) == 36
    assert ctypes.sizeof(L.PlanView) == 56
    # cross-check against the C compiler's view of include/psa.h
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "psa.h"\nint main(void){printf("%zu %zu %zu", '
                   'sizeof(psa_problem), sizeof(psa_plan_opts), sizeof(psa_plan_view));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run([cc, "-I", inc, str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(L.Problem), ctypes.sizeof(L.PlanOpts), ctypes.sizeof(L.PlanView)]
