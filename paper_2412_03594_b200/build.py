"""Build libpsa.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2412_03594_b200.build [-v]

The shared library is the C-ABI boundary declared in include/psa.h. cudart is
linked statically so the library does not depend on which CUDA runtime the
host process (PyTorch) brought; streams and device pointers are driver
objects and cross that boundary freely.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpsa.so")
# Debug variant: bounded mbarrier waits that trap with a record of the hung wait
# (psa_device.cuh, PSA_BOUNDED_WAIT). Load it with PSA_LIB_PATH=<path of libpsa_debug.so>.
DEBUG_LIB = os.path.join(PKG, "libpsa_debug.so")
# Trace variant: per-block clock64 event hooks (PSA_TRACE_EVENTS; tools/trace_report.py --tile2).
TRACE_LIB = os.path.join(PKG, "libpsa_trace.so")
SOURCES = ["psa_kernel.cu", "psa_api.cpp", "psa_plan.cpp", "psa_prefix.cpp"]
HEADERS = ["psa_kernel.h", "psa_plan.h", "psa_device.cuh", "psa_tile.cuh", "psa_vec.cuh",
           "psa_dec.cuh", "psa_tile2.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: libpsa.so cannot be built")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "psa.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.exists(p) and os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False,
          trace: bool = False) -> str:
    lib = DEBUG_LIB if debug else TRACE_LIB if trace else LIB
    if not force and not _stale(lib):
        return lib
    cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
           "-cudart", "static", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"),
           *(["-DPSA_TRACE_EVENTS"] if trace or os.environ.get("PSA_TRACE_EVENTS") == "1" else []),
           *(["-DPSA_BOUNDED_WAIT"] if debug else []),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", lib + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, debug="--debug" in sys.argv,
                trace="--trace" in sys.argv))
