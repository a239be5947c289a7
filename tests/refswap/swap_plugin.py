"""pytest plugin: INTEGRATION.md §1 module swap, applied before the reference's own
test modules are collected. ``prefixbatch.attention`` becomes the GPU-backed drop-in
``paper_2412_03594_b200.attention``; the drop-in's ValidationError is re-based on the
reference's so ``pytest.raises(prefixbatch.ValidationError)`` catches ours."""

import sys

import prefixbatch
import prefixbatch.errors as _ref_errors

from paper_2412_03594_b200 import attention as _ours
from paper_2412_03594_b200 import errors as _e

_e.ValidationError.__bases__ = (_ref_errors.ValidationError,)
sys.modules["prefixbatch.attention"] = _ours
prefixbatch.attention = _ours


def pytest_sessionstart(session):
    import prefixbatch.attention as a
    assert a is _ours, "module swap not in effect"
    print(f"SWAPPED prefixbatch.attention -> {a.__name__}")


def pytest_sessionfinish(session, exitstatus):
    from paper_2412_03594_b200 import _lib
    print(f"NATIVE {_lib.LIB_PATH} loaded={_lib._lib is not None}")
