import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


import contextlib
import os as _os


@contextlib.contextmanager
def no_tail_shift():
    """Packed launches with full forward boxes for partial last blocks (PSA_DEBUG bit
    1024): the packed kernel then does exactly the paged kernel's arithmetic, so the
    two can be compared bit for bit (the default back-shifted boxes change only the
    column positions of a partial block's keys, i.e. rounding)."""
    old = _os.environ.get("PSA_DEBUG")
    _os.environ["PSA_DEBUG"] = str(int(old or 0) | 1024)
    try:
        yield
    finally:
        if old is None:
            _os.environ.pop("PSA_DEBUG", None)
        else:
            _os.environ["PSA_DEBUG"] = old
