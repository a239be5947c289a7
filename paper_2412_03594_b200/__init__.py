"""B200-native prefix-shared attention (BatchLLM hot path, arxiv 2412.03594).

Public surface:
  attention  — drop-in for ``prefixbatch.attention`` (same names/semantics).
  packed     — packed multi-group multi-head op (one persistent launch per batch).
  workloads  — synthetic batches for BASELINE.json configs C1..C5.
  errors     — PrefixBatchError / ValidationError (mirror of the reference's errors.py).
The compute lives in libpsa.so (C ABI: include/psa.h); there is no CPU fallback.
"""

from .errors import PrefixBatchError, ValidationError  # noqa: F401

__version__ = "0.1.0"
