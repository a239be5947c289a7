"""Exception types of the drop-in boundary.

Mirror of the reference's ``pkg/src/prefixbatch/errors.py:4-19``: every
hot-path rejection raises ``ValidationError``, which subclasses
``PrefixBatchError`` (not ``ValueError``). Native status codes map as
PSA_INVALID_ARGUMENT / PSA_UNSUPPORTED -> ValidationError and
PSA_CUDA_ERROR -> RuntimeError (include/psa.h).
"""


class PrefixBatchError(Exception):
    """Base class for all errors raised by this package (errors.py:4-5)."""


class ValidationError(PrefixBatchError):
    """Input violated a documented invariant (errors.py:18-19)."""
