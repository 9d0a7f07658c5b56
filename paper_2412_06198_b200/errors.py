"""Exception hierarchy of the drop-in, same names and bases as the reference.

Reference: core.py:32-45 (SparseAttnError, DimensionError, NonFiniteError,
EmptyRowError), patterns.py:55-56 (PatternParamError), search.py:47-48
(SearchError), runtime.py:35-36 (CacheOverflowError).  The C ABI returns the
matching status code (include/sparseattn_b200.h) and ``_lib.check`` raises the
class below.
"""


class SparseAttnError(Exception):
    """Base class for all errors raised by this library."""


class DimensionError(SparseAttnError):
    """Array shapes disagree with the documented contract."""


class NonFiniteError(SparseAttnError):
    """An input tensor contains NaN or Inf."""


class EmptyRowError(SparseAttnError):
    """A softmax row has no included positions."""


class PatternParamError(SparseAttnError):
    """A sparsity pattern or index parameter is out of its legal range."""


class SearchError(SparseAttnError):
    """Search configuration or preconditions are invalid."""


class CacheOverflowError(SparseAttnError):
    """Appending would exceed the configured maximum context."""
