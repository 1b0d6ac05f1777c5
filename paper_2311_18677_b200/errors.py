"""Exception hierarchy of the hot path, mirroring the reference's
``splitsim.errors`` (reference errors.py:4-31) so callers of the reference
API catch the same types.  The C-ABI status codes (include/swb200.h) map onto
these in ``_abi.check``."""


class SplitsimError(Exception):
    """Base class (reference errors.py:4)."""


class ValidationError(SplitsimError):
    """Input violates a documented precondition (reference errors.py:8)."""


class CapacityError(SplitsimError):
    """Requested batch or memory exceeds machine capacity (errors.py:26)."""


class ConfigurationError(SplitsimError):
    """Inconsistent or incomplete cluster/run configuration (errors.py:30)."""


class NativeError(RuntimeError):
    """A CUDA error reported by libswb200 (no reference counterpart: the
    reference never touches a device)."""
