"""Error hierarchy of the B200 conv path.

Every failure raised by this package derives from ``CuclgenError``, the base
class the reference uses for all of its errors (cuclgen/errors.py:1-2), so a
caller that catches the reference's base class keeps working.  The C ABI's
status codes (include/b2conv.h) map onto the subclasses below.
"""

from __future__ import annotations


class CuclgenError(Exception):
    """Base class for all errors raised by this package (cuclgen/errors.py:1-2)."""


class Inapplicable(CuclgenError):
    """A variant cannot run an op (cuclgen/variants.py:31; status B2C_INAPPLICABLE)."""


class ShapeMismatch(CuclgenError):
    """Operand shapes disagree with the op description (cuclgen/oracle.py:19; status B2C_BAD_ARGS)."""


class DeviceError(CuclgenError):
    """CUDA runtime or launch failure (the InterpError family, cuclgen/backend.py:61-82; status B2C_CUDA_ERROR)."""


class Unsupported(CuclgenError):
    """Feature/precision not built into libb2conv (status B2C_UNSUPPORTED)."""


class ExtensionMissing(CuclgenError):
    """libb2conv.so is not built or cannot be loaded: the product path has no CPU fallback."""
