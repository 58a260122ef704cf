"""Error taxonomy of the reference (kronblur errors.py:11-37), restated for the drop-in.

When the reference package is importable, its own classes are re-used so that callers that
catch ``kronblur.errors.NumericError`` keep working after ``install()``; otherwise the same
hierarchy is defined here.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on whether kronblur is on the path
    from kronblur.errors import (  # type: ignore
        ArgumentError,
        CapacityError,
        FormatError,
        KronblurError,
        NumericError,
    )
except Exception:  # kronblur absent (e.g. on the GPU box)

    class KronblurError(Exception):
        """Base class for all domain errors (errors.py:11)."""

    class ArgumentError(KronblurError):
        """Out-of-range value, wrong shape or inconsistent input (errors.py:15)."""

    class FormatError(KronblurError):
        """Unparseable payload (errors.py:19-30)."""

        def __init__(self, message: str, offset: int | None = None):
            if offset is not None:
                message = f"{message} (byte offset {offset})"
            super().__init__(message)
            self.offset = offset

    class CapacityError(ArgumentError):
        """Dense materialisation above the size guard (errors.py:33)."""

    class NumericError(KronblurError):
        """Non-finite values or failed factorisation (errors.py:37)."""


__all__ = ["KronblurError", "ArgumentError", "FormatError", "CapacityError", "NumericError"]
