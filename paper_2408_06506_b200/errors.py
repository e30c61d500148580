"""Exception types of the drop-in boundary.

The reference raises classes from ``gelsim.errors`` (errors.py:4-70).  When
the reference package is importable those exact classes are re-exported, so a
caller's ``except gelsim.errors.LutResolutionMismatch`` keeps working after
``paper_2408_06506_b200.patch()``; otherwise same-named local classes with
the same hierarchy are defined.
"""
from __future__ import annotations

try:  # pragma: no cover - depends on whether gelsim is installed
    from gelsim.errors import (  # type: ignore
        DimensionMismatch,
        GelsimError,
        InvalidQuery,
        LutResolutionMismatch,
        ResolutionTooFine,
    )
except Exception:  # noqa: BLE001
    class GelsimError(Exception):
        """Base class for all library errors (errors.py:4-5)."""

    class InvalidQuery(GelsimError):
        """SDF query result used outside its valid region (errors.py:16-17)."""

    class DimensionMismatch(GelsimError):
        """Array shapes of paired inputs disagree (errors.py:37-38)."""

    class LutResolutionMismatch(GelsimError):
        """Look-up table was calibrated for a different image size (errors.py:41-42)."""

    class ResolutionTooFine(GelsimError):
        """Requested tactile grid is finer than the surface mesh resolves (errors.py:33-34)."""

__all__ = ["GelsimError", "InvalidQuery", "DimensionMismatch", "LutResolutionMismatch", "ResolutionTooFine"]
