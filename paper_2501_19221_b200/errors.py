"""Exception types, mirroring the reference (qubokit/errors.py:4-25).

If the reference package is importable, its classes are reused so that
``except qubokit.ValidationError`` keeps working after the swap.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from qubokit.errors import QubokitError, ValidationError  # type: ignore
except Exception:  # noqa: BLE001
    class QubokitError(Exception):
        """Base class for all toolkit errors."""

    class ValidationError(QubokitError, ValueError):
        """Raised when a model, vector, or parameter record is malformed."""

__all__ = ["QubokitError", "ValidationError"]
