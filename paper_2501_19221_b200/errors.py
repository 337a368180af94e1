"""Exception types, mirroring the reference (qubokit/errors.py:4-25).

The product path never imports the reference.  When the solvers are swapped into an
imported reference (``harness.use_in_reference``), the harness translates these into the
reference's own classes so its ``except qubokit.ValidationError`` clauses keep working.
"""

from __future__ import annotations


class QubokitError(Exception):
    """Base class for all toolkit errors."""


class ValidationError(QubokitError, ValueError):
    """Raised when a model, vector, or parameter record is malformed."""


__all__ = ["QubokitError", "ValidationError"]
