"""Callers either side of the path: the reference's bench harness.

``use_in_reference(qubokit)`` swaps this package's solvers into an imported reference at
every place it resolves them -- the package namespace (``__init__.py:47-64``),
``qubokit.solvers``, the bench harness table (``bench.py:196``) and the CLI table
(``cli.py:253``) -- so the reference's own ``run_suite`` / ``solve`` commands run the B200
loop unmodified.  Models and parameter records pass through as-is (duck-typed), and the
returned ``SampleSet`` has the reference's fields (``samples``, ``best``, ``energies()``,
``replica_count``, ``seed``, ``wall_time``).

``optimality_gap`` / ``spectrum`` restate ``bench.py:47-54`` / ``:268-279`` for callers
without the reference; ``time_to_target`` (solvers.py) reads the per-step energy trace.
"""

from __future__ import annotations

import functools
import sys

import numpy as np

from . import solvers
from .errors import QubokitError, ValidationError

_NAMES = ("solve_pa", "solve_sbm", "solve_sa")


def _translating(fn, qubokit):
    """`fn` raising the reference's own exception classes (qubokit/errors.py) instead of
    this package's, so the reference's `except` clauses see what they expect."""
    ref_val = getattr(qubokit, "ValidationError", None)
    ref_base = getattr(qubokit, "QubokitError", None)

    @functools.wraps(fn)
    def call(*a, **kw):
        try:
            return fn(*a, **kw)
        except ValidationError as e:
            if ref_val is None:
                raise
            raise ref_val(str(e)) from e
        except QubokitError as e:
            if ref_base is None:
                raise
            raise ref_base(str(e)) from e

    call._vxq_wrapped = fn
    return call


def use_in_reference(qubokit, restore: bool = False) -> dict:
    """Patch (or, with restore=True, un-patch) the reference's solver lookups.
    Returns {module name: {attr: previous object}} for the patched modules."""
    mods = [qubokit]
    for sub in ("solvers", "bench", "cli"):
        m = sys.modules.get(f"{qubokit.__name__}.{sub}")
        if m is not None:
            mods.append(m)
    saved = {}
    for m in mods:
        prev = {}
        for name in _NAMES:
            if hasattr(m, name):
                prev[name] = getattr(m, name)
                if restore:
                    orig = getattr(m, f"_vxq_orig_{name}", None)
                    if orig is not None:
                        setattr(m, name, orig)
                else:
                    if not hasattr(m, f"_vxq_orig_{name}"):
                        setattr(m, f"_vxq_orig_{name}", prev[name])
                    setattr(m, name, _translating(getattr(solvers, name), qubokit))
        saved[m.__name__] = prev
    return saved


def optimality_gap(e: float, e_ref: float) -> float:
    """(e - e_ref) / |e_ref|; negative means better (bench.py:47-54)."""
    if e_ref == 0:
        raise ValidationError("optimality gap undefined for zero reference energy; "
                              "use an absolute difference explicitly")
    return (e - e_ref) / abs(e_ref)


def spectrum(sampleset, bins: int):
    """Equal-width histogram of sample energies (bench.py:268-279)."""
    energies = np.asarray(sampleset.energies() if hasattr(sampleset, "energies")
                          else sampleset, dtype=np.float64)
    if energies.size == 0:
        raise ValidationError("spectrum needs at least one sample")
    lo, hi = float(energies.min()), float(energies.max())
    if lo == hi:
        return np.array([lo, hi]), np.array([energies.size])
    counts, edges = np.histogram(energies, bins=bins, range=(lo, hi))
    return edges, counts
