"""Data in/out of the hot path: Ising/QUBO models and spin helpers.

Mirrors the parts of the reference's ``qubokit/model.py`` the dynamics loop
touches (model.py:36-38, 65-67, 81-200): the frozen canonical COO arrays
(``rows < cols`` sorted unique, ``values``, ``h``, ``offset``), ``sign_pm`` and
the spin/bit maps.  Energies are evaluated on the GPU as correctly rounded
exact sums (``vxq_energies``); there is no CPU evaluation path.

Any object with ``n, h, rows, cols, values, offset`` attributes (for example
the reference's own ``qubokit.IsingModel``) is accepted by the solvers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .errors import ValidationError


def sign_pm(x) -> np.ndarray:
    """Sign with sign(0) = +1 as int8 spins (model.py:36-38)."""
    return np.where(np.asarray(x) >= 0, 1, -1).astype(np.int8)


def as_spins(values, n: int | None = None) -> np.ndarray:
    v = np.asarray(values)
    if v.ndim != 1:
        raise ValidationError(f"spin vector must be 1-d, got shape {v.shape}")
    if not np.all(np.abs(v) == 1):
        raise ValidationError("spin vector entries must be -1 or +1")
    if n is not None and v.shape[0] != n:
        raise ValidationError(f"spin vector has length {v.shape[0]}, expected {n}")
    return v.astype(np.int8)


def as_bits(values, n: int | None = None) -> np.ndarray:
    v = np.asarray(values)
    if v.ndim != 1:
        raise ValidationError(f"binary vector must be 1-d, got shape {v.shape}")
    if not np.all((v == 0) | (v == 1)):
        raise ValidationError("binary vector entries must be 0 or 1")
    if n is not None and v.shape[0] != n:
        raise ValidationError(f"binary vector has length {v.shape[0]}, expected {n}")
    return v.astype(np.int8)


def spins_to_bits(s) -> np.ndarray:
    """x = (1 + s) / 2 (model.py:65-67)."""
    return ((1 + as_spins(s)) // 2).astype(np.int8)


def bits_to_spins(x) -> np.ndarray:
    return (2 * as_bits(x) - 1).astype(np.int8)


def _freeze(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    a.setflags(write=False)
    return a


def canonical_pairs(rows, cols, vals, n: int, allow_diagonal: bool):
    """Vectorised ``_canonical_pairs`` (model.py:81-104): normalise i<=j, sum duplicates
    in input order, sort by (i, j).  Duplicate sums are accumulated sequentially in input
    order exactly like the reference's dict accumulation."""
    r = np.asarray(rows, dtype=np.int64).ravel()
    c = np.asarray(cols, dtype=np.int64).ravel()
    v = np.asarray(vals, dtype=np.float64).ravel()
    if not (r.shape == c.shape == v.shape):
        raise ValidationError("rows, cols and values must have the same length")
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    if lo.size and (lo.min() < 0 or hi.max() >= n):
        bad = int(np.argmax((lo < 0) | (hi >= n)))
        raise ValidationError(f"term index pair ({lo[bad]}, {hi[bad]}) out of range for n={n}")
    if not allow_diagonal and np.any(lo == hi):
        i = int(lo[np.argmax(lo == hi)])
        raise ValidationError(f"diagonal coupling ({i}, {i}) not allowed; use the linear field")
    if not np.all(np.isfinite(v)):
        k = int(np.argmax(~np.isfinite(v)))
        raise ValidationError(f"non-finite coefficient for pair ({lo[k]}, {hi[k]})")
    key = lo * n + hi
    order = np.argsort(key, kind="stable")
    key_s = key[order]
    uniq, start = np.unique(key_s, return_index=True)
    if uniq.size == key_s.size:
        out_v = v[order] + 0.0  # dict accumulation starts at 0.0 (-0.0 -> +0.0)
    else:  # sequential per-key accumulation in input order
        out_v = np.zeros(uniq.size)
        grp = np.searchsorted(uniq, key_s)
        np.add.at(out_v, grp, v[order])
    return (uniq // n).astype(np.int64), (uniq % n).astype(np.int64), out_v.astype(np.float64)


@dataclass(frozen=True, eq=False)
class IsingModel:
    """Sparse symmetric Ising model: couplings on i<j pairs, fields, offset (model.py:113)."""

    n: int
    h: np.ndarray
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    offset: float = 0.0

    @classmethod
    def from_terms(cls, n: int, h=None, couplings: Iterable[tuple[int, int, float]] = (),
                   offset: float = 0.0) -> "IsingModel":
        if n < 1:
            raise ValidationError("model needs at least one variable")
        hv = np.zeros(n, dtype=np.float64) if h is None else np.asarray(h, dtype=np.float64)
        if hv.shape != (n,):
            raise ValidationError(f"field vector has shape {hv.shape}, expected ({n},)")
        if not np.all(np.isfinite(hv)):
            raise ValidationError("field vector must be finite")
        if not math.isfinite(offset):
            raise ValidationError("offset must be finite")
        terms = list(couplings)
        if terms:
            arr = np.array([(t[0], t[1]) for t in terms], dtype=np.int64)
            vals = np.array([float(t[2]) for t in terms], dtype=np.float64)
            rows, cols, vals = canonical_pairs(arr[:, 0], arr[:, 1], vals, n, False)
        else:
            rows = cols = np.zeros(0, dtype=np.int64)
            vals = np.zeros(0)
        return cls(n=n, h=hv, rows=rows, cols=cols, values=vals, offset=float(offset))

    @classmethod
    def from_arrays(cls, n: int, rows, cols, values, h=None, offset: float = 0.0,
                    canonical: bool = False) -> "IsingModel":
        """Vectorised constructor; ``canonical=True`` skips re-canonicalisation."""
        hv = np.zeros(n) if h is None else np.asarray(h, dtype=np.float64)
        if not canonical:
            rows, cols, values = canonical_pairs(rows, cols, values, n, False)
        return cls(n=n, h=hv, rows=rows, cols=cols, values=values, offset=float(offset))

    def __post_init__(self):
        object.__setattr__(self, "h", _freeze(np.asarray(self.h, dtype=np.float64)))
        object.__setattr__(self, "rows", _freeze(np.asarray(self.rows, dtype=np.int64)))
        object.__setattr__(self, "cols", _freeze(np.asarray(self.cols, dtype=np.int64)))
        object.__setattr__(self, "values", _freeze(np.asarray(self.values, dtype=np.float64)))

    @property
    def num_couplings(self) -> int:
        return int(self.values.shape[0])

    def couplings(self) -> list[tuple[int, int, float]]:
        return [(int(i), int(j), float(v)) for i, j, v in zip(self.rows, self.cols, self.values)]

    def energy(self, s) -> float:
        """Exact energy of one spin state (GPU, correctly rounded)."""
        s = as_spins(s, self.n)
        return float(self.energies(s[None, :])[0])

    def energies(self, states: np.ndarray) -> np.ndarray:
        """Exact batch energies for a (replicas, n) spin array (GPU, vxq_energies)."""
        from .device import energies as _energies
        return _energies(self, states)

    def coupling_matrix(self) -> np.ndarray:
        """Dense symmetric coupling matrix with zero diagonal (host view, model.py:174-176)."""
        A = np.zeros((self.n, self.n), dtype=np.float64)
        A[self.rows, self.cols] = self.values
        A[self.cols, self.rows] = self.values
        A.setflags(write=False)
        return A

    @property
    def field_scale(self) -> float:
        """max_i (|h_i| + sum_j |J_ij|), computed on the GPU (vxq_problem_lambda0)."""
        from .device import lambda0
        return lambda0(self)


@dataclass(frozen=True, eq=False)
class QuboModel:
    """Sparse QUBO: terms on i<=j pairs (model.py:203)."""

    n: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    offset: float = 0.0

    @classmethod
    def from_terms(cls, n: int, terms: Iterable[tuple[int, int, float]] = (),
                   offset: float = 0.0) -> "QuboModel":
        if n < 1:
            raise ValidationError("model needs at least one variable")
        if not math.isfinite(offset):
            raise ValidationError("offset must be finite")
        terms = list(terms)
        if terms:
            arr = np.array([(t[0], t[1]) for t in terms], dtype=np.int64)
            vals = np.array([float(t[2]) for t in terms], dtype=np.float64)
            rows, cols, vals = canonical_pairs(arr[:, 0], arr[:, 1], vals, n, True)
        else:
            rows = cols = np.zeros(0, dtype=np.int64)
            vals = np.zeros(0)
        return cls(n=n, rows=rows, cols=cols, values=vals, offset=float(offset))

    @classmethod
    def from_arrays(cls, n: int, rows, cols, values, offset: float = 0.0) -> "QuboModel":
        rows, cols, values = canonical_pairs(rows, cols, values, n, True)
        return cls(n=n, rows=rows, cols=cols, values=values, offset=float(offset))

    def __post_init__(self):
        object.__setattr__(self, "rows", _freeze(np.asarray(self.rows, dtype=np.int64)))
        object.__setattr__(self, "cols", _freeze(np.asarray(self.cols, dtype=np.int64)))
        object.__setattr__(self, "values", _freeze(np.asarray(self.values, dtype=np.float64)))

    @property
    def num_terms(self) -> int:
        return int(self.values.shape[0])
