"""Device-resident problems: one ``vxq_problem`` per (model object, device).

The reference caches its coupling operator on the frozen model
(``cached_property _matrix/_csr``, model.py:166-183); here the device CSR and
the exact-energy encoding are cached the same way, keyed on model identity, and
released when the model is garbage collected.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _lib
from .errors import ValidationError

_cache: dict[tuple[int, int], "DeviceProblem"] = {}
_cache_lock = threading.Lock()


def full_triangle(n: int, rows, cols) -> bool:
    """True when the canonical COO arrays are the full upper triangle (a dense model):
    n (n - 1) / 2 sorted unique pairs i < j can only be all of them, so the check is the
    count plus a strided sample (insurance against non-canonical input).  Such a model is
    uploaded as values only -- vxq_problem_create generates the indices on the device."""
    m = len(rows)
    if n < 2 or m == 0 or m != n * (n - 1) // 2 or len(cols) != m:
        return False
    k = np.unique(np.r_[np.linspace(0, m - 1, 4096).astype(np.int64), 0, m - 1])
    i = np.floor(((2 * n - 1) - np.sqrt((2.0 * n - 1) ** 2 - 8.0 * k)) / 2).astype(np.int64)
    st = i * (n - 1) - i * (i - 1) // 2
    i = np.where(st > k, i - 1, i)  # floating-point edge of the closed form
    st = i * (n - 1) - i * (i - 1) // 2
    i = np.where(k >= st + (n - 1 - i), i + 1, i)
    st = i * (n - 1) - i * (i - 1) // 2
    return bool(np.array_equal(np.asarray(rows)[k], i) and
                np.array_equal(np.asarray(cols)[k], i + 1 + (k - st)))


def upload_bytes(model) -> int:
    """Host -> device bytes of a problem upload (COO + h)."""
    n = int(model.n)
    m = len(model.values)
    idx = 0 if full_triangle(n, model.rows, model.cols) else 16 * m
    return idx + 8 * m + 8 * n


class DeviceProblem:
    """Owns one vxq_problem handle."""

    def __init__(self, model, device: int = 0):
        L = _lib.load()
        _lib.require_gpu()
        n = int(model.n)
        rows = np.ascontiguousarray(model.rows, dtype=np.int64)
        cols = np.ascontiguousarray(model.cols, dtype=np.int64)
        vals = np.ascontiguousarray(model.values, dtype=np.float64)
        h = np.ascontiguousarray(model.h, dtype=np.float64)
        if h.shape != (n,):
            raise ValidationError(f"field vector has shape {h.shape}, expected ({n},)")
        handle = ctypes.c_void_p()
        dense = full_triangle(n, rows, cols)  # values only; indices generated on the device
        _lib.check(L.vxq_problem_create(n, int(vals.shape[0]), None if dense else _lib.ptr(rows),
                                        None if dense else _lib.ptr(cols),
                                        _lib.ptr(vals), _lib.ptr(h), float(model.offset),
                                        int(device), ctypes.byref(handle)))
        self.handle = handle
        self.n = n
        self.device = device
        self._finalizer = weakref.finalize(self, L.vxq_problem_destroy, handle)

    def info(self) -> dict:
        out = np.zeros(5, dtype=np.int64)
        _lib.check(_lib.load().vxq_problem_info(self.handle, _lib.ptr(out)))
        return {"n": int(out[0]), "num_couplings": int(out[1]), "nnz": int(out[2]),
                "max_row_nnz": int(out[3]), "uniform_magnitude": bool(out[4])}

    def dense_eligible(self, solver: str, replicas: int, q_cap: float = 1.0,
                       init_noise: float = 1.0) -> bool:
        """Would path="auto" run this fp32 solve on the tensor cores (vxq_dense_eligible)?"""
        v = ctypes.c_int32()
        _lib.check(_lib.load().vxq_dense_eligible(self.handle, 0 if solver == "pa" else 1,
                                                  int(replicas), float(q_cap),
                                                  float(init_noise), ctypes.byref(v)))
        return bool(v.value)

    def lambda0(self) -> float:
        v = ctypes.c_double()
        _lib.check(_lib.load().vxq_problem_lambda0(self.handle, ctypes.byref(v)))
        return v.value

    def c0(self) -> float:
        v = ctypes.c_double()
        _lib.check(_lib.load().vxq_problem_c0(self.handle, ctypes.byref(v)))
        return v.value

    def eig_info(self) -> dict:
        """How the automatic c0 was obtained (vxq_problem_eig_info)."""
        out = np.zeros(6)
        _lib.check(_lib.load().vxq_problem_eig_info(self.handle, _lib.ptr(out)))
        return {"lambda_max": float(out[0]), "theta": float(out[1]), "residual": float(out[2]),
                "iterations": int(out[3]) if out[3] == out[3] else 0,
                "method": {0: "dense-exact", 1: "lanczos", 2: "gershgorin"}.get(int(out[4]),
                                                                                "none"),
                "c0": float(out[5])}

    def close(self):
        self._finalizer()


class GeneratedModel:
    """An instance synthesised on the GPU (vxq_problem_generate): no host arrays unless
    exported.  Accepted by every solver like an IsingModel; `export()` returns the
    canonical IsingModel (host copy) for small instances / cross-checks."""

    FAMILIES = {"qubo_deg6": 0}

    def __init__(self, family: str, n: int, seed: int, device: int = 0):
        if family not in self.FAMILIES:
            raise ValidationError(f"unknown family {family!r}")
        L = _lib.load()
        _lib.require_gpu()
        handle = ctypes.c_void_p()
        _lib.check(L.vxq_problem_generate(self.FAMILIES[family], int(n), int(seed),
                                          int(device), ctypes.byref(handle)))
        dp = DeviceProblem.__new__(DeviceProblem)
        dp.handle, dp.n, dp.device = handle, int(n), device
        dp._finalizer = weakref.finalize(dp, L.vxq_problem_destroy, handle)
        self._dp = dp
        self.family, self.n, self.seed, self.device = family, int(n), int(seed), device
        self.num_couplings = dp.info()["num_couplings"]

    def export(self):
        from .model import IsingModel
        m = self.num_couplings
        rows = np.empty(m, dtype=np.int64)
        cols = np.empty(m, dtype=np.int64)
        vals = np.empty(m)
        h = np.empty(self.n)
        off = ctypes.c_double()
        _lib.check(_lib.load().vxq_problem_export(self._dp.handle, _lib.ptr(rows), _lib.ptr(cols),
                                                  _lib.ptr(vals), _lib.ptr(h), ctypes.byref(off)))
        return IsingModel(n=self.n, h=h, rows=rows, cols=cols, values=vals, offset=off.value)


def get_problem(model, device: int = 0, cache: bool = True) -> DeviceProblem:
    if isinstance(model, GeneratedModel):
        if model.device != device:
            raise ValidationError("generated model lives on another device")
        return model._dp
    if not cache:
        return DeviceProblem(model, device)
    try:  # identity-keyed caching needs a finalizer on the model to drop the entry
        weakref.ref(model)
    except TypeError:  # no weakref support: a later object could reuse the id -> no cache
        return DeviceProblem(model, device)
    key = (id(model), device)
    with _cache_lock:
        dp = _cache.get(key)
        if dp is not None:
            return dp
    dp = DeviceProblem(model, device)
    with _cache_lock:
        existing = _cache.get(key)
        if existing is not None:
            dp.close()
            return existing
        _cache[key] = dp
    weakref.finalize(model, _drop, key)
    return dp


def _drop(key):
    with _cache_lock:
        dp = _cache.pop(key, None)
    if dp is not None:
        dp.close()


def clear_cache(model=None):
    """Release cached device problems (all, or those of one model)."""
    with _cache_lock:
        keys = [k for k in _cache if model is None or k[0] == id(model)]
        dps = [_cache.pop(k) for k in keys]
    for dp in dps:
        dp.close()


def energies(model, states, device: int = 0) -> np.ndarray:
    """Exact energies of (R, n) spin states on the GPU (vxq_energies)."""
    S = np.asarray(states)
    if S.ndim == 1:
        S = S[None, :]
    if S.ndim != 2 or S.shape[1] != model.n:
        raise ValidationError(f"states must have shape (R, {model.n}), got {S.shape}")
    S = np.ascontiguousarray(np.where(S >= 0, 1, -1).astype(np.int8))
    dp = get_problem(model, device)
    out = np.empty(S.shape[0], dtype=np.float64)
    opts = _lib.RunOptsC()
    _lib.check(_lib.load().vxq_energies(dp.handle, _lib.ptr(S), S.shape[0], _lib.ptr(out),
                                        ctypes.byref(opts)))
    return out


def lambda0(model, device: int = 0) -> float:
    return get_problem(model, device).lambda0()


def c0(model, device: int = 0) -> float:
    return get_problem(model, device).c0()
