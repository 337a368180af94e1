"""oracle -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's batched multi-replica dynamics loop
(qubokit PA / SBM) used as the *checker* by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` leg of ``bench.py``.
The product package (``paper_2501_19221_b200``) never imports this module.

Pinned against the reference: ``tests/golden/*.npz`` were produced by running
the unmodified reference (``/root/reference/pkg/src/qubokit``) through
``tests/golden/make_golden.py``; ``tests/test_oracle.py`` checks this oracle
against every one of those vectors (Philox draws, lambda0, c0, PA/SBM
trajectories, final states and energies).

Reference file:line anchors for each function are given in its docstring.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile oracle.c (plain C, gcc) into oracle/_build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or (os.path.getmtime(_SO) <
                                        os.path.getmtime(os.path.join(_HERE, "oracle.c"))):
            build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, u64, f64, f32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_float
        L.orc_philox_raw.restype = u64
        L.orc_philox_raw.argtypes = [u64, u64, u64]
        L.orc_uniform.argtypes = [u64, u64, u64, i64, f64, f64, P]
        L.orc_field_scale.restype = f64
        L.orc_field_scale.argtypes = [i64, i64, P, P, P, P, P]
        L.orc_pa_run_f64.argtypes = [i64, i64, P, P, P, P, P, i64, f64, f64, P, P, P, P]
        L.orc_pa_run_f32.argtypes = [i64, i64, P, P, P, P, P, i64, f32, f32, P, P, P, P]
        L.orc_sbm_run_f64.argtypes = [i64, i64, P, P, P, P, P, i64, f64, f64, f64, f64, f64,
                                      P, P, P]
        L.orc_sbm_run_f32.argtypes = [i64, i64, P, P, P, P, P, i64, f32, f32, f32, f32, f32,
                                      P, P, P]
        L.orc_sa_init_spins.argtypes = [i64, u64, u64, P]
        L.orc_sa_run_f64.argtypes = [i64, i64, P, P, P, P, P, i64, u64, i64, P, P, P, P, P]
        L.orc_sa_run_f32.argtypes = [i64, i64, P, P, P, P, P, i64, u64, i64, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# replica streams -- generators.py:35-40, solvers/common.py:64-65
# --------------------------------------------------------------------------
M64 = (1 << 64) - 1
_PM0, _PM1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_PW0, _PW1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def philox4x64_10_py(ctr, key):
    """Pure-Python Philox4x64-10 (numpy's bit generator), for KATs."""
    c = list(ctr)
    k0, k1 = key
    for _ in range(10):
        p0, p1 = _PM0 * c[0], _PM1 * c[2]
        c = [((p1 >> 64) ^ c[1] ^ k0) & M64, p1 & M64, ((p0 >> 64) ^ c[3] ^ k1) & M64, p0 & M64]
        k0, k1 = (k0 + _PW0) & M64, (k1 + _PW1) & M64
    return c


def philox_raw_py(seed: int, replica: int, k: int) -> int:
    """Raw draw k of rng_stream(seed, replica): ctr=(k//4+1, 0, replica, 0), key=(seed, 0)."""
    return philox4x64_10_py((k // 4 + 1, 0, replica, 0), (seed, 0))[k % 4]


def uniform(seed: int, replica: int, first: int, count: int, lo: float, hi: float) -> np.ndarray:
    """numpy Generator.uniform on rng_stream(seed, replica), draws [first, first+count)."""
    out = np.empty(count, dtype=np.float64)
    lib().orc_uniform(seed, replica, first, count, lo, hi, _p(out))
    return out


def pa_init(seed: int, R: int, n: int) -> np.ndarray:
    """X0 of solve_pa: stream r -> uniform(-1, 1, n)  (parallel_annealing.py:35-36)."""
    return np.stack([uniform(seed, r, 0, n, -1.0, 1.0) for r in range(R)])


def sbm_init(seed: int, R: int, n: int, amp: float):
    """Q0, P0 of solve_sbm: stream r -> n Q draws then n P draws (bifurcation.py:59-61)."""
    Q = np.stack([uniform(seed, r, 0, n, -amp, amp) for r in range(R)])
    P = np.stack([uniform(seed, r, n, n, -amp, amp) for r in range(R)])
    return Q, P


# --------------------------------------------------------------------------
# operators -- model.py:166-192
# --------------------------------------------------------------------------
def symmetric_csr(n, rows, cols, values):
    """Symmetric coupling CSR with ascending columns per row (both triangles)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    m = rows.shape[0]
    canonical = m == 0 or (np.all(rows < cols) and np.all(
        (rows[1:] > rows[:-1]) | ((rows[1:] == rows[:-1]) & (cols[1:] > cols[:-1]))))
    if canonical:
        # row i = [j < i ascending (from the stable col-grouping)] + [j > i ascending]
        deg_up = np.bincount(rows, minlength=n)
        deg_lo = np.bincount(cols, minlength=n)
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(deg_up + deg_lo, out=indptr[1:])
        ustart = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(deg_up, out=ustart[1:])
        lstart = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(deg_lo, out=lstart[1:])
        indices = np.empty(2 * m, dtype=np.int32)
        data = np.empty(2 * m, dtype=np.float64)
        k = np.arange(m, dtype=np.int64)
        pos_up = indptr[rows] + deg_lo[rows] + (k - ustart[rows])
        indices[pos_up] = cols
        data[pos_up] = values
        perm = np.argsort(cols, kind="stable")
        c = cols[perm]
        pos_lo = indptr[c] + (k - lstart[c])
        indices[pos_lo] = rows[perm]
        data[pos_lo] = values[perm]
        return indptr, indices, data
    r = np.concatenate([rows, cols])
    c = np.concatenate([cols, rows])
    v = np.concatenate([values, values])
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, r + 1, 1)
    indptr = np.cumsum(indptr)
    return indptr, c.astype(np.int32), v


def transpose_csr(B):
    """CSR of B^T with ascending columns: field_i = sum_j B[j, i] q_j (Q @ B)."""
    import scipy.sparse as sp
    if sp.issparse(B):
        Bt = sp.csr_array(B.T)
    else:
        Bt = sp.csr_array(np.asarray(B, dtype=np.float64).T)
    Bt.sum_duplicates()
    Bt.sort_indices()
    return (Bt.indptr.astype(np.int64), Bt.indices.astype(np.int32),
            Bt.data.astype(np.float64))


def field_scale(model) -> float:
    """model.field_scale (model.py:194-200), same np.add.at accumulation order."""
    n = model.n
    rows = np.ascontiguousarray(model.rows, dtype=np.int64)
    cols = np.ascontiguousarray(model.cols, dtype=np.int64)
    vals = np.ascontiguousarray(model.values, dtype=np.float64)
    h = np.ascontiguousarray(model.h, dtype=np.float64)
    out = np.empty(n, dtype=np.float64)
    return float(lib().orc_field_scale(n, len(vals), _p(rows), _p(cols), _p(vals), _p(h),
                                       _p(out)))


def resolve_lambda0(model) -> float:
    """parallel_annealing.py:23-25."""
    return max(field_scale(model), 1e-12)


def resolve_c0(model) -> float:
    """bifurcation.py:25-34 with a dense eigensolve (numpy eigvalsh)."""
    if len(model.values) == 0:
        return 1.0
    A = np.zeros((model.n, model.n))
    A[model.rows, model.cols] = model.values
    A[model.cols, model.rows] = model.values
    lam = float(np.linalg.eigvalsh(-A)[-1])
    return 1.0 / lam if lam > 1e-12 else 1.0


def pa_schedule(lam0: float, T: int) -> np.ndarray:
    """lam_t = lam0 * (1.0 - t / T) in Python floats (parallel_annealing.py:42)."""
    return np.array([lam0 * (1.0 - t / T) for t in range(T)], dtype=np.float64)


def sbm_schedule(a0: float, T: int) -> np.ndarray:
    """a_schedule = np.linspace(0.0, a0, T) (bifurcation.py:63)."""
    return np.linspace(0.0, a0, T)


# --------------------------------------------------------------------------
# dynamics loops
# --------------------------------------------------------------------------
def pa_run(indptr, indices, data, h, lam_sched, eta, alpha, X, M, dtype=np.float64):
    """Run the PA loop (parallel_annealing.py:41-45) in place on X, M (R, n)."""
    dt = np.dtype(dtype)
    X = np.ascontiguousarray(X, dtype=dt)
    M = np.ascontiguousarray(M, dtype=dt)
    R, n = X.shape
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    dv = np.ascontiguousarray(data, dtype=dt)
    hv = np.ascontiguousarray(h, dtype=dt)
    ls = np.ascontiguousarray(lam_sched, dtype=dt)
    s1 = np.empty(n, dtype=dt)
    s2 = np.empty(n, dtype=dt)
    fn = lib().orc_pa_run_f64 if dt == np.float64 else lib().orc_pa_run_f32
    fn(n, R, _p(ip), _p(ix), _p(dv), _p(hv), _p(ls), len(ls), float(eta), float(alpha),
       _p(X), _p(M), _p(s1), _p(s2))
    return X, M


def sbm_run(indptr, indices, data, g, a_sched, dt_, a0, c0, q_cap, Q, P, dtype=np.float64):
    """Run SBM integrate (bifurcation.py:37-47) on (Q, P); B given as CSR of B^T."""
    dt = np.dtype(dtype)
    Q = np.ascontiguousarray(Q, dtype=dt)
    P = np.ascontiguousarray(P, dtype=dt)
    R, n = Q.shape
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    dv = np.ascontiguousarray(data, dtype=dt)
    gv = np.ascontiguousarray(g, dtype=dt)
    sa = np.ascontiguousarray(a_sched, dtype=dt)
    tmp = np.empty(n, dtype=dt)
    fn = lib().orc_sbm_run_f64 if dt == np.float64 else lib().orc_sbm_run_f32
    fn(n, R, _p(ip), _p(ix), _p(dv), _p(gv), _p(sa), len(sa), float(dt_), float(a0),
       float(c0), float(q_cap), float(dt_ * a0), _p(Q), _p(P), _p(tmp))
    return Q, P


def sign_pm(x) -> np.ndarray:
    """model.py:36-38: where(x >= 0, 1, -1) as int8 (sign(0) = sign(-0) = +1)."""
    return np.where(np.asarray(x) >= 0, 1, -1).astype(np.int8)


def pa_solve(model, steps, lr=0.05, momentum=0.9, lambda0=None, replicas=32, seed=0,
             dtype=np.float64):
    """solve_pa restated (parallel_annealing.py:28-48): returns (states, X, M)."""
    lam0 = lambda0 if lambda0 is not None else resolve_lambda0(model)
    ip, ix, dv = symmetric_csr(model.n, model.rows, model.cols, model.values)
    X = pa_init(seed, replicas, model.n)
    M = np.zeros_like(X)
    X, M = pa_run(ip, ix, dv, model.h, pa_schedule(lam0, steps), lr, momentum, X, M, dtype)
    return sign_pm(X), X, M


def sbm_solve(model, steps, dt=0.01, a0=1.0, c0=None, q_cap=1.0, init_noise=1.0,
              replicas=32, seed=0, dtype=np.float64):
    """solve_sbm restated (bifurcation.py:50-67): returns (states, Q, P)."""
    c0 = c0 if c0 is not None else resolve_c0(model)
    ip, ix, dv = symmetric_csr(model.n, model.rows, model.cols, model.values)
    Q, P = sbm_init(seed, replicas, model.n, init_noise)
    Q, P = sbm_run(ip, ix, -dv, -np.asarray(model.h, dtype=np.float64),
                   sbm_schedule(a0, steps), dt, a0, c0, q_cap, Q, P, dtype)
    return sign_pm(Q), Q, P


def sa_init(seed: int, R: int, n: int, replica_begin: int = 0) -> np.ndarray:
    """Initial SA spins: stream r -> 2 * integers(0, 2, n) - 1 (annealing.py:40)."""
    S = np.empty((R, n), dtype=np.int8)
    for r in range(R):
        lib().orc_sa_init_spins(n, seed, replica_begin + r, _p(S[r]))
    return S


def sa_schedule(T_init, T_final, sweeps) -> np.ndarray:
    """annealing.py:31-35."""
    if sweeps > 1:
        ratio = (T_final / T_init) ** (1.0 / (sweeps - 1))
        return T_init * ratio ** np.arange(sweeps)
    return np.array([T_init], dtype=np.float64)


def sa_solve(model, sweeps, T_init=None, T_final=None, replicas=32, seed=0,
             dtype=np.float64, replica_begin=0):
    """solve_sa restated (annealing.py:24-74): returns (best states, tracked best E)."""
    n = model.n
    T0 = T_init if T_init is not None else 2.0 * resolve_lambda0(model)
    T1 = T_final if T_final is not None else 1e-3 * T0
    temps = np.ascontiguousarray(sa_schedule(T0, T1, sweeps), dtype=np.float64)
    ip, ix, dv = symmetric_csr(n, model.rows, model.cols, model.values)
    S0 = sa_init(seed, replicas, n, replica_begin)
    E0 = np.array([energy_exact(model, s) - float(model.offset) for s in S0])
    best = np.empty((replicas, n), dtype=np.int8)
    bestE = np.empty(replicas)
    work = np.empty(n, dtype=np.int8)
    if dtype == np.float64:
        F = np.empty(n)
        hv = np.ascontiguousarray(model.h, dtype=np.float64)
        fn, dd = lib().orc_sa_run_f64, np.ascontiguousarray(dv, dtype=np.float64)
    else:
        F = np.empty(n, dtype=np.float32)
        hv = np.ascontiguousarray(model.h, dtype=np.float32)
        fn, dd = lib().orc_sa_run_f32, np.ascontiguousarray(dv, dtype=np.float32)
    fn(n, replicas, _p(ip), _p(ix), _p(dd), _p(hv), _p(temps), int(sweeps), int(seed),
       int(replica_begin), _p(E0), _p(best), _p(bestE), _p(F), _p(work))
    return best, bestE


# --------------------------------------------------------------------------
# energies -- model.py:153-164 (correctly rounded exact sum)
# --------------------------------------------------------------------------
def energy_exact(model, s) -> float:
    """Correctly rounded H(s) = offset + sum J_ij s_i s_j + sum h_i s_i (math.fsum).

    Every term is an exact double (J * (+-1)), so fsum returns the correctly
    rounded exact value; this is independent of the GPU's fixed-point method.
    """
    s = np.asarray(s, dtype=np.float64)
    rows = np.asarray(model.rows)
    cols = np.asarray(model.cols)
    terms = np.asarray(model.values) * s[rows] * s[cols]
    lin = np.asarray(model.h) * s
    return math.fsum([float(model.offset)] + terms.tolist() + lin.tolist())


def energy_fraction(model, s) -> float:
    """Same as energy_exact through Fraction arithmetic (slow; cross-check)."""
    tot = Fraction(float(model.offset))
    for i, j, v in zip(model.rows, model.cols, model.values):
        tot += Fraction(float(v)) * int(s[i]) * int(s[j])
    for i, hv in enumerate(model.h):
        tot += Fraction(float(hv)) * int(s[i])
    return float(tot)


def energies_exact(model, states) -> np.ndarray:
    return np.array([energy_exact(model, s) for s in np.asarray(states)], dtype=np.float64)


def sampleset_order(energies) -> np.ndarray:
    """make_sampleset ordering: argsort(kind='stable') (common.py:57)."""
    return np.argsort(np.asarray(energies), kind="stable")
