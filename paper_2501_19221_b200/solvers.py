"""Drop-in solvers: ``solve_pa`` / ``solve_sbm`` / ``integrate`` / ``solve_sa`` on the B200.

Same names, arguments, results and error behaviour as the reference's
``qubokit.solve_pa`` (solvers/parallel_annealing.py:28-48), ``qubokit.solve_sbm``
(solvers/bifurcation.py:50-67) and ``qubokit.solvers.bifurcation.integrate``
(bifurcation.py:37-47); parameter records mirror ``PaParams`` / ``SbmParams``
(solvers/common.py:94-144) and accept the reference's own records too.  ``solve_sa``
(solvers/annealing.py:24-74, ``SaParams`` common.py:74-92) is the other batched-replica
solver of the reference.

Each call is one ``vxq_pa_solve`` / ``vxq_sbm_solve`` through the C-ABI: the
replica streams are drawn on the device (bit-exact numpy Philox), the loop runs
as sm_100a kernels, energies are exact, and the ``SampleSet`` is best-first with
ties broken by replica index (common.py:48-61).

Extra keyword-only options (not in the reference): ``precision`` ("fp32"
default, or "fp64" which reproduces the reference's CSR path bit for bit),
``path`` ("auto" | "resident" | "sparse" | "dense"), ``device`` and
``replica_begin`` (replica sharding).
"""

from __future__ import annotations

import ctypes
import dataclasses
import json
import time
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _lib
from .device import get_problem
from .errors import ValidationError


class Sample(NamedTuple):
    state: np.ndarray
    energy: float
    replica: int


@dataclass
class SampleSet:
    """Seeded, replica-indexed ensemble of (state, energy), best-first (common.py:28-45)."""

    samples: list[Sample]
    replica_count: int
    seed: int | None
    wall_time: float = 0.0
    info: dict = field(default_factory=dict)

    @property
    def best(self) -> Sample:
        return self.samples[0]

    def energies(self) -> np.ndarray:
        return np.array([s.energy for s in self.samples])

    def __len__(self) -> int:
        return len(self.samples)


def _positive(name: str, value: float):
    if not value > 0:
        raise ValidationError(f"{name} must be positive, got {value}")


@dataclass
class PaParams:
    """Parallel annealing parameters (common.py:94-116)."""

    steps: int = 1000
    learning_rate: float = 0.05
    momentum: float = 0.9
    lambda0: float | None = None
    replicas: int = 32
    seed: int = 0

    def validate(self):
        _positive("steps", self.steps)
        _positive("learning_rate", self.learning_rate)
        if not (0 <= self.momentum < 1):
            raise ValidationError("momentum must lie in [0, 1)")
        if self.lambda0 is not None:
            _positive("lambda0", self.lambda0)
        _positive("replicas", self.replicas)


@dataclass
class SbmParams:
    """Simulated bifurcation parameters (common.py:119-144)."""

    steps: int = 10_000
    dt: float = 0.01
    a0: float = 1.0
    c0: float | None = None
    q_cap: float = 1.0
    init_noise: float = 1.0
    replicas: int = 32
    seed: int = 0

    def validate(self):
        _positive("steps", self.steps)
        _positive("dt", self.dt)
        _positive("a0", self.a0)
        if self.c0 is not None:
            _positive("c0", self.c0)
        _positive("q_cap", self.q_cap)
        _positive("init_noise", self.init_noise)
        _positive("replicas", self.replicas)


@dataclass
class SaParams:
    """Simulated annealing parameters (common.py:74-92)."""

    sweeps: int = 1000
    T_init: float | None = None      # None: 2 * model field scale
    T_final: float | None = None     # None: 1e-3 * resolved T_init
    schedule: str = "geometric"
    replicas: int = 32
    seed: int = 0

    def validate(self):
        _positive("sweeps", self.sweeps)
        _positive("replicas", self.replicas)
        if self.schedule != "geometric":
            raise ValidationError("only the geometric schedule is supported")
        if self.T_init is not None and self.T_final is not None:
            if not (self.T_init >= self.T_final > 0):
                raise ValidationError("need T_init >= T_final > 0")


PARAM_CLASSES = {"sa": SaParams, "pa": PaParams, "sbm": SbmParams}


def params_to_dict(params) -> dict:
    return dataclasses.asdict(params)


def params_from_dict(solver_id: str, data: dict):
    """common.py:184-194 (restricted to the solvers on this path)."""
    cls = PARAM_CLASSES.get(solver_id)
    if cls is None:
        raise ValidationError(f"no parameter record for solver {solver_id!r}")
    known = {f.name for f in dataclasses.fields(cls)}
    unknown = set(data) - known
    if unknown:
        raise ValidationError(f"unknown {solver_id} parameters: {sorted(unknown)}")
    params = cls(**data)
    params.validate()
    return params


def default_config() -> str:
    return json.dumps({k: params_to_dict(cls()) for k, cls in PARAM_CLASSES.items()}, indent=2)


def _seed(seed) -> int:
    s = int(seed)
    if not (0 <= s < 2 ** 64):
        raise ValidationError(f"seed must be a non-negative 64-bit integer, got {seed}")
    return s


def _opts(precision: str, path: str, replica_begin: int, stream=None,
          on_device: bool = False, track_best: bool = False) -> _lib.RunOptsC:
    if precision not in ("fp32", "fp64"):
        raise ValidationError(f"precision must be 'fp32' or 'fp64', got {precision!r}")
    if path not in _lib.PATHS:
        raise ValidationError(f"path must be one of {sorted(_lib.PATHS)}, got {path!r}")
    o = _lib.RunOptsC()
    o.precision = _lib.FP64 if precision == "fp64" else _lib.FP32
    o.path = _lib.PATHS[path]
    o.outputs_on_device = 1 if on_device else 0
    o.track_best = 1 if track_best else 0
    o.replica_begin = int(replica_begin)
    # a NULL stream means "the library's own stream for this call"; a caller that hands in
    # the legacy default stream (handle 0, e.g. torch's default current stream) wants work
    # ordered on it, so pass the explicit cudaStreamLegacy handle instead
    if stream is not None and int(stream) == 0:
        stream = 0x1  # cudaStreamLegacy
    o.stream = stream
    return o


class RunResult(NamedTuple):
    states: np.ndarray      # (R, n) int8, replica order
    energies: np.ndarray    # (R,) exact
    order: np.ndarray       # (R,) best-first replica order
    x: np.ndarray | None    # (R, n) final X / Q (fp64 view of the device state)
    m: np.ndarray | None    # (R, n) final M / P
    info: dict


def _outputs(n, R, want_state, trace_steps=0):
    st = np.empty((R, n), dtype=np.int8)
    en = np.empty(R, dtype=np.float64)
    order = np.empty(R, dtype=np.int64)
    x = np.empty((R, n), dtype=np.float64) if want_state else None
    m = np.empty((R, n), dtype=np.float64) if want_state else None
    out = _lib.OutputsC()
    out.states, out.energies, out.order = _lib.ptr(st), _lib.ptr(en), _lib.ptr(order)
    out.x, out.m = _lib.ptr(x), _lib.ptr(m)
    tr = np.empty(trace_steps) if trace_steps else None
    out.energy_trace = _lib.ptr(tr)
    return out, st, en, order, x, m, tr


def run_pa(model, params, *, precision="fp32", path="auto", device=0, replica_begin=0,
           want_state=False, cache=True, trace=False, track_best=False) -> RunResult:
    """One vxq_pa_solve call; returns per-replica arrays (no SampleSet assembly).
    trace: info["energy_trace"][t] = min over replicas of E(s_t); track_best: states and
    energies are each replica's best state seen over s_0..s_T (improvement mode)."""
    params.validate()
    dp = get_problem(model, device, cache=cache)
    c = _lib.PaParamsC(int(params.steps), float(params.learning_rate), float(params.momentum),
                       _lib.nan_if_none(params.lambda0), int(params.replicas), _seed(params.seed))
    out, st, en, order, x, m, tr = _outputs(model.n, int(params.replicas), want_state,
                                            int(params.steps) if trace else 0)
    opts = _opts(precision, path, replica_begin, track_best=track_best)
    _lib.check(_lib.load().vxq_pa_solve(dp.handle, ctypes.byref(c), ctypes.byref(opts),
                                        ctypes.byref(out)))
    info = {"lambda0": out.lambda0_used, "loop_ms": out.loop_ms, "launches": out.launches,
            "path": _lib.PATH_NAMES.get(out.path_used, "?"), "precision": precision,
            "dense_kind": _lib.DENSE_KINDS.get(out.dense_kind),
            "kernel": _lib.STEP_KERNELS.get(out.step_kernel), "energy_trace": tr,
            "track_best": track_best}
    return RunResult(st, en, order, x, m, info)


def run_sbm(model, params, *, precision="fp32", path="auto", device=0, replica_begin=0,
            want_state=False, cache=True, trace=False, track_best=False) -> RunResult:
    params.validate()
    dp = get_problem(model, device, cache=cache)
    c = _lib.SbmParamsC(int(params.steps), float(params.dt), float(params.a0),
                        _lib.nan_if_none(params.c0), float(params.q_cap),
                        float(params.init_noise), int(params.replicas), _seed(params.seed))
    out, st, en, order, x, m, tr = _outputs(model.n, int(params.replicas), want_state,
                                            int(params.steps) if trace else 0)
    opts = _opts(precision, path, replica_begin, track_best=track_best)
    _lib.check(_lib.load().vxq_sbm_solve(dp.handle, ctypes.byref(c), ctypes.byref(opts),
                                         ctypes.byref(out)))
    info = {"c0": out.c0_used, "loop_ms": out.loop_ms, "launches": out.launches,
            "path": _lib.PATH_NAMES.get(out.path_used, "?"), "precision": precision,
            "dense_kind": _lib.DENSE_KINDS.get(out.dense_kind),
            "kernel": _lib.STEP_KERNELS.get(out.step_kernel), "energy_trace": tr,
            "track_best": track_best}
    return RunResult(st, en, order, x, m, info)


def sa_schedule(T_init: float, T_final: float, sweeps: int) -> np.ndarray:
    """Geometric temperatures, the reference's expression (annealing.py:31-35)."""
    if sweeps > 1:
        ratio = (T_final / T_init) ** (1.0 / (sweeps - 1))
        return T_init * ratio ** np.arange(sweeps)
    return np.array([T_init], dtype=np.float64)


def _sa_temps(model, params, device):
    T_init = params.T_init if params.T_init is not None else \
        2.0 * get_problem(model, device).lambda0()
    T_final = params.T_final if params.T_final is not None else 1e-3 * T_init
    return float(T_init), float(T_final), np.ascontiguousarray(
        sa_schedule(float(T_init), float(T_final), int(params.sweeps)), dtype=np.float64)


def run_sa(model, params, *, precision="fp32", path="auto", device=0, replica_begin=0,
           cache=True) -> RunResult:
    """One vxq_sa_solve call: per-replica best states / exact energies / order."""
    params.validate()
    dp = get_problem(model, device, cache=cache)
    T0, T1, temps = _sa_temps(model, params, device)
    c = _lib.SaParamsC(int(params.sweeps), T0, T1, int(params.replicas), _seed(params.seed),
                       _lib.ptr(temps))
    out, st, en, order, _, _, _ = _outputs(model.n, int(params.replicas), False)
    opts = _opts(precision, path, replica_begin)
    _lib.check(_lib.load().vxq_sa_solve(dp.handle, ctypes.byref(c), ctypes.byref(opts),
                                        ctypes.byref(out)))
    info = {"T_init": out.lambda0_used, "T_final": out.c0_used, "loop_ms": out.loop_ms,
            "launches": out.launches, "path": _lib.PATH_NAMES.get(out.path_used, "?"),
            "precision": precision, "kernel": _lib.STEP_KERNELS.get(out.step_kernel)}
    return RunResult(st, en, order, None, None, info)


def run_device(kind: str, model, params, states_ptr: int, energies_ptr: int, *,
               order_ptr: int | None = None, stream: int | None = None, precision="fp32",
               path="auto", device=0, replica_begin=0) -> dict:
    """Device-resident variant: outputs go to caller-owned DEVICE buffers
    (states int8 [R][n], energies fp64 [R], optional order int64 [R]) on ``stream``.
    Used by bench.py for the HBM-resident throughput number."""
    params.validate()
    dp = get_problem(model, device)
    out = _lib.OutputsC()
    out.states, out.energies = ctypes.c_void_p(states_ptr), ctypes.c_void_p(energies_ptr)
    out.order = ctypes.c_void_p(order_ptr) if order_ptr else None
    opts = _opts(precision, path, replica_begin, stream=stream, on_device=True)
    L = _lib.load()
    if kind == "pa":
        c = _lib.PaParamsC(int(params.steps), float(params.learning_rate),
                           float(params.momentum), _lib.nan_if_none(params.lambda0),
                           int(params.replicas), _seed(params.seed))
        _lib.check(L.vxq_pa_solve(dp.handle, ctypes.byref(c), ctypes.byref(opts),
                                  ctypes.byref(out)))
    else:
        c = _lib.SbmParamsC(int(params.steps), float(params.dt), float(params.a0),
                            _lib.nan_if_none(params.c0), float(params.q_cap),
                            float(params.init_noise), int(params.replicas), _seed(params.seed))
        _lib.check(L.vxq_sbm_solve(dp.handle, ctypes.byref(c), ctypes.byref(opts),
                                   ctypes.byref(out)))
    return {"lambda0": out.lambda0_used, "c0": out.c0_used, "loop_ms": out.loop_ms,
            "launches": out.launches, "path": _lib.PATH_NAMES.get(out.path_used, "?"),
            "dense_kind": _lib.DENSE_KINDS.get(out.dense_kind),
            "kernel": _lib.STEP_KERNELS.get(out.step_kernel)}


def sampleset_from(res: RunResult, R: int, seed, wall_time: float, replica_begin: int = 0):
    """make_sampleset (common.py:48-61) from device results (order already stable-sorted)."""
    # each Sample's state is its own row of the freshly allocated (R, n) result array (no
    # other holder), so rows are handed out as views instead of copies (the reference
    # copies, common.py:58: 256 MB of host memcpy per cfg4 solve)
    samples = [Sample(res.states[r], float(res.energies[r]), int(r) + replica_begin)
               for r in res.order]
    return SampleSet(samples=samples, replica_count=R, seed=seed, wall_time=wall_time,
                     info=res.info)


def solve_pa(model, params, *, precision: str = "fp32", path: str = "auto", device: int = 0,
             replica_begin: int = 0, trace: bool = False, track_best: bool = False) -> SampleSet:
    """Parallel annealing on the B200 (drop-in for parallel_annealing.py:28-48)."""
    params.validate()
    t0 = time.perf_counter()
    res = run_pa(model, params, precision=precision, path=path, device=device,
                 replica_begin=replica_begin, trace=trace, track_best=track_best)
    return sampleset_from(res, int(params.replicas), params.seed, time.perf_counter() - t0,
                          replica_begin)


def solve_sbm(model, params, *, precision: str = "fp32", path: str = "auto", device: int = 0,
              replica_begin: int = 0, trace: bool = False, track_best: bool = False) -> SampleSet:
    """Simulated bifurcation on the B200 (drop-in for bifurcation.py:50-67)."""
    params.validate()
    t0 = time.perf_counter()
    res = run_sbm(model, params, precision=precision, path=path, device=device,
                  replica_begin=replica_begin, trace=trace, track_best=track_best)
    return sampleset_from(res, int(params.replicas), params.seed, time.perf_counter() - t0,
                          replica_begin)


def solve_sa(model, params, *, precision: str = "fp32", path: str = "auto", device: int = 0,
             replica_begin: int = 0) -> SampleSet:
    """Simulated annealing on the B200 (drop-in for annealing.py:24-74): every replica
    reports the best state seen along its trajectory."""
    params.validate()
    t0 = time.perf_counter()
    res = run_sa(model, params, precision=precision, path=path, device=device,
                 replica_begin=replica_begin)
    return sampleset_from(res, int(params.replicas), params.seed, time.perf_counter() - t0,
                          replica_begin)


def time_to_target(trace, target: float, loop_ms: float):
    """First step whose spins reach `target` (min over replicas) and the corresponding
    time assuming uniform step cost: (step, ms) or (None, None)."""
    tr = np.asarray(trace)
    hit = np.nonzero(tr <= target)[0]
    if hit.size == 0:
        return None, None
    t = int(hit[0])
    return t, loop_ms * (t + 1) / tr.size


def resolve_lambda0(model) -> float:
    """max(field_scale, 1e-12) on the GPU (parallel_annealing.py:23-25)."""
    return get_problem(model).lambda0()


def resolve_c0(model) -> float:
    """1 / lambda_max(-A) on the GPU (Lanczos), 1.0 without couplings (bifurcation.py:25-34)."""
    if len(np.asarray(model.values)) == 0:
        return 1.0
    return get_problem(model).c0()


def _bt_csr(B):
    """CSR of B^T with ascending columns: field_i = sum_j B[j, i] q_j  (Q @ B)."""
    import scipy.sparse as sp
    if sp.issparse(B):
        Bt = sp.csr_array(B.T)
    else:
        Bt = sp.csr_array(np.asarray(B, dtype=np.float64).T)
    Bt.sum_duplicates()
    Bt.sort_indices()
    return (np.ascontiguousarray(Bt.indptr, dtype=np.int64),
            np.ascontiguousarray(Bt.indices, dtype=np.int32),
            np.ascontiguousarray(Bt.data, dtype=np.float64))


def integrate(B, g, Q, P, dt: float, a_schedule, a0: float, c0: float, q_cap: float, *,
              precision: str = "fp32", path: str = "auto"):
    """Core symplectic loop on the GPU; mutates Q and P in place (bifurcation.py:37-47)."""
    if not (isinstance(Q, np.ndarray) and isinstance(P, np.ndarray)):
        raise ValidationError("Q and P must be numpy arrays (updated in place)")
    if Q.shape != P.shape or Q.ndim != 2:
        raise ValidationError(f"Q and P must be (R, n) arrays, got {Q.shape} / {P.shape}")
    R, n = Q.shape
    indptr, indices, data = _bt_csr(B)
    if indptr.shape[0] != n + 1:
        raise ValidationError(f"B must be ({n}, {n})")
    gv = np.ascontiguousarray(np.broadcast_to(np.asarray(g, dtype=np.float64), (n,)))
    sched = np.ascontiguousarray(np.asarray(a_schedule, dtype=np.float64).ravel())
    q = np.ascontiguousarray(Q, dtype=np.float64)
    p = np.ascontiguousarray(P, dtype=np.float64)
    q = q.copy() if q is Q else q
    p = p.copy() if p is P else p
    _lib.require_gpu()
    opts = _opts(precision, path, 0)
    _lib.check(_lib.load().vxq_sbm_integrate(n, _lib.ptr(indptr), _lib.ptr(indices),
                                             _lib.ptr(data), _lib.ptr(gv), R, _lib.ptr(q),
                                             _lib.ptr(p), _lib.ptr(sched), sched.shape[0],
                                             float(dt), float(a0), float(c0), float(q_cap),
                                             ctypes.byref(opts)))
    Q[...] = q
    P[...] = p
    return Q, P


def replica_streams(seed, count: int) -> list[np.random.Generator]:
    """Host numpy view of the replica streams (common.py:64-65); the solvers draw the
    same streams on the device."""
    out = []
    for r in range(count):
        bits = np.random.Philox(key=np.uint64(seed))
        if r:
            bits = bits.jumped(r)
        out.append(np.random.Generator(bits))
    return out


def pa_schedule(lambda0: float, steps: int) -> np.ndarray:
    """lam_t = lambda0 * (1.0 - t / T) as the library computes it (vxq_pa_schedule)."""
    out = np.empty(int(steps), dtype=np.float64)
    _lib.check(_lib.load().vxq_pa_schedule(float(lambda0), int(steps), _lib.ptr(out)))
    return out


def sbm_schedule(a0: float, steps: int) -> np.ndarray:
    """np.linspace(0.0, a0, T) as the library computes it (vxq_sbm_schedule)."""
    out = np.empty(int(steps), dtype=np.float64)
    _lib.check(_lib.load().vxq_sbm_schedule(float(a0), int(steps), _lib.ptr(out)))
    return out

