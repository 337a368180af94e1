"""Generate golden vectors by running the UNMODIFIED reference (qubokit).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array stored here is an output of reference code paths:
  - rng_stream / replica_streams         generators.py:35-40, common.py:64-65
  - solve_pa / its loop lines            parallel_annealing.py:28-48
  - solve_sbm / integrate                bifurcation.py:37-67
  - resolve_lambda0 / resolve_c0         parallel_annealing.py:23-25, bifurcation.py:25-34
  - IsingModel.energies / energy         model.py:153-164
  - qubo_to_ising                        transforms.py:36-56
The fixtures travel to the GPU box (the reference does not).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import qubokit as qk  # noqa: E402
from qubokit.model import sign_pm  # noqa: E402
from qubokit.solvers import resolve_c0, resolve_lambda0  # noqa: E402
from qubokit.solvers.bifurcation import integrate  # noqa: E402
from qubokit.solvers.common import replica_streams  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def model_arrays(prefix, m):
    return {f"{prefix}_n": np.int64(m.n), f"{prefix}_rows": m.rows, f"{prefix}_cols": m.cols,
            f"{prefix}_values": m.values, f"{prefix}_h": m.h,
            f"{prefix}_offset": np.float64(m.offset)}


def pa_trajectory(m, params, checkpoints):
    """The reference PA loop verbatim (parallel_annealing.py:35-45), X/M kept at checkpoints."""
    n, R, T = m.n, params.replicas, params.steps
    lam0 = params.lambda0 if params.lambda0 is not None else resolve_lambda0(m)
    eta, alpha = params.learning_rate, params.momentum
    streams = replica_streams(params.seed, R)
    X = np.stack([g.uniform(-1.0, 1.0, size=n) for g in streams])
    M = np.zeros_like(X)
    A = m.coupling_operator()
    h = m.h
    out = {}
    for t in range(T):
        lam = lam0 * (1.0 - t / T)
        grad = lam * X + sign_pm(X).astype(np.float64) @ A + h
        M = alpha * M - eta * grad
        X = np.clip(X + M, -1.0, 1.0)
        if t + 1 in checkpoints:
            out[t + 1] = (X.copy(), M.copy())
    return out


def sbm_trajectory(m, params, checkpoints):
    """solve_sbm's setup + integrate (bifurcation.py:50-63) run piecewise."""
    n, R, T = m.n, params.replicas, params.steps
    c0 = params.c0 if params.c0 is not None else resolve_c0(m)
    B = -m.coupling_operator()
    g = -m.h
    amp = params.init_noise
    streams = replica_streams(params.seed, R)
    Q = np.stack([s.uniform(-amp, amp, size=n) for s in streams])
    P = np.stack([s.uniform(-amp, amp, size=n) for s in streams])
    a_schedule = np.linspace(0.0, params.a0, T)
    out = {}
    done = 0
    for cp in sorted(checkpoints):
        Q, P = integrate(B, g, Q, P, params.dt, a_schedule[done:cp], params.a0, c0,
                         params.q_cap)
        done = cp
        out[cp] = (Q.copy(), P.copy())
    return out, c0


def by_replica(sset, n):
    R = sset.replica_count
    states = np.zeros((R, n), dtype=np.int8)
    energies = np.zeros(R)
    order = np.zeros(R, dtype=np.int64)
    for pos, s in enumerate(sset.samples):
        states[s.replica] = s.state
        energies[s.replica] = s.energy
        order[pos] = s.replica
    return states, energies, order


def qubo_cfg1(seed, n=100):
    """BASELINE config 1: QUBO on all i<=j pairs, Q ~ uniform[-1,1] -> qubo_to_ising."""
    rng = qk.rng_stream(seed)
    pairs = [(i, j) for i in range(n) for j in range(i, n)]
    vals = rng.uniform(-1.0, 1.0, size=len(pairs))
    q = qk.QuboModel.from_terms(n, terms=[(i, j, float(v)) for (i, j), v in zip(pairs, vals)])
    return q, qk.qubo_to_ising(q)


def main():
    g = {}
    # ---- Philox KATs (generators.py:35-40) ----
    kat_seeds = np.array([0, 7, 123, 2**63 + 5, 42], dtype=np.uint64)
    kat_reps = np.array([0, 3, 4095, 77, 1_000_003], dtype=np.uint64)
    raws, unis, amps = [], [], []
    for s, r in zip(kat_seeds, kat_reps):
        bg = np.random.Philox(key=np.uint64(s))
        if r:
            bg = bg.jumped(int(r))
        raws.append([int(bg.random_raw()) for _ in range(11)])
        gen = qk.rng_stream(int(s), int(r))
        unis.append(gen.uniform(-1.0, 1.0, size=11))
        gen = qk.rng_stream(int(s), int(r))
        amps.append(gen.uniform(-0.37, 0.37, size=11))
    g["kat_seed"] = kat_seeds
    g["kat_replica"] = kat_reps
    g["kat_raw"] = np.array(raws, dtype=np.uint64)
    g["kat_uniform"] = np.array(unis)
    g["kat_uniform_amp037"] = np.array(amps)

    # ---- config 1: dense random QUBO N=100 -> Ising, R=64, T=1000 ----
    q, m1 = qubo_cfg1(2501)
    g.update(model_arrays("cfg1", m1))
    g["cfg1_qubo_rows"], g["cfg1_qubo_cols"], g["cfg1_qubo_values"] = q.rows, q.cols, q.values
    g["cfg1_lambda0"] = np.float64(resolve_lambda0(m1))
    g["cfg1_c0"] = np.float64(resolve_c0(m1))
    pa = qk.PaParams(steps=1000, replicas=64, seed=11)
    ss = qk.solve_pa(m1, pa)
    g["cfg1_pa_states"], g["cfg1_pa_energies"], g["cfg1_pa_order"] = by_replica(ss, m1.n)
    tr = pa_trajectory(m1, pa, {1, 10, 100, 1000})
    for t, (X, M) in tr.items():
        g[f"cfg1_pa_X{t}"] = X
        g[f"cfg1_pa_M{t}"] = M
    sb = qk.SbmParams(steps=1000, dt=0.05, replicas=64, seed=13)
    ss = qk.solve_sbm(m1, sb)
    g["cfg1_sbm_states"], g["cfg1_sbm_energies"], g["cfg1_sbm_order"] = by_replica(ss, m1.n)
    tr, _ = sbm_trajectory(m1, sb, {1, 10, 100, 1000})
    for t, (Q, P) in tr.items():
        g[f"cfg1_sbm_Q{t}"] = Q
        g[f"cfg1_sbm_P{t}"] = P

    # ---- sparse n=3000 (reference uses scipy CSR, n > 2048) ----
    rng = np.random.default_rng(3000)
    n = 3000
    edges = set()
    while len(edges) < 3 * n // 2:
        i, j = (int(v) for v in rng.integers(0, n, 2))
        if i != j:
            edges.add((min(i, j), max(i, j)))
    ms = qk.gen_random("edge_list", "uniform", 77, edges=sorted(edges), n=n)
    g.update(model_arrays("sp", ms))
    g["sp_lambda0"] = np.float64(resolve_lambda0(ms))
    g["sp_c0"] = np.float64(resolve_c0(ms))
    pa = qk.PaParams(steps=60, replicas=16, seed=5)
    tr = pa_trajectory(ms, pa, {1, 60})
    for t, (X, M) in tr.items():
        g[f"sp_pa_X{t}"] = X
        g[f"sp_pa_M{t}"] = M
    ss = qk.solve_pa(ms, pa)
    g["sp_pa_states"], g["sp_pa_energies"], _ = by_replica(ss, n)
    sb = qk.SbmParams(steps=60, dt=0.05, replicas=16, seed=6, c0=float(g["sp_c0"]))
    tr, _ = sbm_trajectory(ms, sb, {1, 60})
    for t, (Q, P) in tr.items():
        g[f"sp_sbm_Q{t}"] = Q
        g[f"sp_sbm_P{t}"] = P

    # ---- integer instance: every energy path is exact ----
    mi = qk.gen_random("complete", "int_uniform", 9001, n=50, a=-31, b=31)
    g.update(model_arrays("int", mi))
    S = np.where(rng.random((40, 50)) < 0.5, -1, 1).astype(np.int8)
    g["int_states"] = S
    g["int_energies"] = mi.energies(S)

    # ---- energies of random states on the cfg1 model (BLAS-ordered reference) ----
    S = np.where(rng.random((32, m1.n)) < 0.5, -1, 1).astype(np.int8)
    g["cfg1_rand_states"] = S
    g["cfg1_rand_energies_ref"] = m1.energies(S)
    g["cfg1_rand_energy_scalar_ref"] = np.array([m1.energy(s) for s in S])

    # ---- toy KATs from tests/test_solvers.py ----
    m = qk.IsingModel.from_terms(3, h=[1.0, -2.0, 0.5], couplings=[(0, 1, 2.0), (1, 2, -3.0)])
    g["toy_lambda0"] = np.float64(resolve_lambda0(m))
    mc = qk.gen_random("complete", "uniform", 55, n=12)
    g.update(model_arrays("c0m", mc))
    g["c0m_c0"] = np.float64(resolve_c0(mc))

    np.savez_compressed(os.path.join(OUT, "reference_vectors.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_vectors.npz"), len(g), "arrays")


if __name__ == "__main__":
    main()
