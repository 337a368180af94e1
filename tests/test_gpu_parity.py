"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden vectors
and the oracle, on the same instances and seeds.

Tolerances (BASELINE north star: bit-exact energies, fp32 trajectory tolerance):
  * energies: bit-exact vs the correctly rounded exact sum (oracle.energy_exact / fsum);
    bit-exact vs the reference on integer instances.
  * fp64 mode: bit-exact trajectories vs the reference wherever it runs scipy CSR
    (n > 2048); |dx| <= 1e-12 where it runs BLAS dgemm (n <= 2048).
  * fp32 mode: bit-exact vs the oracle's fp32 restatement; |dx| <= 1e-5 vs the fp64
    reference for t <= 100 with zero sign mismatches.
"""

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from helpers import (brute_force_min, gen_complete, maxcut_model, model_from_golden,
                     random_regular_edges, sk_model)

pytestmark = pytest.mark.gpu

TOL32 = 1e-5


# ---------------------------------------------------------------- reference trajectories
@pytest.mark.parametrize("path", ["resident", "sparse"])
def test_sparse_instance_fp64_bitexact_with_reference(golden, path):
    m = model_from_golden(golden, "sp")
    lam0 = float(golden["sp_lambda0"])
    r = vxq.run_pa(m, vxq.PaParams(steps=60, replicas=16, seed=5), precision="fp64", path=path,
                   want_state=True)
    assert r.info["lambda0"] == lam0
    assert np.array_equal(r.x, golden["sp_pa_X60"])
    assert np.array_equal(r.m, golden["sp_pa_M60"])
    r1 = vxq.run_pa(m, vxq.PaParams(steps=1, replicas=16, seed=5, lambda0=lam0), precision="fp64",
                    path=path, want_state=True)
    assert np.array_equal(r1.x, golden["sp_pa_X1"])
    s = vxq.run_sbm(m, vxq.SbmParams(steps=60, dt=0.05, replicas=16, seed=6,
                                     c0=float(golden["sp_c0"])),
                    precision="fp64", path=path, want_state=True)
    assert np.array_equal(s.x, golden["sp_sbm_Q60"])
    assert np.array_equal(s.m, golden["sp_sbm_P60"])


def test_sparse_instance_fp32_bitexact_with_oracle(golden):
    m = model_from_golden(golden, "sp")
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    lam = O.pa_schedule(float(golden["sp_lambda0"]), 60)
    X = O.pa_init(5, 16, m.n)
    X, M = O.pa_run(ip, ix, dv, m.h, lam, 0.05, 0.9, X, np.zeros_like(X), np.float32)
    for path in ("resident", "sparse"):
        r = vxq.run_pa(m, vxq.PaParams(steps=60, replicas=16, seed=5), path=path,
                       want_state=True)
        assert np.array_equal(r.x, X.astype(np.float64)), path
        assert np.array_equal(r.m, M.astype(np.float64)), path
    Q, P = O.sbm_init(6, 16, m.n, 1.0)
    Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, 60), 0.05, 1.0,
                     float(golden["sp_c0"]), 1.0, Q, P, np.float32)
    for path in ("resident", "sparse"):
        s = vxq.run_sbm(m, vxq.SbmParams(steps=60, dt=0.05, replicas=16, seed=6,
                                         c0=float(golden["sp_c0"])), path=path, want_state=True)
        assert np.array_equal(s.x, Q.astype(np.float64)), path
        assert np.array_equal(s.m, P.astype(np.float64)), path


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", TOL32)])
def test_cfg1_pa_final_and_trajectory(golden, precision, tol):
    m = model_from_golden(golden, "cfg1")
    lam0 = float(golden["cfg1_lambda0"])
    r = vxq.run_pa(m, vxq.PaParams(steps=1000, replicas=64, seed=11), precision=precision,
                   want_state=True)
    assert r.info["lambda0"] == lam0
    assert np.array_equal(r.states, golden["cfg1_pa_states"])          # all 64 final states
    assert np.abs(r.x - golden["cfg1_pa_X1000"]).max() <= (1e-11 if precision == "fp64" else 1e-4)
    # energies bit-exact vs the exact oracle; within BLAS noise of the reference's own
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))
    scale = np.abs(m.values).sum() + np.abs(m.h).sum() + abs(m.offset)
    assert np.all(np.abs(r.energies - golden["cfg1_pa_energies"]) <= 4e-16 * scale)
    # best energy equal or better than the reference's (compared exactly: the reference's
    # own SampleSet energies are BLAS-ordered and off by a few ulp)
    assert r.energies.min() <= O.energies_exact(m, golden["cfg1_pa_states"]).min()


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", TOL32)])
def test_cfg1_short_horizon_trajectories(golden, precision, tol):
    """t <= 100 through integrate (SBM) and 1-step PA: |dx| <= tol, no sign mismatches."""
    m = model_from_golden(golden, "cfg1")
    c0 = float(golden["cfg1_c0"])
    Q, P = O.sbm_init(13, 64, m.n, 1.0)
    A = m.coupling_matrix()
    a = np.linspace(0.0, 1.0, 1000)
    done = 0
    for t in (1, 10, 100):
        vxq.integrate(-A, -m.h, Q, P, 0.05, a[done:t], 1.0, c0, 1.0, precision=precision)
        done = t
        assert np.abs(Q - golden[f"cfg1_sbm_Q{t}"]).max() <= tol
        assert np.abs(P - golden[f"cfg1_sbm_P{t}"]).max() <= tol
        assert np.array_equal(vxq.sign_pm(Q), vxq.sign_pm(golden[f"cfg1_sbm_Q{t}"]))
    r = vxq.run_pa(m, vxq.PaParams(steps=1000, replicas=64, seed=11), precision=precision,
                   want_state=True)
    assert np.abs(r.x - golden["cfg1_pa_X1000"]).max() <= 100 * tol


def test_cfg1_sbm_solve(golden):
    m = model_from_golden(golden, "cfg1")
    for precision in ("fp64", "fp32"):
        ss = vxq.solve_sbm(m, vxq.SbmParams(steps=1000, dt=0.05, replicas=64, seed=13),
                           precision=precision)
        assert ss.info["c0"] == pytest.approx(float(golden["cfg1_c0"]), rel=1e-9)
        st = np.stack([s.state for s in sorted(ss.samples, key=lambda s: s.replica)])
        assert np.array_equal(st, golden["cfg1_sbm_states"])
        assert ss.best.energy <= O.energies_exact(m, golden["cfg1_sbm_states"]).min()
        assert np.all(np.diff(ss.energies()) >= 0)


# ---------------------------------------------------------------- energies / setup scalars
def test_energies_bitexact(golden):
    m = model_from_golden(golden, "cfg1")
    S = golden["cfg1_rand_states"]
    assert np.array_equal(m.energies(S), O.energies_exact(m, S))
    mi = model_from_golden(golden, "int")
    assert np.array_equal(mi.energies(golden["int_states"]), golden["int_energies"])
    # awkward dynamic range: tiny and huge coefficients mixed
    rng = np.random.default_rng(1)
    n = 40
    iu, ju = np.triu_indices(n, 1)
    v = rng.uniform(-1, 1, len(iu)) * 2.0 ** rng.integers(-60, 40, len(iu))
    mm = vxq.IsingModel.from_arrays(n, iu, ju, v, h=rng.normal(size=n) * 1e-9, offset=1e12,
                                    canonical=True)
    S = np.where(rng.random((70, n)) < 0.5, -1, 1).astype(np.int8)
    assert np.array_equal(mm.energies(S), O.energies_exact(mm, S))


def test_lambda0_and_c0(golden):
    for p in ("cfg1", "sp"):
        m = model_from_golden(golden, p)
        assert vxq.resolve_lambda0(m) == golden[f"{p}_lambda0"]
        # n <= 512: reference uses eigvalsh; n > 512: ARPACK theta + residual (tol 1e-8),
        # so the reference value itself sits ~1e-8 above 1/lambda_max
        assert vxq.resolve_c0(m) == pytest.approx(float(golden[f"{p}_c0"]), rel=1e-7)
    m = model_from_golden(golden, "c0m")
    assert vxq.resolve_c0(m) == pytest.approx(float(golden["c0m_c0"]), rel=1e-6)
    assert vxq.resolve_c0(vxq.IsingModel.from_terms(3, h=[1, 1, 1])) == 1.0


# ---------------------------------------------------------------- the reference's own unit tests
def test_pa_single_spin_field():
    m = vxq.IsingModel.from_terms(1, h=[-1.0])
    r = vxq.solve_pa(m, vxq.PaParams(steps=200, replicas=4, seed=0))
    assert r.best.energy == -1.0
    assert np.array_equal(r.best.state, [1])


def test_pa_and_sbm_match_brute_force_n16():
    hits_pa = hits_sbm = 0
    for seed in range(10):
        m = gen_complete(300 + seed, 16)
        gs = brute_force_min(m)
        hits_pa += abs(vxq.solve_pa(m, vxq.PaParams(steps=500, replicas=32, seed=seed))
                       .best.energy - gs) < 1e-9
        hits_sbm += abs(vxq.solve_sbm(m, vxq.SbmParams(steps=1000, dt=0.1, replicas=32,
                                                       seed=seed)).best.energy - gs) < 1e-9
    assert hits_pa >= 9 and hits_sbm >= 9


def test_sbm_two_oscillator_sync():
    m = vxq.IsingModel.from_terms(2, couplings=[(0, 1, -10.0)])
    agree = 0
    for seed in range(100):
        s = vxq.solve_sbm(m, vxq.SbmParams(steps=1000, dt=0.1, replicas=1, seed=seed)).best.state
        agree += s[0] == s[1]
    assert agree >= 99


def test_sbm_unbiased_free_oscillator():
    m = vxq.IsingModel.from_terms(1)
    r = vxq.solve_sbm(m, vxq.SbmParams(steps=200, dt=0.05, replicas=10_000, seed=123))
    ups = sum(int(s.state[0] == 1) for s in r.samples)
    assert 0.45 <= ups / 10_000 <= 0.55


def test_sbm_symplectic_drift_bounded():
    a0, dt, steps = 1.0, 0.01, 10_000
    Q = np.array([[0.5]])
    P = np.array([[0.0]])
    e0 = 0.25 * 0.5 ** 4
    drifts = []
    for _ in range(2):
        vxq.integrate(np.zeros((1, 1)), np.zeros(1), Q, P, dt, np.full(steps // 2, a0), a0, 0.0,
                      q_cap=np.inf, precision="fp64")
        drifts.append(abs(0.5 * a0 * P[0, 0] ** 2 + 0.25 * Q[0, 0] ** 4 - e0))
    assert drifts[1] < 0.05 * e0 + 1e-12
    assert drifts[1] < 10 * max(drifts[0], 1e-6)


def test_sbm_divergence_guard():
    m = vxq.IsingModel.from_terms(1, h=[100.0])
    r = vxq.solve_sbm(m, vxq.SbmParams(steps=500, dt=0.1, replicas=2, seed=0, c0=5.0))
    assert r.best.energy == -100.0


def test_determinism_and_replica_sharding():
    m = gen_complete(29, 40, "gaussian")
    a = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=96, seed=5), want_state=True)
    b = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=96, seed=5), want_state=True)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.energies, b.energies)
    # replica r depends only on stream r: a shard [32, 64) equals rows 32..63 of the full run
    c = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=32, seed=5), replica_begin=32,
                   want_state=True)
    assert np.array_equal(c.x, a.x[32:64])
    s1 = vxq.run_sbm(m, vxq.SbmParams(steps=300, dt=0.05, replicas=96, seed=9), want_state=True)
    s2 = vxq.run_sbm(m, vxq.SbmParams(steps=300, dt=0.05, replicas=40, seed=9),
                     replica_begin=50, want_state=True)
    assert np.array_equal(s2.x, s1.x[50:90])


def test_qubo_in_bits_out(golden):
    q = vxq.QuboModel(n=int(golden["cfg1_n"]), rows=golden["cfg1_qubo_rows"],
                      cols=golden["cfg1_qubo_cols"], values=golden["cfg1_qubo_values"])
    ising = vxq.qubo_to_ising(q)
    ss = vxq.solve_pa(ising, vxq.PaParams(steps=1000, replicas=64, seed=11))
    for s in ss.samples[:8]:
        x = vxq.spins_to_bits(s.state).astype(np.float64)
        eq = float((x[q.rows] * x[q.cols]) @ q.values + q.offset)
        assert abs(eq - s.energy) <= 1e-11


# ---------------------------------------------------------------- BASELINE-shaped properties
def test_maxcut_scaled_cfg4_matches_oracle_subset():
    """3-regular MaxCut (cfg 4 family) at n = 2e4, R = 256: GPU replicas 0..7 equal the
    oracle's fp32 restatement bit for bit; cut = (|E| - H) / 2 is an integer."""
    m = maxcut_model(20_000, 3, 7)
    r = vxq.run_pa(m, vxq.PaParams(steps=40, replicas=256, seed=3), path="sparse",
                   want_state=True)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    X = O.pa_init(3, 8, m.n)
    X, M = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), 40), 0.05, 0.9, X,
                    np.zeros_like(X), np.float32)
    assert np.array_equal(r.x[:8], X.astype(np.float64))
    cut = (m.num_couplings - r.energies) / 2
    assert np.all(cut == np.round(cut))
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))


@pytest.mark.parametrize("R", [64, 256])
def test_sparse_sbm_wide_replicas_match_oracle_subset(R):
    """Sparse SBM step with several replicas per lane (R >= 64: the vector widths cfg 3/4
    run) equals the oracle's fp32 restatement bit for bit -- guards against any change
    that lets the compiler contract the in-order a*q products and sums into FMAs."""
    r_, c_ = random_regular_edges(20_000, 6, 7)
    rng = np.random.default_rng(11)
    m = vxq.IsingModel.from_arrays(20_000, r_, c_, rng.uniform(-1, 1, len(r_)),
                                   h=rng.uniform(-1, 1, 20_000), canonical=True)  # inexact a*q
    c0 = 0.3
    s = vxq.run_sbm(m, vxq.SbmParams(steps=40, dt=0.05, replicas=R, seed=4, c0=c0),
                    path="sparse", want_state=True)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q, P = O.sbm_init(4, 8, m.n, 1.0)
    Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, 40), 0.05, 1.0, c0, 1.0, Q, P,
                     np.float32)
    assert np.array_equal(s.x[:8], Q.astype(np.float64))
    assert np.array_equal(s.m[:8], P.astype(np.float64))


def test_sk_dense_family_matches_oracle_subset():
    m = sk_model(600, 2)
    r = vxq.run_pa(m, vxq.PaParams(steps=50, replicas=128, seed=1), path="sparse",
                   want_state=True)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    X = O.pa_init(1, 4, m.n)
    X, M = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), 50), 0.05, 0.9, X,
                    np.zeros_like(X), np.float32)
    assert np.array_equal(r.x[:4], X.astype(np.float64))
    assert np.array_equal(r.energies[:16], O.energies_exact(m, r.states[:16]))


def _dense_pa_emulation(m, R, T, seed):
    """numpy fp32 emulation of the tensor-core path: f = fp32(c) * fp32(K.s) (exact integer
    K.s), then the reference's update order with one rounding per op."""
    n = m.n
    K = np.zeros((n, n), dtype=np.int64)
    K[m.rows, m.cols] = np.sign(m.values).astype(np.int64)
    K[m.cols, m.rows] = np.sign(m.values).astype(np.int64)
    c = np.float32(np.abs(m.values[0]))
    X = O.pa_init(seed, R, n).astype(np.float32)
    M = np.zeros_like(X)
    h = m.h.astype(np.float32)
    eta, alpha = np.float32(0.05), np.float32(0.9)
    for lam in O.pa_schedule(O.resolve_lambda0(m), T).astype(np.float32):
        S = np.where(X >= 0, 1, -1).astype(np.int64)
        f = c * (S @ K.T).astype(np.float32)
        grad = (lam * X + f) + h
        M = alpha * M - eta * grad
        X = np.clip(X + M, np.float32(-1), np.float32(1))
    return X, M


@pytest.mark.parametrize("n,R", [(1000, 256), (700, 300), (2048, 512)])
def test_dense_tensor_core_path_bitexact_with_emulation(n, R):
    """SK (cfg 2 family): the tcgen05 path (auto-selected) equals the fp32 emulation bit for
    bit, including ragged n (not a multiple of 128) and ragged R (not a multiple of 256)."""
    m = sk_model(n, 3)
    r = vxq.run_pa(m, vxq.PaParams(steps=25, replicas=R, seed=4), want_state=True)
    assert r.info["path"] == "dense"
    X, M = _dense_pa_emulation(m, R, 25, 4)
    assert np.array_equal(r.x, X.astype(np.float64))
    assert np.array_equal(r.m, M.astype(np.float64))
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))


@pytest.mark.parametrize("planes", ["2", "3"])
@pytest.mark.parametrize("n,R", [(1000, 256), (700, 200)])
def test_dense_sbm_tensor_core_short_horizon(n, R, planes, monkeypatch):
    """SBM on the tensor cores (q as two fp16 terms -- the default -- or three exact bf16
    terms, f32 accumulation) tracks the fp64 restatement of the reference loop within the
    fp32 tolerance for t <= 30."""
    monkeypatch.setenv("VXQ_SBM_PLANES", planes)
    m = sk_model(n, 6)
    c0 = 0.02
    r = vxq.run_sbm(m, vxq.SbmParams(steps=30, dt=0.05, replicas=R, seed=2, c0=c0),
                    want_state=True)
    assert r.info["path"] == "dense"
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q, P = O.sbm_init(2, 8, m.n, 1.0)
    Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, 30), 0.05, 1.0, c0, 1.0, Q, P)
    assert np.abs(r.x[:8] - Q).max() <= 1e-4
    assert np.abs(r.m[:8] - P).max() <= 1e-4
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))
    s = vxq.run_sbm(m, vxq.SbmParams(steps=30, dt=0.05, replicas=R, seed=2, c0=c0),
                    path="sparse", want_state=True)
    assert np.abs(r.x - s.x).max() <= 1e-4


def test_dense_vs_sparse_same_dynamics_quality():
    m = sk_model(1024, 5)
    d = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=256, seed=1), path="dense")
    s = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=256, seed=1), path="sparse")
    # different (but both fp32-accurate) field roundings: same ensemble statistics
    assert abs(d.energies.mean() - s.energies.mean()) < 0.02 * abs(s.energies.mean())
    assert d.energies.min() / m.n < -0.7  # SK ground-state density ~ -0.763


@pytest.mark.parametrize("R", [1, 3, 32, 33, 64, 100, 129])
def test_ragged_replica_counts(R):
    m = gen_complete(17, 24, "gaussian")
    ref = vxq.run_pa(m, vxq.PaParams(steps=100, replicas=130, seed=2), precision="fp64",
                     want_state=True)
    for path in ("resident", "sparse"):
        r = vxq.run_pa(m, vxq.PaParams(steps=100, replicas=R, seed=2), precision="fp64",
                       path=path, want_state=True)
        assert np.array_equal(r.x, ref.x[:R]), (path, R)


def test_zero_coupling_model():
    m = vxq.IsingModel.from_terms(4)
    r = vxq.solve_pa(m, vxq.PaParams(steps=10, replicas=2, seed=0))
    assert r.best.energy == 0.0


# ---------------------------------------------------------------- improvement mode / trace
def _oracle_pa_states_per_step(m, R, T, seed, dtype=np.float32):
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    lam = O.pa_schedule(O.resolve_lambda0(m), T)
    X = O.pa_init(seed, R, m.n)
    M = np.zeros_like(X)
    states = [O.sign_pm(X)]
    for t in range(T):
        X, M = O.pa_run(ip, ix, dv, m.h, lam[t:t + 1], 0.05, 0.9, X, M, dtype)
        states.append(O.sign_pm(X))
    return states


def test_energy_trace_and_best_tracking_sparse_pa():
    m = gen_complete(44, 40, "uniform")
    R, T = 24, 30
    st = _oracle_pa_states_per_step(m, R, T, 6)
    E = np.array([O.energies_exact(m, s) for s in st])  # (T+1, R), exact
    r = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=6), trace=True, track_best=True)
    assert r.info["path"] == "sparse"
    assert np.array_equal(r.info["energy_trace"], E[:T].min(axis=1))
    assert np.array_equal(r.energies, E.min(axis=0))       # best over s_0..s_T, exact
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))
    plain = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=6))
    assert np.all(r.energies <= plain.energies)
    t, ms = vxq.solvers.time_to_target(r.info["energy_trace"], E.min() + 1e-9, 1.0)
    assert t is not None and E[: t + 1].min() <= E.min() + 1e-9


def test_energy_trace_sparse_sbm():
    m = gen_complete(45, 32, "gaussian")
    R, T = 16, 25
    r = vxq.run_sbm(m, vxq.SbmParams(steps=T, dt=0.05, replicas=R, seed=3, c0=0.2), trace=True,
                    track_best=True)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q, P = O.sbm_init(3, R, m.n, 1.0)
    a = O.sbm_schedule(1.0, T)
    E = [O.energies_exact(m, O.sign_pm(Q))]
    for t in range(T):
        Q, P = O.sbm_run(ip, ix, -dv, -m.h, a[t:t + 1], 0.05, 1.0, 0.2, 1.0, Q, P, np.float32)
        E.append(O.energies_exact(m, O.sign_pm(Q)))
    E = np.array(E)
    assert np.array_equal(r.info["energy_trace"], E[:T].min(axis=1))
    assert np.array_equal(r.energies, E.min(axis=0))


def test_energy_trace_dense_pa_exact():
    m = sk_model(700, 8)
    R, T = 200, 20
    r = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=2), trace=True)
    assert r.info["path"] == "dense"
    n = m.n
    K = np.zeros((n, n), dtype=np.int64)
    K[m.rows, m.cols] = np.sign(m.values).astype(np.int64)
    K[m.cols, m.rows] = np.sign(m.values).astype(np.int64)
    c = np.float32(np.abs(m.values[0]))
    X = O.pa_init(2, R, n).astype(np.float32)
    M = np.zeros_like(X)
    eta, alpha = np.float32(0.05), np.float32(0.9)
    want = []
    for lam in O.pa_schedule(O.resolve_lambda0(m), T).astype(np.float32):
        S = np.where(X >= 0, 1, -1).astype(np.int64)
        want.append(O.energies_exact(m, S.astype(np.int8)).min())
        f = c * (S @ K.T).astype(np.float32)
        grad = (lam * X + f) + m.h.astype(np.float32)
        M = alpha * M - eta * grad
        X = np.clip(X + M, np.float32(-1), np.float32(1))
    assert np.array_equal(r.info["energy_trace"], np.array(want))


@pytest.mark.parametrize("n,R,T", [(700, 300, 40), (1000, 256, 25)])
def test_dense_fused_best_tracking_matches_emulation(n, R, T):
    """track_best on the tcgen05 path (fused in the epilogue: exact integer energies of every
    s_t, t = 0..T, earliest minimum wins) == the fp32 emulation's best states."""
    m = sk_model(n, 11)
    r = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=8), track_best=True)
    assert r.info["path"] == "dense"
    K = np.zeros((n, n), dtype=np.int64)
    K[m.rows, m.cols] = np.sign(m.values).astype(np.int64)
    K[m.cols, m.rows] = np.sign(m.values).astype(np.int64)
    c = np.float32(np.abs(m.values[0]))
    X = O.pa_init(8, R, n).astype(np.float32)
    M = np.zeros_like(X)
    h = m.h.astype(np.float32)
    eta, alpha = np.float32(0.05), np.float32(0.9)
    best_q = np.full(R, np.iinfo(np.int64).max)
    best_S = np.zeros((R, n), dtype=np.int8)

    def observe(S):
        q = np.einsum("ri,ri->r", S, S @ K.T)
        imp = q < best_q
        best_q[imp] = q[imp]
        best_S[imp] = S[imp]

    for lam in O.pa_schedule(O.resolve_lambda0(m), T).astype(np.float32):
        S = np.where(X >= 0, 1, -1).astype(np.int64)
        observe(S)
        f = c * (S @ K.T).astype(np.float32)
        M = alpha * M - eta * ((lam * X + f) + h)
        X = np.clip(X + M, np.float32(-1), np.float32(1))
    observe(np.where(X >= 0, 1, -1).astype(np.int64))
    assert np.array_equal(r.states, best_S)
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))
    # improvement mode never reports worse than the final states
    plain = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=8))
    assert np.all(r.energies <= plain.energies)


@pytest.mark.parametrize("n", [384, 129, 1153])
def test_dense_pair_odd_row_tiles(n):
    """CTA-pair tiles (M = 256) with an odd number of 128-row tiles (the last pair's second
    CTA has no rows): still bit-exact with the fp32 emulation."""
    m = sk_model(n, 5)
    R = 256
    r = vxq.run_pa(m, vxq.PaParams(steps=12, replicas=R, seed=6), path="dense", want_state=True)
    assert r.info["path"] == "dense"
    X, M = _dense_pa_emulation(m, R, 12, 6)
    assert np.array_equal(r.x, X.astype(np.float64))
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))


@pytest.mark.parametrize("n,R", [(1000, 256), (700, 200)])
def test_dense_general_j_tensor_core_short_horizon(n, R):
    """General (non-uniform) dense J on the tensor cores: J as two fp16 planes of 2^e J
    (exact products with the +-1 spins, fp32 accumulation).  One step: within 2e-5 of the
    fp64 reference loop.  This family (complete graph, U[-1,1] couplings and biases,
    lambda0 ~ n/2) amplifies rounding from the first steps on -- the oracle's fp32 CSR
    restatement itself is 7e-4 from fp64 after 5 steps -- so after 5 steps the dense path
    must stay as close to fp64 as fp32 CSR does (99th percentile) and agree on the signs.
    Energies are exact."""
    m = gen_complete(21, n)  # the reference's complete/uniform family with biases
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    lam0 = O.resolve_lambda0(m)
    for T in (1, 5):
        r = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=5), want_state=True)
        assert r.info["path"] == "dense"
        assert np.array_equal(r.energies, O.energies_exact(m, r.states))
        X = O.pa_init(5, 8, m.n)
        X, M = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(lam0, T), 0.05, 0.9, X,
                        np.zeros_like(X))
        dd = np.abs(r.x[:8] - X)
        if T == 1:
            assert dd.max() <= 2e-5 and np.abs(r.m[:8] - M).max() <= 2e-5
            continue
        s = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=5), path="sparse",
                       want_state=True)
        ds = np.abs(s.x[:8] - X)
        assert np.quantile(dd, 0.99) <= 3 * np.quantile(ds, 0.99) + 1e-5
        assert np.mean(r.states == s.states) >= 0.999


def test_dense_general_j_quality_and_fallbacks():
    m = gen_complete(22, 1024)
    d = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=256, seed=1))
    s = vxq.run_pa(m, vxq.PaParams(steps=300, replicas=256, seed=1), path="sparse")
    assert d.info["path"] == "dense" and s.info["path"] == "sparse"
    assert abs(d.energies.mean() - s.energies.mean()) < 0.01 * abs(s.energies.mean())
    # per-step tracking is not fused for general J: auto falls back to the CSR path,
    # an explicit dense request is refused
    t = vxq.run_pa(m, vxq.PaParams(steps=20, replicas=128, seed=1), trace=True)
    assert t.info["path"] == "sparse"
    with pytest.raises(vxq.QubokitError):
        vxq.run_pa(m, vxq.PaParams(steps=20, replicas=128, seed=1), path="dense", trace=True)


@pytest.mark.parametrize("n,R", [(1000, 256), (700, 200)])
def test_dense_general_j_sbm_short_horizon(n, R):
    """SBM with a general dense J on the tensor cores (two fp16 J planes x two fp16 q planes,
    fp32 accumulation): one step within 2e-5 of the fp64 reference loop, ten steps as close
    to it as the fp32 CSR restatement (99th percentile); energies exact."""
    m = gen_complete(23, n)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    c0 = vxq.resolve_c0(m)
    for T in (1, 10):
        prm = vxq.SbmParams(steps=T, dt=0.05, replicas=R, seed=7, c0=c0)
        r = vxq.run_sbm(m, prm, want_state=True)
        assert r.info["path"] == "dense"
        assert np.array_equal(r.energies, O.energies_exact(m, r.states))
        Q, P = O.sbm_init(7, 8, m.n, 1.0)
        Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, T), 0.05, 1.0, c0, 1.0, Q, P)
        dq = np.abs(r.x[:8] - Q)
        if T == 1:
            assert dq.max() <= 2e-5 and np.abs(r.m[:8] - P).max() <= 2e-5
            continue
        s = vxq.run_sbm(m, prm, path="sparse", want_state=True)
        ds = np.abs(s.x[:8] - Q)
        assert np.quantile(dq, 0.99) <= 3 * np.quantile(ds, 0.99) + 1e-5
        assert np.mean(r.states == s.states) >= 0.999


def _random_pairs(n, density, seed):
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < density
    return rng, iu[keep], ju[keep]


def test_dense_paths_selected_at_moderate_density():
    """The tensor paths win far below full density (their cost does not depend on it), so
    auto selects them down to a few percent: a 3 % uniform-|J| instance runs the mxf4 path
    bit-exact with its fp32 emulation; a 10 % general-J instance runs the fp16-plane path
    (one step within 2e-5 of the fp64 reference loop)."""
    rng, iu, ju = _random_pairs(2048, 0.03, 31)
    J = np.where(rng.random(len(iu)) < 0.5, -0.25, 0.25)
    m = vxq.IsingModel.from_arrays(2048, iu, ju, J, h=rng.uniform(-1, 1, 2048), canonical=True)
    r = vxq.run_pa(m, vxq.PaParams(steps=25, replicas=256, seed=4), want_state=True)
    assert r.info["path"] == "dense"
    X, M = _dense_pa_emulation(m, 256, 25, 4)
    assert np.array_equal(r.x, X.astype(np.float64)) and np.array_equal(r.m, M.astype(np.float64))
    assert np.array_equal(r.energies, O.energies_exact(m, r.states))

    rng, iu, ju = _random_pairs(1024, 0.10, 32)
    g = vxq.IsingModel.from_arrays(1024, iu, ju, rng.standard_normal(len(iu)),
                                   h=rng.standard_normal(1024), canonical=True)
    rg = vxq.run_pa(g, vxq.PaParams(steps=1, replicas=128, seed=6), want_state=True)
    assert rg.info["path"] == "dense"
    ip, ix, dv = O.symmetric_csr(g.n, g.rows, g.cols, g.values)
    Xg, Mg = O.pa_run(ip, ix, dv, g.h, O.pa_schedule(O.resolve_lambda0(g), 1), 0.05, 0.9,
                      O.pa_init(6, 8, g.n), np.zeros((8, g.n)))
    assert np.abs(rg.x[:8] - Xg).max() <= 2e-5
    assert np.array_equal(rg.energies, O.energies_exact(g, rg.states))


def test_dense_sbm_fp16_range_fallbacks():
    """|q| may leave the fp16 range (q_cap or init_noise beyond 2^14): the SK tensor path
    then splits q into three exact bf16 planes, and general dense J (fp16 J and q planes
    only) falls back to the CSR path -- both still track the fp64 restatement."""
    m = sk_model(700, 6)
    prm = vxq.SbmParams(steps=5, dt=0.05, replicas=200, seed=2, c0=0.02, q_cap=1e5)
    r = vxq.run_sbm(m, prm, want_state=True)
    assert r.info["path"] == "dense"
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q, P = O.sbm_init(2, 8, m.n, 1.0)
    Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, 5), 0.05, 1.0, 0.02, 1e5, Q, P)
    assert np.abs(r.x[:8] - Q).max() <= 1e-4
    g = gen_complete(24, 600)
    rg = vxq.run_sbm(g, vxq.SbmParams(steps=5, dt=0.05, replicas=128, seed=3, c0=0.01,
                                      init_noise=3e4), want_state=True)
    assert rg.info["path"] == "sparse"
    assert np.array_equal(rg.energies, O.energies_exact(g, rg.states))


@pytest.mark.parametrize("group", ["2", "3"])
def test_dense_tile_order_does_not_change_results(group, monkeypatch):
    """The dense kernels' tile order (replica blocks grouped per row panel, the last group
    possibly smaller; the dynamic tile queue hands tiles out in that order) changes when
    tiles run, never what they compute: PA and exact-field SBM are bit-identical to the
    default order."""
    m = sk_model(1000, 12)
    pa = vxq.PaParams(steps=15, replicas=1024, seed=3)
    sb = vxq.SbmParams(steps=15, dt=0.05, replicas=400, seed=3, c0=0.4)
    ref_pa = vxq.run_pa(m, pa, want_state=True)
    ref_sb = vxq.run_sbm(m, sb, want_state=True)
    monkeypatch.setenv("VXQ_DENSE_GROUP", group)
    r_pa = vxq.run_pa(m, pa, want_state=True)
    r_sb = vxq.run_sbm(m, sb, want_state=True)
    assert r_pa.info["path"] == "dense" and r_sb.info["dense_kind"] == "i8x3"
    assert np.array_equal(r_pa.x, ref_pa.x) and np.array_equal(r_pa.m, ref_pa.m)
    assert np.array_equal(r_sb.x, ref_sb.x) and np.array_equal(r_sb.m, ref_sb.m)


def test_sparse_sbm_r32_irregular_rows_match_oracle():
    """R = 32 (config 5's replica count, one q vector per row): bit-exact with the oracle's
    fp32 loop on an irregular graph with one row of 80+ neighbours."""
    rng = np.random.default_rng(21)
    n = 4000
    r_, c_ = random_regular_edges(n, 6, 3)
    extra_r = np.zeros(80, dtype=np.int64)  # row 0 gets 80 extra neighbours
    extra_c = np.arange(1, 81, dtype=np.int64)
    rows = np.r_[r_, extra_r]
    cols = np.r_[c_, extra_c]
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    m = vxq.IsingModel.from_arrays(n, rows, cols, rng.uniform(-1, 1, len(rows)),
                                   h=rng.uniform(-1, 1, n), canonical=True)
    s = vxq.run_sbm(m, vxq.SbmParams(steps=30, dt=0.05, replicas=32, seed=2, c0=0.3),
                    path="sparse", want_state=True)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q, P = O.sbm_init(2, 32, m.n, 1.0)
    Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, 30), 0.05, 1.0, 0.3, 1.0, Q, P,
                     np.float32)
    assert np.array_equal(s.x, Q.astype(np.float64)) and np.array_equal(s.m, P.astype(np.float64))


def test_dense_model_values_only_upload_is_identical(monkeypatch):
    """A full-upper-triangle model crosses PCIe as values only (indices generated on the
    device by vxq_problem_create): problem, lambda0, c0 and PA / SBM solves equal those of
    the explicit-index upload bit for bit."""
    from paper_2501_19221_b200 import device
    rng = np.random.default_rng(3)
    n = 700
    iu, ju = np.triu_indices(n, 1)
    m = vxq.IsingModel.from_arrays(n, iu, ju, rng.normal(size=len(iu)) / np.sqrt(n),
                                   h=rng.uniform(-1, 1, n), canonical=True)
    assert device.full_triangle(n, m.rows, m.cols)

    def solve(model):
        dp = device.DeviceProblem(model)
        info = dp.info()
        lam, c0 = dp.lambda0(), dp.c0()
        r = vxq.run_pa(model, vxq.PaParams(steps=30, replicas=128, seed=1), want_state=True,
                       cache=False)
        s = vxq.run_sbm(model, vxq.SbmParams(steps=30, dt=0.05, replicas=128, seed=1),
                        want_state=True, cache=False)
        return info, lam, c0, r, s

    a = solve(m)
    monkeypatch.setattr(device, "full_triangle", lambda *args: False)
    b = solve(m)
    assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]
    for ra, rb in ((a[3], b[3]), (a[4], b[4])):
        assert np.array_equal(ra.x, rb.x) and np.array_equal(ra.energies, rb.energies)
        assert np.array_equal(ra.states, rb.states)
