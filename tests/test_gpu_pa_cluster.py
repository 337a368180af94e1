"""PA on the thread-block-cluster kernel (k_pa_cluster, dynamics.cu): every CTA of a cluster
holds one replica chunk's spin words of all n rows in shared memory, the cluster runs all
T steps in one launch.  Its per-(row, replica) arithmetic and CSR order are those of the
step kernel (parallel_annealing.py:41-45), so both must agree bit for bit, and with the
oracle's fp32 / fp64 restatement -- across chunk widths V = 1, 2, 4, cluster sizes C = 1..8,
ragged row splits, ragged last chunks (R < R_pad), rows longer than the 32-entry
lane-parallel CSR batch, and the per-step launch mode used when a trace is requested.
"""

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from paper_2501_19221_b200 import instances

pytestmark = pytest.mark.gpu


def random_sparse(n, deg, seed, hubs=0, hub_deg=0):
    """Random couplings J, h ~ U[-1, 1]; `hubs` rows get `hub_deg` extra neighbours."""
    rng = np.random.default_rng(seed)
    a = rng.integers(0, n, n * deg // 2)
    b = rng.integers(0, n, n * deg // 2)
    if hubs:
        hh = rng.integers(0, n, hubs).repeat(hub_deg)
        a = np.r_[a, hh]
        b = np.r_[b, rng.integers(0, n, len(hh))]
    keep = a != b
    i, j = np.minimum(a[keep], b[keep]), np.maximum(a[keep], b[keep])
    key = np.unique(i * n + j)
    i, j = key // n, key % n
    return vxq.IsingModel.from_arrays(n, i, j, rng.uniform(-1, 1, len(i)),
                                      h=rng.uniform(-1, 1, n), canonical=True)


def run(monkeypatch, m, R, T, mode, C=None, precision="fp32", trace=False, seed=3):
    monkeypatch.setenv("VXQ_PA_CLUSTER", str(mode))
    if C is None:
        monkeypatch.delenv("VXQ_PA_CLUSTER_C", raising=False)
    else:
        monkeypatch.setenv("VXQ_PA_CLUSTER_C", str(C))
    return vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=seed), path="sparse",
                      precision=precision, want_state=True, trace=trace)


@pytest.mark.parametrize("n,R,C,deg,hubs", [
    (3001, 4096, 3, 12, 0),    # V = 4, 32 chunks, ragged 3-way row split
    (1000, 100, 1, 8, 0),      # one ragged chunk (R_pad = 128), one CTA
    (2500, 64, 5, 10, 0),      # V = 2, five CTAs
    (777, 20, 8, 6, 0),        # V = 1 (R <= 32), eight CTAs of ~97 rows
    (2000, 2048, 4, 6, 20),    # hub rows with > 32 and > 64 entries
])
def test_cluster_equals_step_kernel_and_oracle(monkeypatch, n, R, C, deg, hubs):
    m = random_sparse(n, deg, seed=n, hubs=hubs, hub_deg=90)
    T = 25
    a = run(monkeypatch, m, R, T, mode=2, C=C)
    b = run(monkeypatch, m, R, T, mode=0)
    assert a.info["launches"] < b.info["launches"] - T + 5, "cluster kernel did not run"
    assert a.info["kernel"] == "k_pa_cluster"
    assert b.info["kernel"] == ("k_pa_step_coop" if R <= 32 else "k_pa_step")
    assert np.array_equal(a.x, b.x) and np.array_equal(a.m, b.m)
    assert np.array_equal(a.states, b.states) and np.array_equal(a.energies, b.energies)
    reps = np.unique(np.r_[0, 1, R // 2, R - 1])
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    X = np.stack([O.uniform(3, int(r), 0, n, -1.0, 1.0) for r in reps])
    X, M = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), T), 0.05, 0.9, X,
                    np.zeros_like(X), np.float32)
    assert np.array_equal(a.x[reps], X.astype(np.float64))
    assert np.array_equal(a.m[reps], M.astype(np.float64))
    assert np.array_equal(a.energies[reps], O.energies_exact(m, a.states[reps]))


def test_cluster_fp64_bitexact_with_oracle(monkeypatch):
    """fp64 parity mode (V = 2 chunks of 64 replicas) on the cluster kernel."""
    m = random_sparse(1500, 10, seed=7)
    R, T = 256, 15
    a = run(monkeypatch, m, R, T, mode=2, C=2, precision="fp64")
    b = run(monkeypatch, m, R, T, mode=0, precision="fp64")
    assert a.info["launches"] < b.info["launches"]
    assert np.array_equal(a.x, b.x) and np.array_equal(a.m, b.m)
    reps = np.array([0, 63, 64, 255])
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    X, M = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), T), 0.05, 0.9,
                    np.stack([O.uniform(3, int(r), 0, m.n, -1.0, 1.0) for r in reps]),
                    np.zeros((len(reps), m.n)))
    assert np.array_equal(a.x[reps], X) and np.array_equal(a.m[reps], M)


def test_cluster_trace_mode_per_step_launches(monkeypatch):
    """With an energy trace the cluster kernel runs one step per launch (the tracker reads
    s_t between steps): trace, states and analog state equal the step kernel's."""
    m = random_sparse(2048, 8, seed=11)
    R, T = 1024, 20
    a = run(monkeypatch, m, R, T, mode=2, C=8, trace=True)
    b = run(monkeypatch, m, R, T, mode=0, trace=True)
    assert np.array_equal(a.info["energy_trace"], b.info["energy_trace"])
    assert np.array_equal(a.x, b.x) and np.array_equal(a.states, b.states)


def test_cfg3_cluster_mode_auto_eligibility(monkeypatch):
    """cfg 3 as benchmarked (Pegasus P16, R = 4096): VXQ_PA_CLUSTER=1 picks the cluster
    kernel (32 chunks x 4 CTAs) and matches the step kernel, which stays the default."""
    m = instances.build("cfg3")
    T = 10
    monkeypatch.delenv("VXQ_PA_CLUSTER_C", raising=False)
    monkeypatch.delenv("VXQ_PA_CLUSTER", raising=False)
    d = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=4096, seed=0), want_state=True)
    assert d.info["path"] == "sparse" and d.info["launches"] >= T
    assert d.info["kernel"] == "k_pa_step"
    a = run(monkeypatch, m, 4096, T, mode=1, seed=0)
    assert a.info["launches"] < T and a.info["kernel"] == "k_pa_cluster"
    assert np.array_equal(a.x, d.x) and np.array_equal(a.m, d.m)
