"""Sparse SBM on the row-block kernel (k_sbm_block, dynamics.cu): one CTA stages the q_t chunk
rows of a 64-row block's distinct neighbours and the block's CSR entries in shared memory
and sums its rows from there (info["kernel"] reports which step kernel ran, ABI 5).
Per (row, replica) it performs the reference's operations (bifurcation.py:40-46) in CSR
order, so it must equal the step kernel bit for bit and the oracle's fp32 restatement --
on the benchmarked cfg 3 shape, on ragged row counts / replica counts, with rows longer
than the 4-entry batches, isolated rows, and with a per-step energy trace.
"""

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from paper_2501_19221_b200 import instances

pytestmark = pytest.mark.gpu


def banded(n, width, seed, isolated=()):
    """Couplings within a band of `width` around the diagonal (neighbour reuse between
    consecutive rows, like the Pegasus numbering); J, h ~ U[-1, 1]."""
    rng = np.random.default_rng(seed)
    i = np.repeat(np.arange(n), width)
    j = i + rng.integers(1, 3 * width, len(i))
    keep = (j < n) & ~np.isin(i, isolated) & ~np.isin(j, isolated)
    key = np.unique(i[keep] * n + j[keep])
    i, j = key // n, key % n
    return vxq.IsingModel.from_arrays(n, i, j, rng.uniform(-1, 1, len(i)),
                                      h=rng.uniform(-1, 1, n), canonical=True)


def run(monkeypatch, m, R, T, mode, c0=0.3, seed=5, trace=False):
    monkeypatch.setenv("VXQ_SBM_BLOCK", str(mode))
    r = vxq.run_sbm(m, vxq.SbmParams(steps=T, dt=0.05, replicas=R, seed=seed, c0=c0),
                    path="sparse", want_state=True, cache=False, trace=trace)
    return r, r.info["kernel"]


def oracle_rows(m, reps, T, c0, seed):
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q = np.stack([O.uniform(seed, int(r), 0, m.n, -1.0, 1.0) for r in reps])
    P = np.stack([O.uniform(seed, int(r), m.n, m.n, -1.0, 1.0) for r in reps])
    return O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, T), 0.05, 1.0, c0, 1.0, Q, P,
                     np.float32)


@pytest.mark.parametrize("n,width,R", [
    (3000, 8, 256),     # 47 blocks, the last ragged (56 rows)
    (1000, 20, 100),    # ragged replica count (R_pad = 128), rows of up to ~40 entries
    (4097, 4, 32),      # one chunk, n = 64 k + 1
])
def test_block_kernel_equals_step_kernel_and_oracle(monkeypatch, n, width, R):
    m = banded(n, width, seed=n, isolated=(5, 6, n - 2))
    T = 25
    a, ea = run(monkeypatch, m, R, T, mode=2)
    b, eb = run(monkeypatch, m, R, T, mode=0)
    assert ea == "k_sbm_block" and eb == "k_sbm_step"
    assert np.array_equal(a.x, b.x) and np.array_equal(a.m, b.m)
    assert np.array_equal(a.energies, b.energies) and np.array_equal(a.states, b.states)
    reps = np.unique(np.r_[0, 1, R // 2, R - 1])
    Q, P = oracle_rows(m, reps, T, 0.3, 5)
    assert np.array_equal(a.x[reps], Q.astype(np.float64))
    assert np.array_equal(a.m[reps], P.astype(np.float64))
    assert np.array_equal(a.energies[reps], O.energies_exact(m, a.states[reps]))


def test_block_kernel_trace(monkeypatch):
    m = banded(2048, 10, seed=3)
    a, ea = run(monkeypatch, m, 512, 20, mode=2, trace=True)
    b, _ = run(monkeypatch, m, 512, 20, mode=0, trace=True)
    assert ea == "k_sbm_block"
    assert np.array_equal(a.info["energy_trace"], b.info["energy_trace"])
    assert np.array_equal(a.x, b.x)


def test_cfg3_block_mode_auto_eligibility(monkeypatch):
    """cfg 3 as benchmarked (Pegasus P16, R = 4096): VXQ_SBM_BLOCK=1 finds the neighbour
    reuse (~3 entries per staged row) and picks the block kernel, which equals the step
    kernel (the default) and the oracle."""
    m = instances.build("cfg3")
    R, T = 4096, 12
    monkeypatch.delenv("VXQ_SBM_BLOCK", raising=False)
    d = vxq.run_sbm(m, vxq.SbmParams(steps=T, dt=0.05, replicas=R, seed=5, c0=0.3),
                    want_state=True, cache=False)
    assert d.info["kernel"] == "k_sbm_step"
    a, ea = run(monkeypatch, m, R, T, mode=1)
    assert ea == "k_sbm_block", ea
    assert np.array_equal(a.x, d.x) and np.array_equal(a.m, d.m)
    reps = np.r_[0:4, R - 4:R]
    Q, P = oracle_rows(m, reps, T, 0.3, 5)
    assert np.array_equal(a.x[reps], Q.astype(np.float64))


def test_random_graph_keeps_step_kernel(monkeypatch):
    """No neighbour reuse (random 3-regular-like graph): auto stays on k_sbm_step."""
    rng = np.random.default_rng(0)
    n = 20_000
    i = rng.integers(0, n, 3 * n)
    j = rng.integers(0, n, 3 * n)
    keep = i != j
    key = np.unique(np.minimum(i, j)[keep] * n + np.maximum(i, j)[keep])
    m = vxq.IsingModel.from_arrays(n, key // n, key % n, np.ones(len(key)), canonical=True)
    _, e = run(monkeypatch, m, 256, 3, mode=1)
    assert e == "k_sbm_step"
