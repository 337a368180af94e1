"""GPU simulated annealing (annealing.py:24-74) through the C-ABI, against the reference's
golden vectors (tests/golden/reference_sa.npz) and the oracle's restatement.

Tolerances: fp64 mode reproduces the reference's best state of every replica (one
rounding per numpy operation; CUDA's exp is within an ulp of numpy's, which can flip an
acceptance only if the uniform lands inside that ulp -- not hit on these seeds).  fp32
mode (fields in fp32) is bit-exact against the oracle's fp32 restatement.  Energies are
the correctly rounded exact sums (oracle.energy_exact).
"""

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from helpers import brute_force_min, gen_complete, model_from_golden

pytestmark = pytest.mark.gpu

SA_CASES = ("int20", "csr2100", "dense40")


def _params(g, case, **kw):
    return vxq.SaParams(sweeps=int(g[f"{case}_sweeps"]), replicas=int(g[f"{case}_replicas"]),
                        seed=int(g[f"{case}_seed"]), **kw)


def _by_replica(ss, n):
    st = np.zeros((ss.replica_count, n), dtype=np.int8)
    en = np.zeros(ss.replica_count)
    for s in ss.samples:
        st[s.replica] = s.state
        en[s.replica] = s.energy
    return st, en


# the resident path keeps a warp's fields in shared memory: n (32 * 8 + 8) bytes in fp64
SA_PATHS = [(c, p) for c in SA_CASES for p in ("resident", "sparse")
            if not (c == "csr2100" and p == "resident")]


@pytest.mark.parametrize("case,path", SA_PATHS)
def test_sa_fp64_reproduces_reference(golden_sa, case, path):
    g = golden_sa
    m = model_from_golden(g, case)
    ss = vxq.solve_sa(m, _params(g, case), precision="fp64", path=path)
    assert ss.info["path"] == path
    st, en = _by_replica(ss, m.n)
    assert np.array_equal(st, g[f"{case}_states"])
    assert np.array_equal(en, O.energies_exact(m, st))
    # best-first, ties by replica (common.py:57)
    E = ss.energies()
    assert np.all(np.diff(E) >= 0)


@pytest.mark.parametrize("case", ["csr2100", "dense40"])
def test_sa_fp32_bitexact_with_oracle(golden_sa, case):
    g = golden_sa
    m = model_from_golden(g, case)
    best, _ = O.sa_solve(m, int(g[f"{case}_sweeps"]), replicas=int(g[f"{case}_replicas"]),
                         seed=int(g[f"{case}_seed"]), dtype=np.float32)
    for path in (("sparse",) if case == "csr2100" else ("resident", "sparse")):
        r = vxq.run_sa(m, _params(g, case), path=path)
        assert np.array_equal(r.states, best), path
    if case == "csr2100":  # too large for the resident path: explicit request fails loudly
        with pytest.raises(vxq.QubokitError):
            vxq.run_sa(m, _params(g, case), path="resident", precision="fp64")


def test_sa_ragged_replicas_and_sharding_match_oracle():
    """R = 40 (padded to 64), replica_begin offsets, on a Pegasus P4 instance."""
    from paper_2501_19221_b200 import instances
    m = instances.pegasus(4, seed=21)
    p = vxq.SaParams(sweeps=50, replicas=40, seed=9)
    full = vxq.run_sa(m, p, precision="fp64", path="sparse")
    best, _ = O.sa_solve(m, 50, replicas=5, seed=9, replica_begin=17)
    assert np.array_equal(full.states[17:22], best)
    part = vxq.run_sa(m, vxq.SaParams(sweeps=50, replicas=5, seed=9), precision="fp64",
                      replica_begin=17)
    assert np.array_equal(part.states, best)
    assert np.array_equal(part.energies, full.energies[17:22])


def test_sa_determinism_and_paths_agree():
    m = gen_complete(4, 60, dist="uniform")
    p = vxq.SaParams(sweeps=200, replicas=96, seed=1)
    a = vxq.run_sa(m, p, path="resident")
    b = vxq.run_sa(m, p, path="resident")
    c = vxq.run_sa(m, p, path="sparse")
    assert np.array_equal(a.states, b.states) and np.array_equal(a.states, c.states)
    assert np.array_equal(a.energies, c.energies)


def test_sa_finds_brute_force_minimum():
    """test_solvers.py:38-43 restated: >= 9 of 10 instances reach the exact minimum."""
    hits = 0
    for seed in range(10):
        m = gen_complete(100 + seed, 12, dist="uniform")
        ss = vxq.solve_sa(m, vxq.SaParams(sweeps=500, replicas=32, seed=seed))
        hits += abs(ss.best.energy - brute_force_min(m)) <= 1e-9
    assert hits >= 9


def test_sa_explicit_temperatures_and_schedule():
    m = gen_complete(3, 30, dist="int_uniform", a=-2, b=2)
    p = vxq.SaParams(sweeps=64, T_init=5.0, T_final=0.01, replicas=32, seed=4)
    r = vxq.run_sa(m, p, precision="fp64")
    assert r.info["T_init"] == 5.0 and r.info["T_final"] == 0.01
    best, _ = O.sa_solve(m, 64, T_init=5.0, T_final=0.01, replicas=32, seed=4)
    assert np.array_equal(r.states, best)
    one = vxq.run_sa(m, vxq.SaParams(sweeps=1, replicas=32, seed=4), precision="fp64")
    b1, _ = O.sa_solve(m, 1, replicas=32, seed=4)
    assert np.array_equal(one.states, b1)
