"""The reference's acceptance criteria that touch the path, against the unmodified
reference's own outputs (tests/golden/make_golden_acceptance.py), through the C-ABI.

#8 (test_acceptance.py:220-235): 1024-replica PA on random n = 100, 1000 steps: sorted
   sample set, spectrum whose lowest bin holds the best sample -- and here, beyond the
   reference's test, the per-replica final states compared with the reference's own.
#9 (test_acceptance.py:238-255): on five n = 50 integer instances the best of 1024-replica
   SA and PA equals the exact optimum of the reference's branch and bound (0 % gap).
"""

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from helpers import model_from_golden
from paper_2501_19221_b200.harness import spectrum

pytestmark = pytest.mark.gpu


def _by_replica(ss, n):
    states = np.zeros((ss.replica_count, n), dtype=np.int8)
    for s in ss.samples:
        states[s.replica] = s.state
    return states


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_criterion_08_spectrum_and_reference_states(golden_acc, precision):
    g = golden_acc
    m = model_from_golden(g, "c8")
    ss = vxq.solve_pa(m, vxq.PaParams(steps=1000, replicas=1024, seed=8), precision=precision)
    assert len(ss) == 1024
    e = ss.energies()
    assert np.all(np.diff(e) >= 0)
    edges, counts = spectrum(ss, bins=32)
    assert counts.sum() == 1024
    assert edges[0] <= ss.best.energy <= edges[1] and counts[0] >= 1
    # the reference's final states, replica by replica (its dense BLAS field sums differ
    # from the CSR order by ulps, so a replica sitting on a sign decision may differ)
    st = _by_replica(ss, m.n)
    same = np.all(st == g["c8_states"], axis=1)
    print(f"{precision}: {same.sum()}/1024 final states equal the reference's")
    assert same.mean() >= 0.98
    # energies are the correctly rounded exact sums; the reference's BLAS-ordered ones
    # are within a few ulps
    ex = O.energies_exact(m, g["c8_states"])
    assert np.all(np.abs(ex - g["c8_energies"]) <= 1e-12 * np.abs(ex).max())
    assert ss.best.energy <= ex.min() + 1e-9


@pytest.mark.parametrize("k", range(5))
def test_criterion_09_best_of_1024_equals_branch_and_bound(golden_acc, k):
    g = golden_acc
    m = model_from_golden(g, f"c9_{k}")
    bb = float(g[f"c9_{k}_bb_energy"])
    sa = vxq.solve_sa(m, vxq.SaParams(sweeps=1000, replicas=1024, seed=k)).best.energy
    pa = vxq.solve_pa(m, vxq.PaParams(steps=1000, replicas=1024, seed=k)).best.energy
    assert min(sa, pa) == bb
    # integer instance: every energy is exact, so equal-or-better than the reference's
    assert sa <= float(g[f"c9_{k}_sa_best"]) and pa <= float(g[f"c9_{k}_pa_best"])
