"""Automatic c0 = 1 / lambda_max(-A) (bifurcation.py:25-34 -> eig_extreme(-A, "max"),
solvers/eigen.py:35-56) on the device, against the UNMODIFIED reference's resolve_c0 at the
benchmarked sizes (tests/golden/reference_c0.npz, make_golden_c0.py):

  * n <= 512: the reference's exact eigvalsh value; the device runs Lanczos with full
    reorthogonalisation to the full dimension -> rel <= 1e-12.
  * n > 512: the reference returns ARPACK's theta + ||B v - theta v|| (tol 1e-8); the
    device returns its Lanczos theta + the explicit residual of its Ritz vector at the
    same tol -> both are within ~1e-8 relative of lambda_max: rel <= 1e-7.
  * no convergence: the Gershgorin bound (eigen.py:21-32, 49-52).
"""

import os

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from paper_2501_19221_b200 import instances
from paper_2501_19221_b200.device import get_problem

pytestmark = pytest.mark.gpu

GOLDEN_C0 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                         "reference_c0.npz")

CASES = {
    "maxcut3_1e5": lambda: instances.maxcut3(100_000),
    "maxcut3_1e6": lambda: instances.maxcut3(1_000_000),
    "pegasus16": lambda: instances.pegasus(),
    "sk_1000": lambda: instances.sk(1000),
    "sk_400": lambda: instances.sk(400),
    "cfg1": lambda: instances.cfg1_qubo()[1],
}


@pytest.fixture(scope="module")
def golden_c0():
    return dict(np.load(GOLDEN_C0))


@pytest.mark.parametrize("name", sorted(CASES))
def test_c0_matches_reference(golden_c0, name):
    m = CASES[name]()
    c0 = vxq.resolve_c0(m)
    ref = float(golden_c0[f"{name}_c0"])
    info = get_problem(m).eig_info()
    if m.n <= 512:
        assert info["method"] == "dense-exact"
        assert c0 == pytest.approx(ref, rel=1e-12)
        assert c0 == pytest.approx(O.resolve_c0(m), rel=1e-12)
    else:
        assert info["method"] == "lanczos"
        # the residual push-out: lambda = theta + ||B y - theta y||, never below theta
        assert info["residual"] >= 0 and info["lambda_max"] == info["theta"] + info["residual"]
        assert info["residual"] <= 1e-7 * abs(info["theta"])
        assert c0 == pytest.approx(ref, rel=1e-7)
    assert c0 == info["c0"]


def test_c0_dense_exact_equals_eigvalsh_small():
    """n <= 512 on irregular spectra (random weights, disconnected parts)."""
    rng = np.random.default_rng(7)
    for n in (2, 3, 17, 200, 512):
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(len(iu)) < 0.3
        keep[0] = True
        m = vxq.IsingModel.from_arrays(n, iu[keep], ju[keep], rng.normal(size=keep.sum()),
                                       canonical=True)
        assert vxq.resolve_c0(m) == pytest.approx(O.resolve_c0(m), rel=1e-12), n


def test_c0_gershgorin_fallback(monkeypatch):
    """ArpackNoConvergence -> Gershgorin (eigen.py:49-52): max_i sum_j |A_ij|."""
    monkeypatch.setenv("VXQ_LANCZOS_MAXITER", "20")
    m = instances.maxcut3(20_000, seed=11)
    c0 = vxq.resolve_c0(m)
    info = get_problem(m).eig_info()
    assert info["method"] == "gershgorin"
    deg = np.bincount(np.r_[m.rows, m.cols], minlength=m.n)
    assert info["lambda_max"] == float(deg.max())
    assert c0 == 1.0 / deg.max()


def test_c0_sbm_solve_uses_it():
    m = instances.maxcut3(100_000)
    s = vxq.run_sbm(m, vxq.SbmParams(steps=3, dt=0.05, replicas=32, seed=0))
    assert s.info["c0"] == vxq.resolve_c0(m)


def test_c0_dense_int8_spmv_matches_csr_spmv(monkeypatch):
    """Dense uniform-|J| problems run the Lanczos SpMV over an int8 K (n^2 bytes) instead of
    the CSR (12 bytes per entry): the returned c0 agrees with the CSR-SpMV value and with
    the exact lambda_max of -A (numpy eigvalsh) to the ARPACK-level tolerance."""
    n = 2500
    m = instances.sk(n)
    a = get_problem(m, cache=False).c0()
    monkeypatch.setenv("VXQ_EIG_DENSE", "0")
    b = get_problem(m, cache=False).c0()
    A = np.zeros((n, n))
    A[m.rows, m.cols] = m.values
    A[m.cols, m.rows] = m.values
    lam = np.linalg.eigvalsh(-A)[-1]
    assert abs(a - b) <= 1e-7 * abs(b)
    assert abs(1.0 / a - lam) <= 1e-7 * abs(lam)
