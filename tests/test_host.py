"""Host logic on CPU: QUBO-in conversion, canonicalisation, spin maps, SampleSet assembly."""

import numpy as np
import pytest

import paper_2501_19221_b200 as vxq
from helpers import model_from_golden


def test_qubo_to_ising_bitexact_with_reference(golden):
    q = vxq.QuboModel(n=int(golden["cfg1_n"]), rows=golden["cfg1_qubo_rows"],
                      cols=golden["cfg1_qubo_cols"], values=golden["cfg1_qubo_values"])
    m = vxq.qubo_to_ising(q)
    ref = model_from_golden(golden, "cfg1")
    for f in ("rows", "cols", "values", "h"):
        assert np.array_equal(getattr(m, f), getattr(ref, f)), f
    assert m.offset == ref.offset


def test_qubo_ising_energy_identity_small():
    # all 2^8 states: QUBO energy == Ising energy (transforms.py:36-41)
    rng = np.random.default_rng(4)
    n = 8
    iu, ju = np.triu_indices(n, 0)
    q = vxq.QuboModel.from_arrays(n, iu, ju, rng.uniform(-1, 1, len(iu)), offset=0.25)
    m = vxq.qubo_to_ising(q)
    bits = ((np.arange(2 ** n)[:, None] >> np.arange(n)) & 1).astype(np.float64)
    Eq = (bits[:, q.rows] * bits[:, q.cols]) @ q.values + q.offset
    S = 2 * bits - 1
    Ei = (S[:, m.rows] * S[:, m.cols]) @ m.values + S @ m.h + m.offset
    assert np.allclose(Eq, Ei, atol=1e-12)


def test_canonical_pairs_sums_duplicates_in_order():
    m = vxq.IsingModel.from_terms(4, couplings=[(2, 0, 0.1), (0, 2, 0.2), (1, 3, -1.0),
                                                (0, 2, 0.3)])
    assert m.rows.tolist() == [0, 1] and m.cols.tolist() == [2, 3]
    assert m.values[0] == (0.0 + 0.1 + 0.2) + 0.3
    assert not m.values.flags.writeable


def test_spin_maps():
    s = np.array([1, -1, 1])
    assert vxq.spins_to_bits(s).tolist() == [1, 0, 1]
    assert vxq.bits_to_spins([1, 0, 1]).tolist() == [1, -1, 1]
    assert vxq.sign_pm(np.array([0.0, -0.0, -1e-300, 2.0])).tolist() == [1, 1, -1, 1]
    with pytest.raises(vxq.ValidationError):
        vxq.as_spins([0, 1])


def test_sampleset_assembly_is_stable_best_first():
    from paper_2501_19221_b200.solvers import RunResult, sampleset_from
    E = np.array([1.0, -2.0, 1.0, -2.0, 0.5])
    order = np.argsort(E, kind="stable")
    st = np.arange(10, dtype=np.int8).reshape(5, 2)
    ss = sampleset_from(RunResult(st, E, order, None, None, {}), 5, 7, 0.1, replica_begin=0)
    assert [s.replica for s in ss.samples] == [1, 3, 4, 0, 2]
    assert ss.best.energy == -2.0 and len(ss) == 5 and ss.seed == 7
    assert np.all(np.diff(ss.energies()) >= 0)


def test_replica_streams_match_reference_layout():
    g = vxq.replica_streams(123, 3)
    bg = np.random.Philox(key=np.uint64(123)).jumped(2)
    assert np.array_equal(g[2].uniform(-1, 1, 5), np.random.Generator(bg).uniform(-1, 1, 5))


def test_harness_gap_and_spectrum_mirror_reference():
    from paper_2501_19221_b200 import harness
    assert harness.optimality_gap(-9.0, -10.0) == pytest.approx(0.1)
    assert harness.optimality_gap(-11.0, -10.0) == pytest.approx(-0.1)
    with pytest.raises(vxq.ValidationError):
        harness.optimality_gap(1.0, 0.0)
    e, c = harness.spectrum(np.array([1.0, 2.0, 2.0, 4.0]), 3)
    assert c.sum() == 4 and e[0] == 1.0 and e[-1] == 4.0
    e, c = harness.spectrum(np.array([3.0, 3.0]), 5)
    assert list(c) == [2]
    with pytest.raises(vxq.ValidationError):
        harness.spectrum(np.array([]), 2)


def test_use_in_reference_patches_every_lookup(monkeypatch):
    import sys
    import types
    from paper_2501_19221_b200 import harness
    pkg = types.ModuleType("fakeqk")
    subs = {}
    for sub in ("solvers", "bench", "cli"):
        m = types.ModuleType(f"fakeqk.{sub}")
        for name in ("solve_pa", "solve_sbm", "solve_sa"):
            setattr(m, name, name)
        subs[sub] = m
        monkeypatch.setitem(sys.modules, f"fakeqk.{sub}", m)
    for name in ("solve_pa", "solve_sbm", "solve_sa"):
        setattr(pkg, name, name)
    harness.use_in_reference(pkg)
    for m in [pkg, *subs.values()]:
        assert m.solve_pa._vxq_wrapped is vxq.solve_pa and m.solve_sa._vxq_wrapped is vxq.solve_sa
    harness.use_in_reference(pkg, restore=True)
    for m in [pkg, *subs.values()]:
        assert m.solve_pa == "solve_pa" and m.solve_sbm == "solve_sbm"


def test_use_in_reference_translates_errors(monkeypatch):
    """The product never imports the reference; swapped into it, our errors surface as the
    reference's own classes (qubokit/errors.py) so its `except` clauses still catch them."""
    import types
    from paper_2501_19221_b200 import harness

    class RefBase(Exception):
        pass

    class RefVal(RefBase, ValueError):
        pass

    pkg = types.ModuleType("fakeqk2")
    pkg.QubokitError, pkg.ValidationError = RefBase, RefVal
    pkg.solve_pa = pkg.solve_sbm = pkg.solve_sa = None
    harness.use_in_reference(pkg)
    with pytest.raises(RefVal):
        pkg.solve_pa(None, vxq.PaParams(steps=0))
    import paper_2501_19221_b200.errors as E
    assert E.ValidationError.__module__ == "paper_2501_19221_b200.errors"


def test_run_opts_stream_mapping():
    """NULL = the library's own stream per call; a caller's legacy default stream (handle
    0, e.g. torch's default current stream) becomes cudaStreamLegacy so work is ordered on
    it (three row-partition sessions on one stream must not race)."""
    from paper_2501_19221_b200.solvers import _opts
    assert _opts("fp32", "auto", 0).stream is None
    assert _opts("fp32", "auto", 0, stream=0).stream == 0x1
    assert _opts("fp32", "auto", 0, stream=0x7f00).stream == 0x7f00


def test_full_triangle_detection():
    """Dense models upload values only (vxq_problem_create with rows = cols = NULL): the
    detection accepts exactly the canonical full upper triangle."""
    from paper_2501_19221_b200.device import full_triangle, upload_bytes
    for n in (2, 3, 17, 300, 2049):
        iu, ju = np.triu_indices(n, 1)
        assert full_triangle(n, iu.astype(np.int64), ju.astype(np.int64))
        assert not full_triangle(n + 1, iu, ju)
        if len(iu) > 1:
            assert not full_triangle(n, iu[:-1], ju[:-1])
    iu, ju = np.triu_indices(300, 1)
    bad = ju.copy()
    bad[-1] = 0  # the last pair is always sampled
    assert not full_triangle(300, iu, bad)
    sk = vxq.IsingModel.from_arrays(300, iu, ju, np.ones(len(iu)), canonical=True)
    assert upload_bytes(sk) == 8 * len(iu) + 8 * 300
    sparse = vxq.IsingModel.from_arrays(300, iu[:10], ju[:10], np.ones(10), canonical=True)
    assert upload_bytes(sparse) == 24 * 10 + 8 * 300
