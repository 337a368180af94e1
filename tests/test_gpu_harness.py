"""Drop-in at the reference's own swap points: the UNMODIFIED reference bench
harness (qubokit.bench.run_suite, bench.py:196-263, installed in baseline/_ref) drives the
B200 solvers after `use_in_reference` patches its solver table.  Skipped when the
reference install is absent."""

import os
import sys

import numpy as np
import pytest

import paper_2501_19221_b200 as vxq
from paper_2501_19221_b200 import harness

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline",
                   "_ref")


@pytest.fixture()
def qk():
    if not os.path.isdir(os.path.join(REF, "qubokit")):
        pytest.skip("baseline/_ref not installed")
    sys.path.insert(0, REF)
    try:
        import qubokit
        import qubokit.bench
        saved = {k: getattr(qubokit.bench, k) for k in ("solve_pa", "solve_sbm", "solve_sa")}
        yield qubokit
        for k, v in saved.items():
            setattr(qubokit.bench, k, v)
    finally:
        sys.path.remove(REF)


def test_reference_run_suite_with_b200_solvers(qk):
    harness.use_in_reference(qk)
    spec = qk.bench.SuiteSpec(
        source={"generator": {"family": "random", "sizes": [12], "seeds": [1, 2, 3]}},
        solvers=[{"id": "sa", "params": {"sweeps": 300}},
                 {"id": "pa", "params": {"steps": 500}},
                 {"id": "sbm", "params": {"steps": 2000, "dt": 0.05}}],
        reference="brute_force", replicas=64)
    recs = qk.bench.run_suite(spec)
    assert len(recs) == 9 and not any(r.error for r in recs)
    # every B200 solver reaches the exhaustive optimum on these n = 12 instances
    for r in recs:
        assert r.gap <= 1e-9, (r.instance_id, r.solver_id, r.gap)
    # the records came from this package's solvers (wall time of GPU calls, exact energies)
    assert qk.bench.solve_pa._vxq_wrapped is vxq.solve_pa
    assert qk.bench.solve_sa._vxq_wrapped is vxq.solve_sa


def test_reference_models_and_params_accepted_directly(qk):
    m = qk.generators.gen_random("complete", "uniform", 4, n=10)
    ss = vxq.solve_pa(m, qk.PaParams(steps=300, replicas=32, seed=1))
    assert ss.best.energy == pytest.approx(min(s.energy for s in ss.samples))
    sa = vxq.solve_sa(m, qk.SaParams(sweeps=200, replicas=16, seed=2))
    assert len(sa) == 16
    e, c = qk.bench.spectrum(sa, 5)
    assert c.sum() == 16 and np.all(np.diff(e) > 0)
