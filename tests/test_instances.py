"""Instance generators on the path's input side."""

import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2501_19221_b200 import instances

REF_SRC = "/root/reference/pkg/src"


@pytest.mark.parametrize("m,n,e", [(6, 680, 4484), (16, 5640, 40484)])
def test_pegasus_counts(m, n, e):
    nn, edges = instances.pegasus_edges(m)
    assert nn == n and edges.shape == (e, 2)
    assert (edges[:, 0] != edges[:, 1]).all()
    assert len(np.unique(np.sort(edges, 1), axis=0)) == e
    deg = np.bincount(edges.ravel(), minlength=nn)
    assert deg.min() >= 1 and deg.max() == 15


def test_pegasus_degree_histogram():
    """P16 fabric: 4472 qubits of degree 15, 688 of 14, boundary qubits lower."""
    _, e16 = instances.pegasus_edges(16)
    h = np.bincount(np.bincount(e16.ravel()))
    assert h[15] == 4472 and h[14] == 688 and h[11] == 208 and h[10] == 32
    assert h.sum() == 5640


def test_pegasus_instance_recipe():
    m = instances.pegasus(6, seed=3)
    assert m.n == 680 and m.num_couplings == 4484
    assert (m.rows < m.cols).all()
    assert np.all(np.abs(m.values) <= 1) and np.all(np.abs(m.h) <= 1)
    # deterministic
    m2 = instances.pegasus(6, seed=3)
    assert np.array_equal(m.values, m2.values) and np.array_equal(m.h, m2.h)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_pegasus_instance_matches_reference_gen_random():
    """Our vectorised instance == the reference's gen_random("edge_list", "uniform") fed
    the same edge list (coupling draws first, then biases, one Philox stream)."""
    n, e = instances.pegasus_edges(6)
    ours = instances.pegasus(6, seed=11)
    code = (
        "import sys, numpy as np, hashlib\n"
        "from qubokit.generators import gen_random\n"
        "e = np.load(sys.argv[1])\n"
        "m = gen_random('edge_list', 'uniform', 11, n=int(sys.argv[2]), "
        "edges=[tuple(x) for x in e.tolist()])\n"
        "d = hashlib.sha256()\n"
        "for a in (m.rows, m.cols, m.values, m.h): d.update(np.ascontiguousarray(a).tobytes())\n"
        "print(d.hexdigest())\n"
    )
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "e.npy")
        np.save(p, e)
        env = dict(os.environ, PYTHONPATH=REF_SRC)
        out = subprocess.run([sys.executable, "-c", code, p, str(n)], env=env,
                             capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    d = hashlib.sha256()
    for a in (ours.rows.astype(np.int64), ours.cols.astype(np.int64),
              ours.values.astype(np.float64), ours.h.astype(np.float64)):
        d.update(np.ascontiguousarray(a).tobytes())
    assert out.stdout.strip() == d.hexdigest()
