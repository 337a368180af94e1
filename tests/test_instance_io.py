"""Instance files: the reference's quadratic text/JSON formats (instance_io.py:82-152)."""

import os
import sys

import numpy as np
import pytest

import paper_2501_19221_b200 as vxq
from paper_2501_19221_b200 import instance_io as io_
from paper_2501_19221_b200.instances import cfg1_qubo

REF = "/root/reference/pkg/src"


def _same(a, b, fields):
    for f in fields:
        assert np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(b, f))), f
    assert a.offset == b.offset


@pytest.mark.parametrize("suffix", [".txt", ".json"])
def test_roundtrip_ising_and_qubo(tmp_path, suffix):
    q, m = cfg1_qubo(7, n=30)
    back = io_.read_instance(io_.write_instance(tmp_path / f"m{suffix}", m))
    _same(back, m, ("rows", "cols", "values", "h"))
    back = io_.read_instance(io_.write_instance(tmp_path / f"q{suffix}", q))
    _same(back, q, ("rows", "cols", "values"))


def test_duplicates_accumulate_in_file_order(tmp_path):
    p = tmp_path / "d.txt"
    p.write_text("# offset: 0.5\n3 5 spin\n1 2 0.1\n2 1 0.2\n1 1 -1.0\n1 1 0.25\n3 2 0.3\n")
    m = io_.read_instance(p)
    assert m.rows.tolist() == [0, 1] and m.cols.tolist() == [1, 2]
    assert m.values[0] == (0.0 + 0.1) + 0.2 and m.h[0] == -1.0 + 0.25 and m.offset == 0.5


def test_errors(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("3 2 spin\n1 2 0.5\n")
    with pytest.raises(vxq.ValidationError):
        io_.read_instance(p)
    p.write_text("3 1 spin\n1 9 0.5\n")
    with pytest.raises(vxq.ValidationError):
        io_.read_instance(p)
    p.write_text("# format: hubo\n3 1 spin\n3 1 2 3 0.5\n")
    with pytest.raises(vxq.ValidationError):
        io_.read_instance(p)


def test_reads_reference_written_files_bit_identically(tmp_path):
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    sys.path.insert(0, REF)
    try:
        import qubokit as qk
        from qubokit import instance_io as rio
    finally:
        sys.path.remove(REF)
    for seed, n, dist in ((3, 40, "uniform"), (4, 25, "gaussian")):
        ref_model = qk.gen_random("complete", dist, seed, n=n)
        for suffix in (".txt", ".json"):
            path = rio.write_instance(tmp_path / f"r{seed}{suffix}", ref_model)
            mine, theirs = io_.read_instance(path), rio.read_instance(path)
            _same(mine, theirs, ("rows", "cols", "values", "h"))
    q = qk.QuboModel.from_terms(6, terms=[(0, 0, 1.5), (0, 3, -2.25), (2, 5, 0.125)],
                                offset=0.75)
    path = rio.write_instance(tmp_path / "q.txt", q)
    _same(io_.read_instance(path), rio.read_instance(path), ("rows", "cols", "values"))
