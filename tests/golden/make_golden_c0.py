"""Golden c0 values from the UNMODIFIED reference's resolve_c0 (bifurcation.py:25-34 ->
eig_extreme(-A, "max"), solvers/eigen.py:35-56) at the sizes where the device Lanczos is
the only c0 source:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_c0.py

Instances are rebuilt on the GPU box from their seeded recipes (paper_2501_19221_b200.
instances), so only the recipe parameters and the reference's c0 are stored:
  maxcut3 n = 1e5, 1e6 (cfg 4 family, ARPACK path), Pegasus P16 (cfg 3, ARPACK path),
  SK n = 1000 (cfg 2 family, dense ARPACK path), SK n = 400 and cfg1 (n <= 512: eigvalsh).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for p in (REF, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import qubokit as qk  # noqa: E402
from qubokit.solvers import resolve_c0  # noqa: E402

from paper_2501_19221_b200 import instances  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_model(m):
    return qk.IsingModel(n=m.n, h=np.array(m.h), rows=np.array(m.rows), cols=np.array(m.cols),
                         values=np.array(m.values), offset=m.offset)


CASES = [  # name, builder (seeded recipe)
    ("maxcut3_1e5", lambda: instances.maxcut3(100_000)),
    ("maxcut3_1e6", lambda: instances.maxcut3(1_000_000)),
    ("pegasus16", lambda: instances.pegasus()),
    ("sk_1000", lambda: instances.sk(1000)),
    ("sk_400", lambda: instances.sk(400)),
    ("cfg1", lambda: instances.cfg1_qubo()[1]),
]


def main():
    out = {}
    for name, build in CASES:
        m = build()
        t0 = time.perf_counter()
        c0 = resolve_c0(ref_model(m))
        dt = time.perf_counter() - t0
        print(f"{name}: n={m.n} c0={c0!r} ({dt:.1f} s)", flush=True)
        out[f"{name}_c0"] = np.float64(c0)
        out[f"{name}_seconds"] = np.float64(dt)
    np.savez_compressed(os.path.join(OUT, "reference_c0.npz"), **out)


if __name__ == "__main__":
    main()
