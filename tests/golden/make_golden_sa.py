"""Golden vectors for simulated annealing, from the UNMODIFIED reference (qubokit).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_sa.py

Stores, per case, the instance arrays, the reference's solve_sa (annealing.py:24-74)
per-replica best states (SampleSet re-indexed by replica) and sample energies, plus the
initial spins 2*integers(0,2,n)-1 of a few streams (annealing.py:40).
Cases:
  int20    n=20 complete, int_uniform couplings and biases in [-3, 3]: every quantity is
           an integer, so any summation order is exact (BLAS or CSR alike)
  csr2100  n=2100 random sparse, uniform [-1, 1] -> the reference runs scipy CSR
           (n > 2048), whose S @ A order the restatement follows
  dense40  n=40 complete, uniform [-1, 1] (dense BLAS operator: F/E0 orders differ by ulps)
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import qubokit as qk  # noqa: E402
from qubokit.generators import gen_random  # noqa: E402
from qubokit.solvers.common import replica_streams  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def by_replica(sset, n):
    R = sset.replica_count
    states = np.zeros((R, n), dtype=np.int8)
    energies = np.zeros(R)
    for s in sset.samples:
        states[s.replica] = s.state
        energies[s.replica] = s.energy
    return states, energies


def sparse_edges(n, m, seed):
    rng = np.random.default_rng(seed)
    keys = set()
    while len(keys) < m:
        a, b = (int(v) for v in rng.integers(0, n, 2))
        if a != b:
            keys.add((min(a, b), max(a, b)))
    return sorted(keys)


def main():
    g = {}
    cases = {
        "int20": (gen_random("complete", "int_uniform", 5, n=20, a=-3, b=3),
                  dict(sweeps=200, replicas=16, seed=3)),
        "csr2100": (gen_random("edge_list", "uniform", 7, n=2100,
                               edges=sparse_edges(2100, 6300, 1)),
                    dict(sweeps=12, replicas=8, seed=11)),
        "dense40": (gen_random("complete", "uniform", 9, n=40),
                    dict(sweeps=300, replicas=32, seed=2)),
    }
    for name, (m, kw) in cases.items():
        ss = qk.solve_sa(m, qk.SaParams(**kw))
        st, en = by_replica(ss, m.n)
        g.update({f"{name}_n": np.int64(m.n), f"{name}_rows": m.rows, f"{name}_cols": m.cols,
                  f"{name}_values": m.values, f"{name}_h": m.h,
                  f"{name}_offset": np.float64(m.offset), f"{name}_states": st,
                  f"{name}_energies": en, f"{name}_sweeps": np.int64(kw["sweeps"]),
                  f"{name}_replicas": np.int64(kw["replicas"]),
                  f"{name}_seed": np.int64(kw["seed"])})
        print(name, m.n, len(m.rows), "best", ss.best.energy)
    # initial spins of three streams, n = 101 (odd: the buffered 32-bit half is dropped)
    S0 = np.stack([2 * s.integers(0, 2, size=101) - 1 for s in replica_streams(123, 3)])
    g["init_seed123_n101"] = S0.astype(np.int8)
    np.savez_compressed(os.path.join(OUT, "reference_sa.npz"), **g)


if __name__ == "__main__":
    main()
