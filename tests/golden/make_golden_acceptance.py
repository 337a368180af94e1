"""Golden vectors for the reference's acceptance criteria #8 and #9 that touch the path,
from the UNMODIFIED reference (qubokit).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_acceptance.py

c8   test_acceptance.py:220-235: gen_random("complete", "uniform", 8000, n=100), solve_pa
     with 1000 steps, 1024 replicas, seed 8 -> per-replica final states and energies (the
     SampleSet re-indexed by replica) and the sorted energies.
c9_k test_acceptance.py:238-255, seeds k = 0..4: gen_random("complete", "int_uniform",
     9000 + k, n=50, a=-31, b=31) -> the exact optimum from the reference's branch and bound
     (solve_bb, spd_admissible, leaf 14) and the reference's best-of-1024 SA / PA energies.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import qubokit as qk  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def put_model(d, prefix, m):
    d[f"{prefix}_n"] = np.int64(m.n)
    d[f"{prefix}_rows"] = np.asarray(m.rows)
    d[f"{prefix}_cols"] = np.asarray(m.cols)
    d[f"{prefix}_values"] = np.asarray(m.values)
    d[f"{prefix}_h"] = np.asarray(m.h)
    d[f"{prefix}_offset"] = np.float64(m.offset)


def main():
    d = {}
    m = qk.gen_random("complete", "uniform", 8000, n=100)
    ss = qk.solve_pa(m, qk.PaParams(steps=1000, replicas=1024, seed=8))
    put_model(d, "c8", m)
    states = np.zeros((1024, m.n), dtype=np.int8)
    energies = np.zeros(1024)
    for s in ss.samples:
        states[s.replica] = s.state
        energies[s.replica] = s.energy
    d["c8_states"] = states
    d["c8_energies"] = energies
    d["c8_sorted"] = ss.energies()
    for k in range(5):
        m = qk.gen_random("complete", "int_uniform", 9000 + k, n=50, a=-31, b=31)
        put_model(d, f"c9_{k}", m)
        sa = qk.solve_sa(m, qk.SaParams(sweeps=1000, replicas=1024, seed=k)).best.energy
        pa = qk.solve_pa(m, qk.PaParams(steps=1000, replicas=1024, seed=k)).best.energy
        bb = qk.solve_bb(m, qk.BBParams(bound_kind="spd_admissible", leaf_size=14,
                                        time_limit=25.0))
        d[f"c9_{k}_sa_best"] = np.float64(sa)
        d[f"c9_{k}_pa_best"] = np.float64(pa)
        d[f"c9_{k}_bb_energy"] = np.float64(bb.energy)
        print(f"c9 seed {k}: bb {bb.energy} sa {sa} pa {pa}", flush=True)
    np.savez_compressed(os.path.join(OUT, "reference_acceptance.npz"), **d)


if __name__ == "__main__":
    main()
