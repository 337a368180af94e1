"""Randomised shape sweep of the persistent tensor-core kernels against their numpy
emulations (bit-exact): k_dense_run<mxf4, pair> (PA) and k_dense_run<i8x3, pair> (SBM, exact
field).  Ragged n (not a multiple of 128 / odd row-tile counts) and ragged R exercise the
tile queue, the half-empty last pair and the ragged last replica block.

    python tools/dense_fuzz.py [--cases 40] [--seed 0]

Prints one JSON line per case and a summary; exit status 1 on any mismatch.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=40)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--rmin", type=int, default=128)
    ap.add_argument("--rmax", type=int, default=1300)
    args = ap.parse_args()

    import paper_2501_19221_b200 as vxq
    from test_gpu_shapes import (dense_pa_emulation_rows, dense_sbm_exact_emulation_rows,
                                 sign_matrix_f32, uniform_energies)

    rng = np.random.default_rng(args.seed)
    bad = 0
    for case in range(args.cases):
        n = int(rng.integers(256, 3200))
        R = int(rng.integers(args.rmin, args.rmax))
        T = int(rng.integers(2, 40))
        seed = int(rng.integers(0, 2 ** 31))
        density = float(rng.choice([1.0, 0.3, 0.05]))
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(len(iu)) < density
        J = np.where(rng.random(keep.sum()) < 0.5, -1.0, 1.0) / np.sqrt(n)
        m = vxq.IsingModel.from_arrays(n, iu[keep], ju[keep], J, canonical=True)
        reps = np.unique(np.r_[0, R // 2, R - 1, rng.integers(0, R, 3)])
        K = sign_matrix_f32(m)
        r = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=R, seed=seed), path="dense",
                       want_state=True)
        X, M = dense_pa_emulation_rows(m, K, reps, T, seed)
        ok_pa = (r.info["dense_kind"] == "mxf4" and np.array_equal(r.x[reps], X) and
                 np.array_equal(r.m[reps], M))
        c0 = float(rng.uniform(0.1, 1.0))
        s = vxq.run_sbm(m, vxq.SbmParams(steps=T, dt=0.05, replicas=R, seed=seed, c0=c0),
                        path="dense", want_state=True)
        Q, P = dense_sbm_exact_emulation_rows(m, K, reps, T, seed, c0)
        ok_sbm = (s.info["dense_kind"] == "i8x3" and np.array_equal(s.x[reps], Q) and
                  np.array_equal(s.m[reps], P))
        ok_e = (np.array_equal(r.energies[reps], uniform_energies(m, r.states[reps], K)) and
                np.array_equal(s.energies[reps], uniform_energies(m, s.states[reps], K)))
        bad += not (ok_pa and ok_sbm and ok_e)
        print(json.dumps({"case": case, "n": n, "R": R, "T": T, "density": density,
                          "pa": bool(ok_pa), "sbm": bool(ok_sbm), "energies": bool(ok_e)}),
              flush=True)
    print(json.dumps({"cases": args.cases, "mismatches": bad}))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
