"""Time the GPU simulated-annealing kernel (k_sa_run) on cfg 3 (Pegasus P16) and print a
fingerprint of its results, so side builds (VXQ_LIB=...) can be compared for speed AND for
bit-identical output.

    python tools/sa_probe.py [--R 4096] [--sweeps 200] [--precision fp32 fp64] [--path ...]

One JSON line per (precision, path): device ms per sweep (the C-ABI's loop_ms), the best
energy, and a SHA-1 of the per-replica energies and best states.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=4096)
    ap.add_argument("--sweeps", type=int, default=200)
    ap.add_argument("--precision", nargs="+", default=["fp32", "fp64"])
    ap.add_argument("--path", nargs="+", default=["auto"])
    args = ap.parse_args()

    import paper_2501_19221_b200 as vxq
    from paper_2501_19221_b200 import instances

    m = instances.build("cfg3")
    for prec in args.precision:
        for path in args.path:
            p = vxq.SaParams(sweeps=args.sweeps, replicas=args.R, seed=0)
            vxq.run_sa(m, vxq.SaParams(sweeps=2, replicas=args.R, seed=0), precision=prec,
                       path=path)  # warm-up
            r = vxq.run_sa(m, p, precision=prec, path=path)
            h = hashlib.sha1(np.ascontiguousarray(r.energies).tobytes() +
                             np.ascontiguousarray(r.states).tobytes()).hexdigest()
            print(json.dumps({"precision": prec, "path": r.info.get("path", path),
                              "R": args.R, "sweeps": args.sweeps,
                              "ms_per_sweep": r.info["loop_ms"] / args.sweeps,
                              "best_energy": float(np.min(r.energies)), "sha1": h}),
                  flush=True)


if __name__ == "__main__":
    main()
