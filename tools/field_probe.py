"""Field-error probe for the dense SBM tensor paths: one SBM step, the field f = Q0 @ B
recovered from the momentum update (bifurcation.py:41) and compared with the exact field
(fp64 of the fp32 initial state).  Prints mean / max / bias of the error per path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2501_19221_b200 as vxq  # noqa: E402
from paper_2501_19221_b200 import instances  # noqa: E402


def probe(m, R, path, planes, c0=1.0, dt=0.5):
    if planes == "exact":
        os.environ.pop("VXQ_SBM_PLANES", None)
    else:
        os.environ["VXQ_SBM_PLANES"] = planes
    r = vxq.run_sbm(m, vxq.SbmParams(steps=1, dt=dt, replicas=R, seed=2, c0=c0, q_cap=2.0), path=path,
                    want_state=True)
    reps = np.r_[0:4, R - 4:R]
    Q0 = np.stack([O.uniform(2, int(k), 0, m.n, -1, 1) for k in reps]).astype(np.float32)
    P0 = np.stack([O.uniform(2, int(k), m.n, m.n, -1, 1) for k in reps]).astype(np.float32)
    Q0 = Q0.astype(np.float64)
    P0 = P0.astype(np.float64)
    B = np.zeros((m.n, m.n))
    B[m.rows, m.cols] = -m.values
    B[m.cols, m.rows] = -m.values
    f_exact = Q0 @ B
    P1 = r.m[reps]
    f_gpu = ((P1 - P0) / dt + (Q0 * Q0 + 1.0) * Q0) / c0 + m.h
    e = f_gpu - f_exact
    return r.info["path"], float(np.abs(e).mean()), float(np.abs(e).max()), float(e.mean()), \
        float(np.abs(f_exact).mean())


for n in (1000, 10000):
    m = instances.sk(n)
    R = 256
    for path, planes in (("sparse", "2"), ("dense", "exact"), ("dense", "2"), ("dense", "3")):
        print(n, path, planes, probe(m, R, path, planes), flush=True)
