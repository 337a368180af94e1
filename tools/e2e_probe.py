"""Phase breakdown of one end-to-end solve through the public API (cfg2 by default):
problem upload/build, dynamics, result assembly -- pageable vs pinned host inputs.

    python tools/e2e_probe.py [--config cfg2] [--T 1000]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def pinned_like(a):
    import torch
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    v = t.numpy()
    v[...] = a
    return v, t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--T", type=int, default=1000)
    a = ap.parse_args()
    import torch
    import paper_2501_19221_b200 as vxq
    from paper_2501_19221_b200 import instances
    from paper_2501_19221_b200.device import get_problem
    cfg = instances.CONFIGS[a.config]
    m = instances.build(a.config)
    R = cfg["R"]
    p = vxq.PaParams(steps=a.T, replicas=R, seed=0)
    keep = []
    variants = {"pageable": (m.rows, m.cols, m.values, m.h)}
    arrs = []
    for x in (m.rows, m.cols, m.values, m.h):
        v, t = pinned_like(np.ascontiguousarray(x))
        keep.append(t)
        arrs.append(v)
    variants["pinned"] = tuple(arrs)
    for name, (r, c, v, h) in variants.items():
        for rep in range(3):
            fresh = vxq.IsingModel(n=m.n, h=h, rows=r, cols=c, values=v, offset=m.offset)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dp = get_problem(fresh)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            res = vxq.run_pa(fresh, p)
            t2 = time.perf_counter()
            ss = vxq.solvers.sampleset_from(res, R, 0, t2 - t1)
            t3 = time.perf_counter()
            print(f"{name} rep{rep}: create {1e3 * (t1 - t0):.1f} ms  run {1e3 * (t2 - t1):.1f} ms "
                  f"(loop {res.info['loop_ms']:.1f})  sampleset {1e3 * (t3 - t2):.1f} ms  "
                  f"total {1e3 * (t3 - t0):.1f} ms  best {ss.best.energy:.6g}", flush=True)
            vxq.clear_cache(fresh)
            del fresh, dp


if __name__ == "__main__":
    main()
