"""One short solve for profiling (ncu launch lists / --set full captures).

    python tools/profile_run.py --config cfg2 --T 8 [--solver pa] [--path auto]

Prints per-phase host timings; the kernels it launches are the ones bench.py times.
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--solver", default="pa")
    ap.add_argument("--path", default="auto")
    ap.add_argument("--replicas", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    import paper_2501_19221_b200 as vxq
    from paper_2501_19221_b200 import instances
    R = a.replicas or instances.CONFIGS[a.config]["R"]
    t0 = time.perf_counter()
    m = instances.build(a.config, a.n)
    t1 = time.perf_counter()
    from paper_2501_19221_b200.device import get_problem
    get_problem(m)
    t2 = time.perf_counter()
    print(f"build {t1 - t0:.2f}s  upload+csr {t2 - t1:.2f}s  n={m.n} m={m.num_couplings}")
    for k in range(a.repeat):
        t3 = time.perf_counter()
        if a.solver == "sa":
            r = vxq.run_sa(m, vxq.SaParams(sweeps=a.T, replicas=R, seed=k), path=a.path)
        elif a.solver == "pa":
            r = vxq.run_pa(m, vxq.PaParams(steps=a.T, replicas=R, seed=k), path=a.path)
        else:
            r = vxq.run_sbm(m, vxq.SbmParams(steps=a.T, dt=0.05, replicas=R, seed=k),
                            path=a.path)
        t4 = time.perf_counter()
        print(f"solve {k}: wall {1e3 * (t4 - t3):.1f} ms  loop {r.info['loop_ms']:.2f} ms "
              f"({r.info['loop_ms'] / a.T * 1e3:.1f} us/step)  path {r.info['path']}  "
              f"bestE {r.energies.min():.6g}")


if __name__ == "__main__":
    main()
