"""Small solves over every kernel path, one process per case if wanted (compute-sanitizer
is closed on this GPU pool, so bad accesses are hunted with small cases, the kernels' own
bounds checks and the CPU oracle):

    python tools/path_sweep.py                 # all cases
    python tools/path_sweep.py --case pa_dense
    python tools/path_sweep.py --list

Each case checks its energies against the oracle's exact sums.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def sparse_model(n=300, seed=0):
    import paper_2501_19221_b200 as vxq
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, n * n, 6 * n))
    r, c = keys // n, keys % n
    keep = r < c
    return vxq.IsingModel.from_arrays(n, r[keep], c[keep], rng.uniform(-1, 1, keep.sum()),
                                      h=rng.uniform(-1, 1, n), canonical=True)


def sk_model(n=384, seed=4):
    import paper_2501_19221_b200 as vxq
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    J = np.where(rng.random(len(iu)) < 0.5, -1.0, 1.0) / np.sqrt(n)
    return vxq.IsingModel.from_arrays(n, iu, ju, J, canonical=True)


def check_energies(model, states, energies):
    import oracle as O
    assert np.array_equal(energies, O.energies_exact(model, states)), "energies"


def main():
    import paper_2501_19221_b200 as vxq
    P, S = vxq.PaParams, vxq.SbmParams
    sp, sp3k, sp40, sk = sparse_model(), sparse_model(3000), sparse_model(40), sk_model()
    cases = {  # name -> (model, run)
        "pa_resident": (sp, lambda m: vxq.run_pa(m, P(steps=30, replicas=64, seed=1),
                                                 path="resident")),
        "pa_sparse": (sp, lambda m: vxq.run_pa(m, P(steps=30, replicas=256, seed=1),
                                               path="sparse")),
        "pa_sparse_fp64": (sp, lambda m: vxq.run_pa(m, P(steps=30, replicas=96, seed=1),
                                                    path="sparse", precision="fp64")),
        "pa_coop": (sp3k, lambda m: vxq.run_pa(m, P(steps=20, replicas=32, seed=1),
                                               path="sparse")),
        "pa_track": (sp, lambda m: vxq.run_pa(m, P(steps=30, replicas=100, seed=1),
                                              path="sparse", trace=True, track_best=True)),
        "sbm_resident": (sp, lambda m: vxq.run_sbm(m, S(steps=30, dt=0.05, replicas=64, seed=2),
                                                   path="resident")),
        "sbm_sparse": (sp, lambda m: vxq.run_sbm(m, S(steps=30, dt=0.05, replicas=256, seed=2),
                                                 path="sparse")),
        "pa_dense": (sk, lambda m: vxq.run_pa(m, P(steps=10, replicas=256, seed=4))),
        "pa_dense_track": (sk, lambda m: vxq.run_pa(m, P(steps=10, replicas=200, seed=4),
                                                    trace=True, track_best=True)),
        "sbm_dense": (sk, lambda m: vxq.run_sbm(m, S(steps=10, dt=0.05, replicas=256, seed=4,
                                                     c0=0.02))),
        "sa": (sp, lambda m: vxq.run_sa(m, vxq.SaParams(sweeps=20, replicas=64, seed=3))),
        "sa_n40": (sp40, lambda m: vxq.run_sa(m, vxq.SaParams(sweeps=20, replicas=64, seed=3))),
        "lanczos": (sp3k, lambda m: vxq.device.c0(m)),
        "generate": (None, lambda m: vxq.device.GeneratedModel("qubo_deg6", 20000, 5).export()),
    }
    if os.environ.get("VXQ_SBM_PLANES") == "3":
        pass  # sbm_dense then runs the bf16x3 kernel
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append")
    ap.add_argument("--list", action="store_true")
    a = ap.parse_args()
    if a.list:
        print(" ".join(cases))
        return 0
    for name in a.case or list(cases):
        m, run = cases[name]
        r = run(m)
        if getattr(r, "states", None) is not None and not name.endswith("track"):
            check_energies(m, r.states, r.energies)
        print(f"{name}: ok", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
