import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle as O
import paper_2501_19221_b200 as vxq
from helpers import gen_complete
for n in (1000, 700):
    m = gen_complete(21, n)
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    for T in (5, 10, 20):
        r = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=256, seed=5), want_state=True)
        s = vxq.run_pa(m, vxq.PaParams(steps=T, replicas=256, seed=5), path="sparse", want_state=True)
        X = O.pa_init(5, 8, m.n)
        X, M = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), T), 0.05, 0.9, X, np.zeros_like(X))
        dd, ds, dds = np.abs(r.x[:8] - X), np.abs(s.x[:8] - X), np.abs(r.x - s.x)
        print(n, T, r.info["path"], "dense-fp64 max %.2e p99 %.2e" % (dd.max(), np.quantile(dd, .99)),
              "| sparse32-fp64 max %.2e p99 %.2e" % (ds.max(), np.quantile(ds, .99)),
              "| dense-sparse max %.2e frac>1e-4 %.4f" % (dds.max(), (dds > 1e-4).mean()),
              "| sign agree %.5f" % np.mean(r.states == s.states))
