"""Time the device c0 (eig_extreme restatement) on fresh models and print how it was
obtained (vxq_problem_eig_info)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import paper_2501_19221_b200 as vxq  # noqa: E402
from paper_2501_19221_b200 import instances  # noqa: E402
from paper_2501_19221_b200.device import get_problem  # noqa: E402

for name, build in (("maxcut3_1e6", lambda: instances.maxcut3(1_000_000)),
                    ("maxcut3_1e5", lambda: instances.maxcut3(100_000)),
                    ("sk_1e4", lambda: instances.sk(10_000)),
                    ("pegasus16", instances.pegasus)):
    for rep in range(2):  # fresh model each time; the second reuses the memory pool
        m = build()
        dp = get_problem(m)
        t0 = time.perf_counter()
        c0 = vxq.resolve_c0(m)
        dt = time.perf_counter() - t0
        print(json.dumps({"case": name, "rep": rep, "n": m.n, "seconds": dt, **dp.eig_info()}),
              flush=True)
        vxq.clear_cache(m)
