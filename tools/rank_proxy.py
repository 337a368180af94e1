"""One rank's share of the 8-GPU row-partitioned config 5, measured on one GPU.

A session over rows [0, n/8) of the full N = 2e8 instance (vxq_session_*, the same step
kernels a rank runs) steps against the full exchange buffer -- every neighbour gather goes
into the whole 2e8-row spin / q table, as it would on rank 0 of 8 -- with no exchange
between steps (the all-gather is the only thing missing; its bytes are reported).

    python tools/rank_proxy.py [--ranks 8] [--R 32 64 128 256] [--solver pa sbm] [--T 10]

One JSON line per (solver, R): device ms per step (CUDA events), rv-updates/s of the rank,
the algorithmic roofline fraction (SURVEY 8d bytes per update), the random-gather sector
floor (each neighbour gather moves at least one 32-byte sector, so a row's R/8 bytes cost
max(32, R/8) bytes) and the exchange bytes each rank would receive per step.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000_000)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--R", type=int, nargs="+", default=[32, 64, 128, 256])
    ap.add_argument("--solver", nargs="+", default=["pa", "sbm"])
    ap.add_argument("--T", type=int, default=10)
    args = ap.parse_args()

    import torch
    import paper_2501_19221_b200 as vxq
    from paper_2501_19221_b200 import instances
    from paper_2501_19221_b200.rowpart import GpuSession, exchange_row_bytes

    hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6451.0
    model = instances.build("cfg5", args.n)
    n = model.n
    dbar = 2.0 * model.num_couplings / n
    rows = -(-n // args.ranks)
    stream = torch.cuda.Stream()
    for solver in args.solver:
        for R in args.R:
            params = (vxq.PaParams(steps=args.T + 3, replicas=R, seed=5) if solver == "pa" else
                      vxq.SbmParams(steps=args.T + 3, dt=0.05, replicas=R, seed=5, c0=0.3))
            rb = exchange_row_bytes(solver, R)
            try:
                bufs = [torch.zeros(n * rb, dtype=torch.uint8, device="cuda") for _ in range(2)]
                sess = GpuSession(model, solver, params, 0, rows, n, bufs, "fp32", 0,
                                  stream.cuda_stream)
            except Exception as e:  # noqa: BLE001 (out of memory at large R)
                print(json.dumps({"solver": solver, "R": R, "error": str(e)[:200]}), flush=True)
                continue
            with torch.cuda.stream(stream):
                for t in range(3):  # warm-up steps
                    sess.step(t)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for t in range(3, 3 + args.T):
                    sess.step(t)
                e1.record(stream)
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.T
            units = rows * R
            if solver == "pa":
                alg = 16.0 + (1.0 + dbar) / 8.0 + (8.0 * dbar + 4.0) / R
                floor = 16.0 + (max(32.0, R / 8.0) * dbar + R / 8.0) / R + (8 * dbar + 4) / R
            else:
                alg = 16.0 + 4.0 * dbar + (8.0 * dbar + 4.0) / R
                floor = 16.0 + max(32.0, 4.0 * R) * dbar / R + (8 * dbar + 4) / R
            gbs = alg * units / (ms * 1e-3) / 1e9
            line = {"solver": solver, "R": R, "rows_per_rank": rows, "n": n, "dbar": dbar,
                    "ms_per_step": ms, "rv_per_s_rank": units / (ms * 1e-3),
                    "bytes_per_update_alg": alg, "frac_alg": gbs / hbm,
                    "bytes_per_update_sector_floor": floor,
                    "frac_sector_floor": floor * units / (ms * 1e-3) / 1e9 / hbm,
                    "exchange_bytes_received_per_step": (args.ranks - 1) * rows * rb,
                    "hbm_gbs": hbm}
            print(json.dumps(line), flush=True)
            sess.close()
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
