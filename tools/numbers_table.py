"""Print the DESIGN.md numbers table from the committed bench lines (profiles/r02/bench_*.json
and the reference arm ref_*.json), so the document quotes exactly what the files hold.

    python tools/numbers_table.py [profiles/r02]
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROWS = [
    ("cfg1 dense random QUBO 100 × 64, PA", "bench_cfg1_pa", "ref_cfg1_pa"),
    ("cfg1, SBM", "bench_cfg1_sbm", "ref_cfg1_sbm"),
    ("**cfg2 dense SK 10⁴ × 1024, PA**", "bench_cfg2_pa", "ref_cfg2_pa"),
    ("cfg2, SBM (exact field)", "bench_cfg2_sbm", "ref_cfg2_sbm"),
    ("cfg3 Pegasus P16 × 4096, PA", "bench_cfg3_pa", "ref_cfg3_pa"),
    ("cfg3, SBM", "bench_cfg3_sbm", "ref_cfg3_sbm"),
    ("cfg4 3-regular 10⁶ × 256, PA", "bench_cfg4_pa", "ref_cfg4_pa"),
    ("cfg4, SBM", "bench_cfg4_sbm", "ref_cfg4_sbm"),
    ("cfg5 random QUBO 2·10⁸ × 32, PA (1 GPU)", "bench_cfg5_pa", None),
    ("cfg5, SBM (1 GPU)", "bench_cfg5_sbm", None),
    ("general dense J 10⁴ × 1024, PA", "bench_general_pa", None),
    ("general dense J 10⁴ × 1024, SBM", "bench_general_sbm", None),
]


def sci(v):
    if v is None:
        return "—"
    e = 0
    while abs(v) >= 10:
        v /= 10
        e += 1
    sup = str(e).translate(str.maketrans("0123456789-", "⁰¹²³⁴⁵⁶⁷⁸⁹⁻"))
    return f"{v:.2f}·10{sup}"


def load(d, name):
    p = os.path.join(d, name + ".json")
    if not name or not os.path.exists(p):
        return None
    return json.loads(open(p).read().strip().splitlines()[-1])


def ttt_text(b):
    t = b.get("time_to_target") or {}
    if not t:
        return "—"
    hits = [x for x in (t.get("schedule_sweep") or []) if x.get("step")]
    parts = []
    if t.get("step"):
        parts.append(f"at T = {t['steps']}: step {t['step']}, {t['ms']:.1f} ms")
    if hits:
        h = min(hits, key=lambda x: x.get("ms") or 1e30)
        parts.append(f"best schedule T = {h['steps']}: step {h['step']}, {h['ms']:.1f} ms")
    if not parts:
        parts.append(f"not reached (best {t.get('best_energy_seen')})")
    return f"target {t.get('target'):.6g}: " + "; ".join(parts)


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02")
    print("| config | value (rv/s) | e2e (rv/s) | roofline frac (DRAM frac) | kernel | "
          "reference arm: all cores / 1 thread | time to target |")
    print("|---|---|---|---|---|---|---|")
    for label, bn, rn in ROWS:
        b = load(d, bn)
        if b is None:
            continue
        r = load(d, rn) if rn else None
        roof = b["roofline"]
        frac = f"{roof['frac']:.2f}"
        if roof.get("dram_frac"):
            frac += f" ({roof['dram_frac']:.2f})"
        e2e = (b.get("e2e") or {}).get("value")
        kern = roof.get("kernel", "").split(":")[0].split(" (")[0]
        ref = "—"
        if r:
            one = (r.get("cpu_baseline") or {}).get("one_thread") or {}
            ref = f"{sci(r['value'])} / {sci(one.get('value'))}"
        print(f"| {label} | {sci(b['value'])} | {sci(e2e) if e2e else '(device-generated)'} | "
              f"{frac} | `{kern}` | {ref} | {ttt_text(b)} |")


if __name__ == "__main__":
    main()
