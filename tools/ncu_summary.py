"""Summarise ncu outputs: launch-list CSV (per-kernel totals) and --set full reports."""
import collections
import csv
import subprocess
import sys


def launches(path, top=15):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][-60:]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        try:
            a[1] += float(r[vi].replace(",", ""))
        except ValueError:
            pass
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}% x{c:<5d} {k}")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg",
           "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        out.append(f"kernel: {v[h.index('Kernel Name')][:90]}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"  {m:70s} {v[i]:>14s} {units[i]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    if len(rows) > 3:
        h = rows[1]
        si, sc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        def num(x):
            try:
                return float(x or 0)
            except ValueError:
                return 0.0
        data = [r for r in rows[2:] if len(r) > max(si, sc)]
        for r in data:
            r[si] = num(r[si])
        tot = sum(r[si] for r in data) or 1.0
        out.append("  top stall sites (share of warp samples):")
        for r in sorted(data, key=lambda r: -float(r[si] or 0))[:12]:
            out.append(f"    {100 * r[si] / tot:5.1f}%  {r[sc][:100]}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(launches(p) if p.endswith(".csv") else full(p))
