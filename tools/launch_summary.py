"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time per
kernel, launches, and share of the profiled total.

    python tools/launch_summary.py gpurun_out/launches.csv [--skip-prefix glb::k_rmat]
"""
import collections
import csv
import sys


def summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v * scale
    return agg


if __name__ == "__main__":
    agg = summary(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':64s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:64]:64s} {n:8d} {t:11.1f} {t / n:9.2f} {100 * t / tot:5.1f}%")
    print(f"{'total':64s} {sum(v[0] for v in agg.values()):8d} {tot:11.1f}")
