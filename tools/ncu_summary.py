"""Summarise an ncu report: key metrics per profiled launch + top stall SASS lines."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Issued Ipc Active", "Grid Size", "Avg. Active Threads Per Warp", "Eligible Warps Per Scheduler",
        "Static Shared Memory Per Block", "Theoretical Occupancy", "Compute (SM) Throughput",
        "L2 Cache Throughput", "Executed Instructions"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = {k: i for i, k in enumerate(rows[0])}
    res = {}
    for r in rows[1:]:
        kid = r[h["ID"]]
        res.setdefault(kid, {"name": r[h["Kernel Name"]][:60]})
        m = r[h["Metric Name"]]
        if m in KEYS:
            res[kid][m] = r[h["Metric Value"]] + " " + r[h["Metric Unit"]]
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        res.append({n: r[h.index(n)] for n in names if n in h})
    return res


def stalls(rep, top=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    h = rows[hi[0]]
    idx = {k: i for i, k in enumerate(h)}
    end = hi[1] if len(hi) > 1 else len(rows)
    data = [r for r in rows[hi[0] + 1:end] if len(r) > 5]

    def v(r):
        try:
            return int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            return 0
    tot = sum(v(r) for r in data)
    return tot, [(v(r), r[idx["Source"]].strip()[:80]) for r in sorted(data, key=lambda r: -v(r))[:top]]


if __name__ == "__main__":
    rep = sys.argv[1]
    for kid, d in details(rep).items():
        print(kid, d)
    for r in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                       "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]):
        print(r)
    tot, top = stalls(rep)
    print("stall samples", tot)
    for s, src in top:
        print(f"{s:6d} {src}")
