#!/usr/bin/env python
"""GTEPS of the B200 BFS/SSSP task-distribution path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (config C2): a step is one SSSP traversal from source 0 of RMAT
scale-22, edge factor 16 (default R-MAT params, seed 1, integer weights
1..255) with the headline strategy (WD), graph resident in HBM.
N > 1 (config C5): a step is one traversal of RMAT scale-27 (2^31 edges) from
source 0, 1-D edge-balanced vertex partition over the N GPUs, NCCL exchange of
(dist << 32 | v) updates per BSP iteration -- the same graph at every N
(strong scaling).  `--gpus N` without torchrun's environment launches the N
ranks itself (torch.distributed.run on 127.0.0.1).

`value` = E_r / device time per step (E_r = sum of outdegrees over reached
vertices, Graph500-style), whole job, max over ranks.  `e2e` measures the same
traversal through the C-ABI with host buffers: glb_graph_create (host int64
CSR -> HBM) + glb_run + the int64 distances back + glb_graph_destroy.
`roofline.frac` is SURVEY 8(d)'s one-pass algorithmic bytes of the traversal
(12 E_r + 20 N_r for SSSP, 8 E_r + 20 N_r for BFS) over the dominant kernel's
time per step, against the measured HBM peak (x N).

`--impl reference` times the reference's CPU algorithm on the host cores, in a
process that never loads the CUDA library: the reference is pure Python, so
the pinned C port of its node-based strategy (oracle/, oracle_bs_run_u32) runs
on every host thread over the graph built by the pinned C restatement of
generate_rmat (oracle_rmat_u32).  Under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
UNIT = "GTEPS"
TAGS = ("BS", "EP", "WD", "NS", "HP")
INF = (1 << 63) - 1
KERNEL_OF = {"WD": "k_wd_relax", "HP": "k_hp_window + k_hp_bigbin", "BS": "k_bs_relax",
             "NS": "k_ns_relax", "EP": "k_ep_relax"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--strategy", default=os.environ.get("GLB_BENCH_STRATEGY", "WD"))
    ap.add_argument("--algo", default="sssp", choices=("bfs", "sssp"))
    ap.add_argument("--scale", type=int, default=None,
                    help="R-MAT scale (default 22 = C2 at N=1, 27 = C5 at N>1)")
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--loop", default=os.environ.get("GLB_BENCH_LOOP", "graph"),
                    choices=("host", "graph"))
    ap.add_argument("--transport", default=os.environ.get("GLB_BENCH_TRANSPORT", "peer"),
                    choices=("peer", "torch"),
                    help="N>1 exchange: in-library P2P over NVLink (peer) or torch.distributed")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="bound of one CPU-baseline sample (full traversals below it)")
    ap.add_argument("--no-extras", action="store_true", help="skip the per-strategy table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-check", action="store_true", help="skip the parity checks")
    a = ap.parse_args()
    if a.scale is None:
        a.scale = 22 if a.gpus == 1 else 27
    return a


# ------------------------------------------------------------------ helpers
def workload_name(args, n_gpus):
    cfg = {(22, 16): "C2: ", (27, 16): "C5: "}.get((args.scale, args.edge_factor), "")
    part = (f", 1-D edge-balanced vertex partition over {n_gpus} GPUs with a per-iteration "
            f"exchange" if n_gpus > 1 else "")
    return (f"{cfg}{args.algo.upper()} on RMAT scale-{args.scale} edge-factor {args.edge_factor} "
            f"(a,b,c,d)=(0.45,0.15,0.15,0.25) seed 1, integer weights 1..255, source 0{part}")


def reached_edges(deg, dist):
    reached = dist != INF
    return int(deg[reached].sum()), int(reached.sum())


def algorithmic_bytes(algo, edges, items):
    """per edge col 4 + dist[dst] 4 (+ weight 4 for SSSP); per
    frontier vertex row offset 8 + dist write 4 + queue write 4 + queue read 4."""
    return (12 if algo == "sssp" else 8) * edges + 20 * items


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs (measured)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# the reference's CPU algorithm per strategy: C ports of run_wd / run_bs
PORTS = {"WD": ("wd_run_narrow", "run_wd", "workload.py:75-189"),
         "BS": ("bs_run_narrow", "run_bs", "node_based.py:19-82")}


def port_of(strategy):
    """Same strategy as our arm where a port exists (WD, BS), else run_bs."""
    return strategy.upper() if strategy.upper() in PORTS else "BS"


def cpu_sample(ng, algo, seconds, threads=0, strategy="WD"):
    """The pinned port of the strategy's driver on all host threads: full
    traversals while they fit the bound, else one time-bounded traversal
    extrapolated by its share of a full traversal's relaxations."""
    from oracle import oracle

    w = algo == "sssp"
    threads = threads or (os.cpu_count() or 1)
    fn = getattr(oracle, PORTS[port_of(strategy)][0])
    t0 = time.perf_counter()
    d, it, ops, done = fn(ng, 0, w, threads, max_seconds=seconds)
    t = time.perf_counter() - t0
    return d, it, ops, done, t, threads


# ----------------------------------------------------------------- our arm
def run_params(L, tag, algo, loop, timing=True):
    p = L.RunParams()
    p.strategy = {"BS": 0, "EP": 1, "WD": 2, "NS": 3, "HP": 4}[tag]
    p.algo = L.GLB_BFS if algo == "bfs" else L.GLB_SSSP
    p.source = 0
    p.bins = 10
    p.chunked = 1
    p.mdt = 0
    p.max_cells = 1_000_000_000
    p.block_size = 1024
    p.hp_fallback = 1
    p.dist_bits = 0
    p.loop_mode = L.GLB_LOOP_GRAPH if loop == "graph" else L.GLB_LOOP_HOST
    p.record_timing = 1 if timing else 0
    p.instrument = 0
    return p


class DeviceRunner:
    """Direct C-ABI runs on the resident graph (no host copy of distances)."""

    def __init__(self, handle):
        from paper_1711_00231_b200 import _lib

        self.L = _lib
        self.h = handle
        s = ctypes.c_void_p()
        _lib.check(_lib.lib().glb_graph_stream(self.h, ctypes.byref(s)))
        self.stream_ptr = s.value
        self.recs = (_lib.Record * 8192)()

    def run(self, tag, algo, loop, dist_out=None):
        p = run_params(self.L, tag, algo, loop)
        st = self.L.RunStats()
        ptr = None if dist_out is None else self.L.ptr64(dist_out)
        self.L.check(self.L.lib().glb_run(self.h, ctypes.byref(p), ptr, ctypes.byref(st),
                                          self.recs, len(self.recs)), f"glb_run {tag}")
        n = min(st.n_records, len(self.recs))
        return st, [self.recs[i] for i in range(n)]


def time_strategy(runner, torch, tag, algo, loop, steps, warmup):
    stream = torch.cuda.ExternalStream(runner.stream_ptr)
    for _ in range(warmup):
        runner.run(tag, algo, loop)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats, recs = [], []
    e0.record(stream)
    for _ in range(steps):
        st, rr = runner.run(tag, algo, loop)
        stats.append(st)
        recs.extend(rr)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), stats, recs


def roofline_of(args, recs, steps, e_r, n_r, ms_step, n_gpus, kernel_ms_step=None):
    """Dominant kernel against N x the measured HBM peak.  `frac` uses the
    one-pass bytes of the traversal; `examined` keeps the
    bytes of every edge the kernel examined (re-relaxations included)."""
    peak1, src = hbm_peak()
    peak = peak1 * n_gpus
    k_ms = kernel_ms_step if kernel_ms_step is not None else sum(r.kernel_ms for r in recs) / steps
    onepass = algorithmic_bytes(args.algo, e_r, n_r)
    launches = len(recs) / steps if recs else 0
    achieved = onepass / (k_ms / 1e3) / 1e9 if k_ms > 0 else None
    examined = None
    if recs:
        ex_bytes = sum(algorithmic_bytes(args.algo, r.work_total, r.active_items) for r in recs) / steps
        examined = {"bytes_per_step": int(ex_bytes),
                    "achieved_GBs": round(ex_bytes / (k_ms / 1e3) / 1e9, 1) if k_ms > 0 else None,
                    "frac": round(ex_bytes / (k_ms / 1e3) / 1e9 / peak, 4) if k_ms > 0 else None,
                    "what": "bytes of every edge / item the kernel examined (re-relaxations "
                            "counted as useful)"}
    traffic = traffic_note = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists() and launches:
        ps = json.loads(prof.read_text())
        ratio = ps.get(f"{args.strategy}_{args.algo}_traffic_over_algorithmic")
        if ratio and examined:
            traffic = int(ratio * examined["bytes_per_step"] / launches)
            traffic_note = (f"ncu dram read+write / examined bytes = {ratio} on the captured "
                            f"launches ({ps.get('source', '')}), per launch")
    return {
        "bound": "hbm",
        "achieved": round(achieved, 1) if achieved else None,
        "peak": round(peak, 1),
        "unit": "GB/s",
        "frac": round(achieved / peak, 4) if achieved else None,
        "traffic": traffic,
        "traffic_source": traffic_note,
        "kernel": KERNEL_OF[args.strategy],
        "peak_source": src + (f" x {n_gpus} GPUs" if n_gpus > 1 else ""),
        "algorithmic_bytes_per_launch": int(onepass / launches) if launches else int(onepass),
        "algorithmic_bytes_per_step": int(onepass),
        "bytes_def": ("one pass: 12 E_r + 20 N_r (SSSP) / 8 E_r + 20 N_r (BFS), SURVEY 8(d)"),
        "launches_per_step": launches,
        "kernel_ms_per_step": round(k_ms, 5),
        "kernel_share_of_step": round(k_ms / ms_step, 4) if ms_step else None,
        "whole_step_frac": round(onepass / (ms_step / 1e3) / 1e9 / peak, 5),
        "examined": examined,
    }


def ours(args):
    import torch

    import paper_1711_00231_b200 as pkg
    from paper_1711_00231_b200 import _lib

    torch.cuda.set_device(0)
    dev = 0
    t0 = time.time()
    g = pkg.generate_rmat(args.scale, args.edge_factor, seed=1, max_weight=255, device=dev,
                          download=False)
    gen_s = time.time() - t0
    runner = DeviceRunner(g.device_graph(dev))
    row, col, w = g.download_narrow()  # host copy for the oracle / baseline / e2e
    deg = np.diff(row)

    d_gpu = np.empty(g.num_nodes, dtype=np.int64)
    runner.run(args.strategy, args.algo, args.loop, d_gpu)
    e_r, n_r = reached_edges(deg, d_gpu)
    from oracle import oracle

    oracle.build()
    ng = oracle.NarrowGraph(row, col, w)
    parity = None
    if not args.no_check:  # the pinned oracle (tests/test_oracle_golden.py) on the host cores
        parity = bool(np.array_equal(oracle.narrow_distances(ng, 0, args.algo), d_gpu))

    # ---- timed region: K steps, barrier + synchronize on both sides
    launches0 = _lib.lib().glb_kernel_launches()
    clocks = ClockSampler(dev)
    clocks.start()
    torch.cuda.synchronize()
    ms, stats, recs = time_strategy(runner, torch, args.strategy, args.algo, args.loop,
                                    args.steps, args.warmup)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = _lib.lib().glb_kernel_launches() - launches0
    ms_step = ms / args.steps
    value = e_r / (ms_step / 1e3) / 1e9
    roofline = roofline_of(args, recs, args.steps, e_r, n_r, ms_step, 1)
    roofline["relax_per_traversed_edge"] = round(stats[-1].relax_ops / max(e_r, 1), 3)
    # measured ceiling of the relaxation's real bottleneck on the same graph:
    # one random 8 B cell gather per edge (dist[col[e]]) through L1TEX
    gp = (ctypes.c_double * 4)()
    _lib.check(_lib.lib().glb_measure_gather(runner.h, gp), "glb_measure_gather")
    k_ms = sum(r.kernel_ms for r in recs)
    edge_rate = sum(r.work_total for r in recs) / (k_ms / 1e3) if k_ms > 0 else None
    roofline["gather_ceiling"] = {
        "what": "dist[col[e]] gather rate on this graph's col array at full occupancy "
                "(glb_measure_gather), vs the dominant kernel's examined-edge rate",
        "gathers_per_s": round(gp[1] * 1e9, 0), "atomic_min_per_s": round(gp[2] * 1e9, 0),
        "col_stream_GBs": round(gp[0], 1), "cells_MB": round(gp[3], 1),
        "kernel_edges_per_s": round(edge_rate, 0) if edge_rate else None,
        "frac": round(edge_rate / (gp[1] * 1e9), 4) if edge_rate and gp[1] > 0 else None,
    }

    # ---- e2e through the C-ABI with host int64 buffers
    e2e = None
    if args.e2e_steps > 0:
        L = _lib.lib()
        row64, col64 = row, col.astype(np.int64)
        w64 = w.astype(np.int64) if w is not None else None
        out = np.empty(g.num_nodes, dtype=np.int64)
        times = []
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            h = ctypes.c_void_p()
            _lib.check(L.glb_graph_create(_lib.ptr64(row64), _lib.ptr64(col64), _lib.ptr64(w64),
                                          g.num_nodes, g.num_edges, dev, ctypes.byref(h)))
            p = run_params(_lib, args.strategy, args.algo, args.loop)
            st = _lib.RunStats()
            _lib.check(L.glb_run(h, ctypes.byref(p), _lib.ptr64(out), ctypes.byref(st), None, 0))
            L.glb_graph_destroy(h)
            torch.cuda.synchronize()
            if i:  # the first call warms the pinned staging ring
                times.append(time.perf_counter() - t1)
        assert np.array_equal(out, d_gpu)
        t = statistics.median(times)
        e2e = {"value": round(e_r / t / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(row64.nbytes + col64.nbytes + (w64.nbytes if w64 is not None else 0)),
               "d2h_bytes_per_step": int(out.nbytes),
               "ms_per_step": round(t * 1e3, 2),
               "path": "C-ABI: glb_graph_create(host int64 CSR) + glb_run + int64 dist to host + destroy"}
        del col64, w64

    # ---- per-strategy table (not the headline)
    extras = {}
    if not args.no_extras:
        for algo in ("sssp", "bfs"):
            tab = {}
            e_r_a = e_r
            if algo != args.algo:
                dd = np.empty(g.num_nodes, dtype=np.int64)
                runner.run("WD", algo, args.loop, dd)
                e_r_a, _ = reached_edges(deg, dd)
            for tag in TAGS:
                ms_t, st_t, rr = time_strategy(runner, torch, tag, algo, args.loop, 3, 1)
                kms = sum(r.kernel_ms for r in rr)
                tab[tag] = {"ms": round(ms_t / 3, 3), "gteps": round(e_r_a / (ms_t / 3 / 1e3) / 1e9, 3),
                            "launches": st_t[-1].launches, "iterations": st_t[-1].iterations,
                            "relax_per_edge": round(st_t[-1].relax_ops / max(e_r_a, 1), 3),
                            "kernel_share": round(kms / ms_t, 3) if ms_t else None}
            extras[algo] = tab

    # ---- CPU baseline: pinned C port of run_bs on the host cores
    cpu = None
    if not args.no_cpu:
        port = port_of(args.strategy)
        d, it, ops, done, t, thr = cpu_sample(ng, args.algo, args.cpu_seconds, strategy=port)
        rate = e_r / t / 1e9 if done else None
        _, drv, cite = PORTS[port]
        cpu = {"value": round(rate, 5) if rate else round(ops / t / 1e9, 5), "unit": UNIT,
               "cores": thr, "kind": "port", "strategy": port,
               "sample": (f"one full {args.algo.upper()} {drv} traversal of the benchmark graph "
                          f"({t:.2f} s, {it} iterations, {ops} relaxations), C port of "
                          f"{cite} on {thr} threads" if done else
                          f"{drv} stopped after {it} iterations / {t:.1f} s; value = examined "
                          f"edges per second")}

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (RMAT generated on the GPU, bit-identical to graphlb.generate_rmat)",
        "config": {"workload": workload_name(args, 1), "strategy": args.strategy,
                   "nodes": g.num_nodes, "edges": g.num_edges, "loop": args.loop,
                   "l2": "inputs larger than L2 (col+weights %.0f MB vs 126 MB L2); no flush" % (
                       g.num_edges * 8 / 1e6),
                   "parallelism": "single", "E_r": e_r, "N_r": n_r, "gen_s": round(gen_s, 1)},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
        "gpu_launches": int(launches), "parity_vs_oracle": parity,
        "strategies": extras,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------- sharded (N > 1)
def ours_sharded(args, world, rank, local):
    """N ranks, one GPU each (ranks share GPUs only in the gloo test mode):
    RMAT scale args.scale (C5 = 27 by default), the SAME graph at every N
    (strong scaling), 1-D edge-balanced vertex partition, per BSP iteration
    one exchange of (dist << 32 | v) updates.  Time = max over ranks of
    CUDA-event time per traversal; value = E_r of the whole graph / time."""
    import torch
    import torch.distributed as dist

    import paper_1711_00231_b200 as pkg
    from paper_1711_00231_b200 import _lib, sharded

    ndev = torch.cuda.device_count()
    backend = os.environ.get("GLB_BENCH_BACKEND") or ("nccl" if ndev >= world else "gloo")
    dev = local % max(ndev, 1)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    assert dist.get_world_size() == world == args.gpus, (dist.get_world_size(), world, args.gpus)
    tdev = "cuda" if backend == "nccl" else "cpu"
    tag = args.strategy if args.strategy in sharded.SHARD_TAGS else "WD"
    t0 = time.time()
    g = pkg.generate_rmat(args.scale, args.edge_factor, seed=1, max_weight=255, device=dev,
                          download=False)
    bounds = sharded.partition_bounds(g, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    row = np.empty(g.num_nodes + 1, dtype=np.int64)
    _lib.check(_lib.lib().glb_graph_download(g.device_graph(), _lib.ptr64(row), None, None))
    deg = np.diff(row)
    # rank 0: the single-GPU run on the full graph, before it is cut
    ref = None
    if rank == 0 and not args.no_check:
        ref = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(args.algo),
                               pkg.KernelConfig(loop="graph", instrument=False)).dist.array
    host_narrow = None
    if rank == 0 and not args.no_cpu:
        host_narrow = g.download_narrow()
    mdt = sharded.global_mdt(g)  # HP's window of the whole graph, before the cut
    _lib.check(_lib.lib().glb_graph_restrict(g.device_graph(), lo, hi), "glb_graph_restrict")
    m_own = int(row[hi] - row[lo])
    g.num_edges = m_own
    sg = sharded.ShardGraph(g, bounds, rank, dev, mdt=mdt)
    gen_s = time.time() - t0
    transport = sharded.DistTransport(torch) if args.transport == "torch" else "peer"
    cfg = pkg.KernelConfig(record_timing=True, instrument=False)
    op = pkg.RelaxOp(args.algo)

    def step():
        return sharded.run_sharded(tag, sg, 0, op, cfg, transport)

    d_own, info = step()
    e_r_own, n_r_own = reached_edges(deg[lo:hi], d_own)
    t = torch.tensor([e_r_own, n_r_own], dtype=torch.int64, device=tdev)
    dist.all_reduce(t)
    e_r, n_r = int(t[0]), int(t[1])
    parity = cert = None
    if not args.no_check:  # gather the owned ranges on rank 0
        full = [None] * world if rank == 0 else None
        dist.gather_object(d_own, full, dst=0)
        if rank == 0:
            whole = np.concatenate(full)
            parity = bool(np.array_equal(whole, ref))
            # independent exact check: the device distance certificate
            # (glb_validate) on a fresh single-GPU copy of the graph
            g2 = pkg.generate_rmat(args.scale, args.edge_factor, seed=1, max_weight=255,
                                   device=dev, download=False)
            cert = bool(pkg.validate_distances(g2, 0, args.algo, whole).matched)
            g2.release_device()
            del g2
    for _ in range(args.warmup):
        step()
    launches0 = _lib.lib().glb_kernel_launches()
    clocks = ClockSampler(dev)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    iters = 0
    k_ms = 0.0
    xinfo = None
    for _ in range(args.steps):
        _, inf = step()
        iters = inf["bsp_iterations"]
        k_ms += inf["kernel_ms"]
        xinfo = inf.get("exchange")
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = _lib.lib().glb_kernel_launches() - launches0
    ms_step = e0.elapsed_time(e1) / args.steps
    tt = torch.tensor([ms_step, k_ms / args.steps], dtype=torch.float64, device=tdev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step, k_step = float(tt[0]), float(tt[1])
    value = e_r / (ms_step / 1e3) / 1e9
    roofline = roofline_of(args, [], args.steps, e_r, n_r, ms_step, world, kernel_ms_step=k_step)
    roofline["kernel_ms_per_step_note"] = "max over ranks of the local relax kernels' time"

    # e2e: each rank uploads only its own rows from host int64 arrays, runs,
    # and reads its owned int64 distances back (max over ranks)
    e2e = None
    if args.e2e_steps > 0:
        hrow = np.empty(g.num_nodes + 1, dtype=np.int64)
        hcol = np.empty(m_own, dtype=np.int64)
        hw = np.empty(m_own, dtype=np.int64)
        _lib.check(_lib.lib().glb_graph_download(g.device_graph(), _lib.ptr64(hrow),
                                                 _lib.ptr64(hcol), _lib.ptr64(hw)))
        times = []
        for i in range(args.e2e_steps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().glb_graph_create(_lib.ptr64(hrow), _lib.ptr64(hcol), _lib.ptr64(hw),
                                                   g.num_nodes, m_own, dev, ctypes.byref(h)))
            dg = pkg.DeviceCsrGraph(h.value, g.num_nodes, m_own, True, dev)
            sg2 = sharded.ShardGraph(dg, bounds, rank, dev, mdt=mdt)
            d2, _ = sharded.run_sharded(tag, sg2, 0, op, cfg,
                                        sharded.DistTransport(torch) if args.transport == "torch"
                                        else "peer")
            if sg2.peer is not None:
                sg2.peer.close()
            dg.release_device()
            torch.cuda.synchronize()
            if i:
                times.append(time.perf_counter() - t1)
        assert np.array_equal(d2, d_own)
        te = torch.tensor([statistics.median(times)], dtype=torch.float64, device=tdev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        t_e2e = float(te.item())
        e2e = {"value": round(e_r / t_e2e / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(hrow.nbytes + hcol.nbytes + hw.nbytes),
               "d2h_bytes_per_step": int(d_own.nbytes), "ms_per_step": round(t_e2e * 1e3, 2),
               "path": "per rank: glb_graph_create(own rows, host int64) + sharded run + "
                       "owned int64 dist to host (bytes are rank 0's; time is the max over ranks)"}
        del hcol, hw
    cpu = None
    if rank == 0 and host_narrow is not None:
        from oracle import oracle

        oracle.build()
        ng = oracle.NarrowGraph(*host_narrow)
        _, it, ops, done, t, thr = cpu_sample(ng, args.algo, args.cpu_seconds, strategy=tag)
        cpu = {"value": round(e_r / t / 1e9 if done else ops / t / 1e9, 5), "unit": UNIT,
               "cores": thr, "kind": "port",
               "sample": (f"one full traversal of the same graph ({t:.1f} s)" if done else
                          f"run_bs port on the same graph, stopped after {it} iterations / "
                          f"{t:.1f} s; value = examined edges per second")}
    dist.barrier()  # the CPU sample ran on rank 0 only
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (RMAT generated on each GPU, bit-identical to graphlb.generate_rmat)",
            "config": {
                "workload": workload_name(args, world),
                "strategy": tag, "nodes": g.num_nodes, "edges": int(row[-1]),
                "parallelism": f"shard{world}", "backend": backend,
                "transport": ("peer: P2P stores into the owners' HBM (CUDA IPC over NVLink), "
                              "release/acquire mailboxes, one host read per iteration"
                              if args.transport == "peer" else f"torch.distributed {backend}"),
                "ranks_per_gpu": max(1, world // max(ndev, 1)),
                "E_r": e_r, "N_r": n_r, "bsp_iterations": iters, "gen_s": round(gen_s, 1),
                "l2": "inputs larger than L2; no flush"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches), "exchange": xinfo, "parity_vs_single_gpu": parity,
            "parity_certificate": cert,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# ------------------------------------------------------------ reference arm
def reference(args):
    """The reference's algorithm on the host cores, without the CUDA library:
    graph by the pinned C restatement of generate_rmat, steps by the pinned C
    port of the SAME strategy's driver as our arm (run_wd for WD, run_bs for
    BS; other strategies fall back to run_bs) -- full traversals; at scale >
    24 each step is a time-bounded sample whose value extrapolates by its
    share of a full traversal's relaxations, measured once untimed.  The other
    port is timed once beside it (``ports``) for the best-vs-best view."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    t0 = time.time()
    ng = oracle.rmat_narrow(args.scale, args.edge_factor, seed=1, max_weight=255, threads=threads)
    gen_s = time.time() - t0
    w = args.algo == "sssp"
    bounded = args.scale > 24
    port = port_of(args.strategy)
    fn_name, drv, cite = PORTS[port]
    run = getattr(oracle, fn_name)
    d, it, ops_full, done = run(ng, 0, w, threads)
    e_r, n_r = reached_edges(ng.outdegrees(), d)
    vals = []
    for i in range(args.warmup + args.steps):
        t1 = time.perf_counter()
        _, it, ops, done = run(ng, 0, w, threads, max_seconds=args.cpu_seconds if bounded else 0.0)
        t = time.perf_counter() - t1
        if i >= args.warmup:
            vals.append(e_r * (ops / ops_full) / t / 1e9)
    value = statistics.mean(vals)
    ms = e_r / (value * 1e9) * 1e3
    ports = {port: round(value, 5)}
    for other, (fo, _, _) in PORTS.items():  # one sample of the other port
        if other == port:
            continue
        t1 = time.perf_counter()
        _, _, ops, odone = getattr(oracle, fo)(ng, 0, w, threads, max_seconds=args.cpu_seconds)
        t = time.perf_counter() - t1
        # a full traversal: E_r / t; a bounded one: examined edges / t
        ports[other] = round((e_r if odone else ops) / t / 1e9, 5)
    sample = (f"each step = one {'time-bounded (' + str(args.cpu_seconds) + ' s) ' if bounded else 'full '}"
              f"{args.algo.upper()} {drv} traversal of the benchmark graph, C port of "
              f"{cite} on {threads} threads; graph from the C restatement of "
              f"generate_rmat (oracle_rmat_u32, {gen_s:.1f} s)")
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
        "higher_is_better": True, "scaling": "weak" if args.gpus == 1 else "strong",
        "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (RMAT from the pinned C restatement of graphlb.generate_rmat)",
        "config": {"workload": workload_name(args, args.gpus), "strategy": port,
                   "nodes": ng.num_nodes, "edges": ng.num_edges, "E_r": e_r, "N_r": n_r},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": threads, "kind": "port",
                         "strategy": port, "sample": sample},
        "ports": ports,
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- launcher
def self_launch(args) -> int:
    """`--gpus N` outside torchrun: start N local ranks on 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's init log (nranks, NVLS) visible
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


if __name__ == "__main__":
    if os.environ.get("GLB_BENCH_WATCHDOG_S"):  # debugging: dump every thread's stack, then exit
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["GLB_BENCH_WATCHDOG_S"]), exit=True)
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if a.impl == "reference":
        reference(a)
    elif world == 0 and a.gpus > 1:
        sys.exit(self_launch(a))
    elif max(world, 1) != a.gpus:
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    elif a.gpus > 1:
        ours_sharded(a, world, int(os.environ.get("RANK", "0")),
                     int(os.environ.get("LOCAL_RANK", "0")))
    else:
        ours(a)
