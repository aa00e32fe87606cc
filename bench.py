#!/usr/bin/env python
"""GTEPS of the B200 BFS/SSSP task-distribution path (BASELINE.json config C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one SSSP traversal from source 0 of RMAT scale-22, edge factor 16
(default R-MAT params, seed 1, integer weights 1..255) with the headline
strategy, graph already resident in HBM.  `value` = E_r / device time per step
(E_r = sum of outdegrees over reached vertices, Graph500-style), whole-job
over all ranks.  `e2e` measures the same traversal through the C-ABI with host
buffers: glb_graph_create (host int64 CSR -> HBM) + glb_run + the int64
distances back to the host + glb_graph_destroy.

`--impl reference` times the reference's CPU algorithm on the host cores: the
reference is pure Python (not compilable), so the pinned C port of its
node-based strategy (oracle/graphlb_oracle.c, oracle_bs_run) runs with every
host thread.  Under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--strategy", default=os.environ.get("GLB_BENCH_STRATEGY", "WD"))
    ap.add_argument("--algo", default="sssp", choices=("bfs", "sssp"))
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--loop", default=os.environ.get("GLB_BENCH_LOOP", "graph"),
                    choices=("host", "graph"))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-extras", action="store_true", help="skip the per-strategy table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-check", action="store_true", help="N>1: skip the single-GPU self-check")
    return ap.parse_args()


# ------------------------------------------------------------------ workload
def workload(args, device=0):
    """The benchmark graph, generated in HBM by the CUDA R-MAT generator
    (bit-identical to graphlb.generate_rmat; tests pin it) and copied back for
    the CPU oracle / baseline."""
    import paper_1711_00231_b200 as pkg

    t0 = time.time()
    g = pkg.generate_rmat(args.scale, args.edge_factor, seed=1, max_weight=255, device=device)
    return g, time.time() - t0


def workload_desc(args, g):
    return {
        "workload": (f"{'C2: ' if (args.scale, args.edge_factor) == (22, 16) else ''}"
                     f"{args.algo.upper()} on RMAT scale-{args.scale} edge-factor "
                     f"{args.edge_factor} (a,b,c,d)=(0.45,0.15,0.15,0.25) seed 1, "
                     f"integer weights 1..255, source 0"),
        "strategy": args.strategy,
        "nodes": g.num_nodes,
        "edges": g.num_edges,
        "loop": args.loop,
        "l2": "inputs larger than L2 (col+weights %.0f MB vs 126 MB L2); no flush" % (
            g.num_edges * 8 / 1e6),
    }


def reached_edges(g, dist):
    reached = dist != (1 << 63) - 1
    return int(g.outdegrees()[reached].sum()), int(reached.sum())


def algorithmic_bytes(algo, edges, items):
    """per edge col 4 + dist[dst] 4 (+ weight 4 for SSSP); per
    frontier vertex row offset 8 + dist write 4 + queue write 4 + queue read 4."""
    return (12 if algo == "sssp" else 8) * edges + 20 * items


# ------------------------------------------------------------------- clocks
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


# ------------------------------------------------------------------ our arm
def run_params(pkg_lib, tag, algo, loop, timing=True):
    p = pkg_lib.RunParams()
    p.strategy = {"BS": 0, "EP": 1, "WD": 2, "NS": 3, "HP": 4}[tag]
    p.algo = pkg_lib.GLB_BFS if algo == "bfs" else pkg_lib.GLB_SSSP
    p.source = 0
    p.bins = 10
    p.chunked = 1
    p.mdt = 0
    p.max_cells = 1_000_000_000
    p.block_size = 1024
    p.hp_fallback = 1
    p.dist_bits = 0
    p.loop_mode = pkg_lib.GLB_LOOP_GRAPH if loop == "graph" else pkg_lib.GLB_LOOP_HOST
    p.record_timing = 1 if timing else 0
    return p


class DeviceRunner:
    """Direct C-ABI runs on the resident graph (no host copy of distances)."""

    def __init__(self, g, device):
        from paper_1711_00231_b200 import _lib

        self.L = _lib
        self.h = g.device_graph(device)
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


def ours(args):
    import torch
    import torch.distributed as dist

    import paper_1711_00231_b200 as pkg
    from paper_1711_00231_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = local if world > 1 else 0
    g, gen_s = workload(args, dev)
    runner = DeviceRunner(g, dev)

    # parity of the benchmarked configuration against the pinned oracle
    d_gpu = np.empty(g.num_nodes, dtype=np.int64)
    runner.run(args.strategy, args.algo, args.loop, d_gpu)
    e_r, n_r = reached_edges(g, d_gpu)
    parity = None
    cpu = None
    if rank == 0:
        from oracle import oracle

        oracle.build()
        exp = oracle.oracle_distances(g, 0, args.algo)
        parity = bool(np.array_equal(exp, d_gpu))

    # ---- timed region: K steps, barrier + synchronize on both sides
    launches0 = _lib.lib().glb_kernel_launches()
    clocks = ClockSampler(dev)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms, stats, recs = time_strategy(runner, torch, args.strategy, args.algo, args.loop,
                                    args.steps, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = _lib.lib().glb_kernel_launches() - launches0
    ms_step = ms / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = world * e_r / (ms_step / 1e3) / 1e9

    # ---- roofline of the dominant (relax) kernel over the timed steps
    k_ms = sum(r.kernel_ms for r in recs)
    k_bytes = sum(algorithmic_bytes(args.algo, r.work_total, r.active_items) for r in recs)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = k_bytes / (k_ms / 1e3) / 1e9 if k_ms > 0 else None
    # ncu DRAM traffic of the same kernel (one --set full capture, committed
    # under profiles/): traffic / algorithmic bytes measured on the captured
    # launches, applied to this run's mean algorithmic bytes per launch
    traffic = traffic_note = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        ps = json.loads(prof.read_text())
        ratio = ps.get(f"{args.strategy}_{args.algo}_traffic_over_algorithmic")
        if ratio and recs:
            traffic = int(ratio * k_bytes / len(recs))
            traffic_note = (f"ncu dram read+write / algorithmic bytes = {ratio} on the captured "
                            f"launches ({ps.get('source', '')})")
    # measured ceiling of this path's real bottleneck on the same graph: one
    # random 8 B cell gather per edge (dist[col[e]]) through L1TEX
    gp = (ctypes.c_double * 4)()
    _lib.check(_lib.lib().glb_measure_gather(runner.h, gp), "glb_measure_gather")
    k_edges = sum(r.work_total for r in recs)
    edge_rate = k_edges / (k_ms / 1e3) if k_ms > 0 else None
    gather = {
        "what": "dist[col[e]] gather rate on this graph's col array at full occupancy "
                "(glb_measure_gather), vs the dominant kernel's examined-edge rate",
        "gathers_per_s": round(gp[1] * 1e9, 0), "atomic_min_per_s": round(gp[2] * 1e9, 0),
        "col_stream_GBs": round(gp[0], 1), "cells_MB": round(gp[3], 1),
        "kernel_edges_per_s": round(edge_rate, 0) if edge_rate else None,
        "frac": round(edge_rate / (gp[1] * 1e9), 4) if edge_rate and gp[1] > 0 else None,
    }
    roofline = {
        "bound": "hbm",
        "achieved": round(achieved, 1) if achieved else None,
        "peak": peak,
        "unit": "GB/s",
        "frac": round(achieved / peak, 4) if achieved else None,
        "traffic": traffic,
        "traffic_source": traffic_note,
        "kernel": {"WD": "k_wd_relax", "HP": "k_hp_window", "BS": "k_bs_relax",
                   "NS": "k_ns_relax", "EP": "k_ep_relax"}[args.strategy],
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback",
        "algorithmic_bytes_per_launch": int(k_bytes / max(len(recs), 1)),
        "kernel_ms_per_launch": round(k_ms / max(len(recs), 1), 5),
        "kernel_share_of_step": round(k_ms / ms, 4) if ms else None,
        "relax_per_traversed_edge": round(stats[-1].relax_ops / max(e_r, 1), 3),
        "whole_step_frac": round(algorithmic_bytes(args.algo, e_r, n_r) / (ms_step / 1e3) / 1e9 / peak, 5),
        "gather_ceiling": gather,
    }

    # ---- e2e through the C-ABI with host buffers
    e2e = None
    if rank == 0 and args.e2e_steps > 0:
        L = _lib.lib()
        row, col, w = g.row_offsets, g.col_indices, g.weights
        out = np.empty(g.num_nodes, dtype=np.int64)
        times = []
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = ctypes.c_void_p()
            _lib.check(L.glb_graph_create(_lib.ptr64(row), _lib.ptr64(col), _lib.ptr64(w),
                                          g.num_nodes, g.num_edges, dev, ctypes.byref(h)))
            p = run_params(_lib, args.strategy, args.algo, args.loop)
            st = _lib.RunStats()
            _lib.check(L.glb_run(h, ctypes.byref(p), _lib.ptr64(out), ctypes.byref(st), None, 0))
            L.glb_graph_destroy(h)
            torch.cuda.synchronize()
            if i:  # first call warms the pinned staging ring
                times.append(time.perf_counter() - t0)
        assert np.array_equal(out, d_gpu)
        t = statistics.median(times)
        e2e = {"value": round(e_r / t / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(row.nbytes + col.nbytes + (w.nbytes if w is not None else 0)),
               "d2h_bytes_per_step": int(out.nbytes),
               "ms_per_step": round(t * 1e3, 2),
               "path": "C-ABI: glb_graph_create(host int64 CSR) + glb_run + int64 dist to host + destroy"}

    # ---- per-strategy table (not the headline)
    extras = {}
    if rank == 0 and not args.no_extras:
        for algo in ("sssp", "bfs"):
            tab = {}
            for tag in TAGS:
                ms_t, st_t, rr = time_strategy(runner, torch, tag, algo, args.loop, 3, 1)
                e_r_a = e_r
                if algo != args.algo:
                    dd = np.empty(g.num_nodes, dtype=np.int64)
                    runner.run(tag, algo, args.loop, dd)
                    e_r_a, _ = reached_edges(g, dd)
                kms = sum(r.kernel_ms for r in rr)
                tab[tag] = {"ms": round(ms_t / 3, 3), "gteps": round(e_r_a / (ms_t / 3 / 1e3) / 1e9, 3),
                            "launches": st_t[-1].launches, "iterations": st_t[-1].iterations,
                            "relax_per_edge": round(st_t[-1].relax_ops / max(e_r_a, 1), 3),
                            "kernel_share": round(kms / ms_t, 3) if ms_t else None}
            extras[algo] = tab

    # ---- CPU baseline: pinned C port of run_bs on the host cores
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(g, args, e_r)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (RMAT generated on the GPU, bit-identical to graphlb.generate_rmat)",
            "config": dict(workload_desc(args, g), parallelism=f"replicas{world}" if world > 1 else "single",
                           E_r=e_r, N_r=n_r, gen_s=round(gen_s, 1)),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches), "parity_vs_oracle": parity,
            "strategies": extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------- sharded (N > 1)
def ours_sharded(args, world, rank, local):
    """N ranks, one GPU each: RMAT scale args.scale + log2(N) (weak scaling:
    the same 2^(scale+4) edges per GPU as the 1-GPU C2 step), 1-D edge-balanced
    vertex partition, one NCCL all-to-all exchange of (dist << 32 | v)
    updates per BSP iteration plus an all-reduce of frontier sizes
    (paper_1711_00231_b200.sharded).  Each step is one full traversal from
    vertex 0; time = max over ranks of CUDA-event time, value = E_r of the
    whole graph / that time."""
    import math

    import torch
    import torch.distributed as dist

    import paper_1711_00231_b200 as pkg
    from paper_1711_00231_b200 import _lib, sharded

    backend = os.environ.get("GLB_BENCH_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    dev = local % max(ndev, 1)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    scale = args.scale + int(round(math.log2(world)))
    tag = args.strategy if args.strategy in sharded.SHARD_TAGS else "WD"
    t0 = time.time()
    g = pkg.generate_rmat(scale, args.edge_factor, seed=1, max_weight=255, device=dev,
                          download=False)
    bounds = sharded.partition_bounds(g, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    row = np.empty(g.num_nodes + 1, dtype=np.int64)
    _lib.check(_lib.lib().glb_graph_download(g.device_graph(), _lib.ptr64(row), None, None))
    deg_own = np.diff(row[lo:hi + 1])
    # self-check on rank 0: the single-GPU run on the full graph
    ref = None
    if rank == 0 and not args.no_check:
        ref = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(args.algo),
                               pkg.KernelConfig(loop="graph")).dist.array
    _lib.check(_lib.lib().glb_graph_restrict(g.device_graph(), lo, hi), "glb_graph_restrict")
    sg = sharded.ShardGraph(g, bounds, rank, dev)
    gen_s = time.time() - t0
    transport = sharded.DistTransport(torch)
    cfg = pkg.KernelConfig(record_timing=False)
    op = pkg.RelaxOp(args.algo)

    def step():
        return sharded.run_sharded(tag, sg, 0, op, cfg, transport)

    d_own, info = step()
    reached = d_own != (1 << 63) - 1
    t = torch.tensor([int(deg_own[reached].sum()), int(reached.sum())], dtype=torch.int64,
                     device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(t)
    e_r, n_r = int(t[0]), int(t[1])
    parity = None
    if not args.no_check:  # gather the owned ranges on rank 0 and compare
        full = [None] * world if rank == 0 else None
        dist.gather_object(d_own, full, dst=0)
        if rank == 0:
            parity = bool(np.array_equal(np.concatenate(full), ref))
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
    for _ in range(args.steps):
        _, inf = step()
        iters = inf["bsp_iterations"]
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = _lib.lib().glb_kernel_launches() - launches0
    ms_step = e0.elapsed_time(e1) / args.steps
    tt = torch.tensor([ms_step], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step = float(tt.item())
    value = e_r / (ms_step / 1e3) / 1e9

    # e2e: each rank uploads only its own rows from host int64 arrays, runs,
    # and reads its owned int64 distances back (max over ranks)
    e2e = None
    if args.e2e_steps > 0:
        # the device graph is already restricted: its download is the host shard
        hrow = np.empty(g.num_nodes + 1, dtype=np.int64)
        m_own = int(row[hi] - row[lo])
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
            d2, _ = sharded.run_sharded(tag, sharded.ShardGraph(dg, bounds, rank, dev), 0, op, cfg,
                                        transport)
            dg.release_device()
            torch.cuda.synchronize()
            if i:
                times.append(time.perf_counter() - t1)
        assert np.array_equal(d2, d_own)
        te = torch.tensor([statistics.median(times)], dtype=torch.float64,
                          device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        t_e2e = float(te.item())
        e2e = {"value": round(e_r / t_e2e / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(hrow.nbytes + hcol.nbytes + hw.nbytes),
               "d2h_bytes_per_step": int(d_own.nbytes), "ms_per_step": round(t_e2e * 1e3, 2),
               "path": "per rank: glb_graph_create(own rows, host int64) + sharded run + "
                       "owned int64 dist to host (bytes are rank 0's)"}
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
               "sample": "not run at N>1 (the CPU reference is timed on the 1-GPU workload)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (RMAT generated on each GPU, bit-identical to graphlb.generate_rmat)",
            "config": {
                "workload": (f"{args.algo.upper()} on RMAT scale-{scale} edge-factor "
                             f"{args.edge_factor} (0.45,0.15,0.15,0.25) seed 1, weights 1..255, "
                             f"source 0, 1-D edge-balanced vertex partition over {world} GPUs, "
                             f"{backend} all-to-all exchange per BSP iteration"),
                "strategy": tag, "nodes": g.num_nodes, "edges": int(row[-1]),
                "parallelism": f"shard{world}", "E_r": e_r, "N_r": n_r,
                "bsp_iterations": iters, "gen_s": round(gen_s, 1),
                "l2": "inputs larger than L2; no flush"},
            "roofline": None, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches), "parity_vs_single_gpu": parity,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def cpu_baseline(g, args, e_r):
    from oracle import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    w = g.weights if args.algo == "sssp" else None
    t0 = time.perf_counter()
    d, it, ops = oracle.bs_run(g.row_offsets, g.col_indices, w, 0, threads)
    t = time.perf_counter() - t0
    return {"value": round(e_r / t / 1e9, 5), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"one full {args.algo.upper()} run_bs traversal of the benchmark graph "
                      f"({t:.2f} s, {it} iterations, {ops} relaxations)"}


# ------------------------------------------------------------ reference arm
def _has_gpu() -> bool:
    try:
        from paper_1711_00231_b200 import _lib

        return _lib.device_count() > 0
    except Exception:
        return False


def _host_workload(args):
    import paper_1711_00231_b200 as pkg

    t0 = time.time()
    g = pkg.generate_rmat(args.scale, args.edge_factor, seed=1, max_weight=255)
    return g, time.time() - t0


def reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle

    oracle.build()
    g, gen_s = workload(args) if _has_gpu() else _host_workload(args)
    threads = os.cpu_count() or 1
    w = g.weights if args.algo == "sssp" else None
    times = []
    d = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        d, it, ops = oracle.bs_run(g.row_offsets, g.col_indices, w, 0, threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    e_r, n_r = reached_edges(g, d)
    t = sum(times) / len(times)
    value = e_r / t / 1e9
    sample = (f"each step = one full {args.algo.upper()} node-based (run_bs) traversal of the "
              f"benchmark graph, C port of node_based.py:19-82 on {threads} threads")
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (RMAT generated in-process, bit-identical to graphlb.generate_rmat)",
        "config": dict(workload_desc(args, g), strategy="BS", E_r=e_r, N_r=n_r),
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        reference(a)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        ours_sharded(a, int(os.environ["WORLD_SIZE"]), int(os.environ.get("RANK", "0")),
                     int(os.environ.get("LOCAL_RANK", "0")))
    else:
        ours(a)
