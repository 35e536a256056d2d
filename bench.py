#!/usr/bin/env python3
"""bench.py — GTEPS of the edgeset.apply hot path (PageRank 20 iters + BFS) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
                    [--mode partition|replicas]

Workload. BASELINE.json's metric names no config, so N = 1 runs the largest
single-GPU config: configs[3] = "config 4", RMAT scale 25, edge factor 48
(~1.56 B directed edges after cleanup; stands in for Twitter). One step
= the whole hot path: fixed-iteration PageRank (20
iterations, d = 0.85, pull) plus BFS from the config's 16 seeded sources
(direction-optimising; gi_bfs_multi: one bit-parallel pass). The graph build
(a1) runs once before timing and is reported separately (`build_ms`), with the
first PageRank call, which also builds the segmented-pull layout
(`pr_first_call_ms`). `secondary` repeats the device-timed measurement on
config 2 (RMAT s22, 64 sources), the round-1 headline.

value  = (20 m + sum over sources of edges traversed (R16)) / device time,
         all ranks (GTEPS), inputs resident in HBM, CUDA events on the
         library's stream; inputs (CSR + CSC ~ 12 GB) are larger than L2.
e2e    = the same edges over the wall time of the public C-ABI calls with
         HOST buffers: gi_graph_create from pinned host edges (H2D inside),
         gi_pagerank into host memory, gi_bfs_multi into host memory.
roofline: the pull-PageRank iteration (the north_star's >= 50% target):
         algorithmic bytes 4m + (o+12)n per iteration / its
         CUDA-event duration (edge pass + vertex pass); `traffic` = ncu DRAM
         bytes of the same kernels for this config from profiles/ncu_summary.json
         (`traffic_source` names the capture); `roofline.atomics`: the
         segmented edge pass's second bound, its RED.ADD.F32 per piece
         (gi_pr_stats.reductions_per_iter) against the measured random-RED
         rate, with the iteration time that bound allows; roofline_bfs: the bit-parallel
         pull level (k_ms_pull + k_ms_pull_heavy), 4 B per in-edge read + 20 B
         per vertex.
cpu_baseline: the oracle (oracle/, plain C, OpenMP) on a bounded sample of
         the same graph on all host cores, plus one-core numbers on config 2.

Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) when
WORLD_SIZE is unset and aborts if the world size differs from N. The default
for N > 1 is the north_star's design, `--mode partition`: 1-D destination-range
partition, every rank generating and passing its own share of the edge list,
an NCCL allgather of contrib slices / frontier bitmaps every iteration / level
(SURVEY §8(e)); the job is fixed as N grows (strong scaling); its BFS is a loop
of distributed single-source traversals. `--mode replicas` (opt-in) runs N
independent copies, each with its own seeded batch of sources (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS for PageRank iteration and BFS; achieved fraction of HBM roofline"
# the paper's own numbers for the graphs the configs stand in for (context only: other hardware,
# other datasets; BASELINE.md derives GTEPS from the paper's seconds and its edge counts)
PAPER_CONTEXT = {
    "hardware": "2x Intel Xeon E5-2695 v3 (24 cores, 48 threads), 128 GB DDR3-1600 (PAPER.md P:2194-2197)",
    "graphit_pr_20iter_s": {"twitter_1.47B": 8.707, "livejournal_69M": 0.342, "friendster_3.6B": 32.571},
    "graphit_pr_gteps": {"twitter_1.47B": 3.37, "livejournal_69M": 4.04, "friendster_3.6B": 2.21},
    "graphit_bfs_s_per_source": {"twitter_1.47B": 0.298, "livejournal_69M": 0.035, "friendster_3.6B": 0.490},
    "source": "Table 4, PAPER.md P:2291; GTEPS derived in BASELINE.md (edges x iterations / seconds)",
}
DEFAULT_CONFIG = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-2 secondary measurement")
    ap.add_argument("--pr-direction", default="pull", choices=["pull", "push", "direct", "segmented"])
    ap.add_argument("--mode", default=None, choices=["partition", "replicas"],
                    help="N > 1: the destination-partitioned graph over NCCL (default; SURVEY §8(e), strong "
                         "scaling) or N independent replicas with their own source batches (weak scaling)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def relaunch_if_needed(args):
    """--gpus N > 1 without torchrun: re-exec this script under torch.distributed.run with N ranks."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    _, world, _ = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"world size {world} != --gpus {args.gpus}"}), flush=True)
        sys.exit(2)


# random RED.ADD.F32 into an L2-resident 16 MB array, all SMs (tools/microbench/red_rates.cu)
RED_PEAK_GOPS = 180.1
RED_PEAK_SOURCE = "measured: profiles/r01_red_rates.txt (random RED.ADD.F32, 16 MB array, 148 SMs)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(cfg_name):
    """Per-launch DRAM bytes (ncu --set full) of this config's PR iteration and BFS pull level from the
    committed summary (profiles/ncu_summary.json, key configs/<name>); missing entries are None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    out = {"pr_pull": None, "bfs_pull": None, "source": None}
    if os.path.exists(p):
        try:
            d = json.load(open(p)).get("configs", {}).get(cfg_name, {})
            for k in ("pr_pull", "bfs_pull"):
                out[k] = d.get(k, {}).get("dram_bytes_per_launch")
            out["source"] = d.get("sources")
        except Exception:
            pass
    return out


def host_info():
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def bench_config(cfg, n, m, k, args, world, mode):
    """The `config` object of the JSON line (both arms print the same one)."""
    par = "single" if world == 1 else (
        f"dst-partition x{world} (NCCL allgather of contrib / frontier bitmap per iteration / level)"
        if mode == "partition" else f"replicas x{world}")
    return {"workload": f"{cfg.name} (BASELINE configs[{cfg.idx - 1}])", "n": n, "m": m,
            "pr_iters": cfg.pr_iters, "damping": cfg.damping, "bfs_sources": k,
            "pr_direction": args.pr_direction,
            "bfs_policy": ("auto: bit-parallel pass of up to 64 sources, pull iff |F| + sum outdeg F > m/8 "
                           "(m/12 when 16n bytes of vertex state exceed L2) or a listed-row pull is cheaper; dense "
                           "pulls as segmented OR passes when the graph has the layout"
                           if mode != "partition" or world == 1 else
                           "auto per source: pull iff |F| + sum outdeg F > m/20 (distributed level loop)"),
            "l2": "inputs larger than L2 (CSR+CSC ~ 8m bytes > 126 MB), no flush",
            "parallelism": par}


def gen_edges(cfg, device_ok, first=0, count=None):
    """Edge list of cfg (or the slice [first, first+count) of its RMAT stream): device generator when
    allowed (bit-exact twin of the host one), returned as host numpy arrays and device tensors."""
    import graphgen

    if cfg.kind == "rmat" and device_ok:
        a, b, c, _ = cfg.abcd
        ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed, first=first, count=count)
        return ts, td
    if cfg.kind == "rmat":
        a, b, c, _ = cfg.abcd
        return graphgen.rmat(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed, first=first, count=count)
    s, d = cfg.edges()
    if count is not None:
        s, d = s[first:first + count].copy(), d[first:first + count].copy()
    return s, d


# ---------------------------------------------------------------------------------------------- reference arm
def oracle_sample(g, cfg, sources, pr_iters, nsrc):
    """One bounded sample of the workload through the oracle: pr_iters PageRank iterations + BFS from nsrc
    sources (level-synchronous depths, OpenMP). Returns (edges, seconds)."""
    import oracle

    t0 = time.perf_counter()
    edges = 0
    if pr_iters:
        oracle.pagerank(g, pr_iters, cfg.damping)
        edges += g.m * pr_iters
    for src in sources[:nsrc]:
        dep = oracle.bfs_depth_levels(g, int(src))
        edges += oracle.reached_out_edges(g, dep)
    return edges, time.perf_counter() - t0


def run_reference(args):
    """The oracle (plain C, fp64 PR, level-synchronous BFS), as it stands, on this host's cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import graphgen
    import oracle

    cfg = graphgen.CONFIGS[args.config]
    s, d = gen_edges(cfg, device_ok=False)
    sources = cfg.sources(s, d)
    t = time.perf_counter()
    g = oracle.build_graph(cfg.n, s, d, symmetrize=cfg.symmetrize)
    build_s = time.perf_counter() - t
    del s, d
    pr_iters, nsrc = 1, 1
    for _ in range(args.warmup):
        oracle_sample(g, cfg, sources, pr_iters, nsrc)
    tot_e, tot_t = 0, 0.0
    for i in range(args.steps):
        e, dt = oracle_sample(g, cfg, list(sources[i % len(sources):]) + list(sources), pr_iters, nsrc)
        tot_e += e
        tot_t += dt
    gteps = tot_e / tot_t / 1e9
    info = host_info()
    sample = (f"{cfg.name}: per step oracle PageRank {pr_iters} iteration + level-synchronous BFS from "
              f"{nsrc} of the {len(sources)} sources (oracle graph build {build_s:.1f} s untimed)")
    line = {
        "impl": "reference", "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded RMAT/grid generators; paper datasets not available)",
        "config": bench_config(cfg, cfg.n, g.m, len(sources), args, 1, "single"),
        "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": oracle.set_threads(0), "kind": "oracle",
                         "sample": sample, **info},
        "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------- our arm
def cpu_baseline(cfg, s, d, sources):
    """Oracle GTEPS on all host cores (a bounded sample of this workload) and on one core (config 2)."""
    import graphgen
    import oracle

    info = host_info()
    cores = oracle.set_threads(0)
    t = time.perf_counter()
    g = oracle.build_graph(cfg.n, s, d, symmetrize=cfg.symmetrize)
    build_s = time.perf_counter() - t
    e_pr, t_pr = oracle_sample(g, cfg, sources, 2, 0)
    e_bfs, t_bfs = oracle_sample(g, cfg, sources, 0, 2)
    del g
    out = {"value": (e_pr + e_bfs) / (t_pr + t_bfs) / 1e9, "unit": "GTEPS", "cores": cores, "kind": "oracle",
           "sample": (f"{cfg.name}: oracle PageRank 2 iterations ({t_pr:.1f} s) + level-synchronous BFS from 2 of "
                      f"the sources ({t_bfs:.1f} s) on {cores} threads; oracle graph build {build_s:.1f} s untimed"),
           "pr_gteps": e_pr / t_pr / 1e9, "bfs_gteps": e_bfs / t_bfs / 1e9, **info}
    # one core, config 2 (BASELINE.md CPU-baseline plan: 1-core oracle time for configs 1-2)
    c2 = graphgen.CONFIGS[2]
    s2, d2 = c2.edges()
    g2 = oracle.build_graph(c2.n, s2, d2)
    src2 = c2.sources(s2, d2)
    prev = oracle.set_threads(1)
    try:
        e1, t1 = oracle_sample(g2, c2, src2, 1, 0)
        t0 = time.perf_counter()
        dep = oracle.bfs_depth(g2, int(src2[0]))  # the plain FIFO BFS
        tb = time.perf_counter() - t0
        eb = oracle.reached_out_edges(g2, dep)
    finally:
        oracle.set_threads(prev)
    out["single_core"] = {"config": c2.name, "pr_gteps": e1 / t1 / 1e9, "pr_s_per_iter": t1,
                          "bfs_fifo_gteps": eb / tb / 1e9, "bfs_fifo_s": tb, "cores": 1}
    return out


def measure_graph(g, cfg, srcs, args, stream, dev, world, direction, gi):
    """Warm-up, timed steps, per-phase timings and rooflines of one built graph (device-resident)."""
    import torch

    n, m = g.n, g.m
    pr_out = torch.empty(n, dtype=torch.float32, device=dev)
    bfs_out = torch.empty((len(srcs), n), dtype=torch.int32, device=dev)  # one parent row per source

    def step():
        _, ps = g.pagerank(cfg.pr_iters, cfg.damping, out=pr_out, direction=direction)
        _, bss = g.bfs_multi(srcs, out=bfs_out)
        launches = ps.edge_launches + ps.aux_launches + sum(b.launches for b in bss)
        return cfg.pr_iters * m, sum(b.edges_traversed for b in bss), launches

    torch.cuda.synchronize()
    t = time.perf_counter()
    g.pagerank(cfg.pr_iters, cfg.damping, out=pr_out, direction=direction)  # builds + calibrates the layout
    torch.cuda.synchronize()
    first_pr_ms = (time.perf_counter() - t) * 1e3
    for _ in range(max(args.warmup, 0)):
        step()
    # phase timings (PR vs BFS), outside the main timed region
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    g.pagerank(cfg.pr_iters, cfg.damping, out=pr_out, direction=direction)
    ev[1].record(stream)
    _, bss = g.bfs_multi(srcs, out=bfs_out)
    ev[2].record(stream)
    torch.cuda.synchronize()
    pr_ms, bfs_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])

    # timed region
    sampler = ClockSampler(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tot_pr = tot_bfs = launches = 0
    for _ in range(args.steps):
        a, b, l = step()
        tot_pr += a
        tot_bfs += b
        launches += l
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)

    # rooflines, kernel durations from CUDA events on the library's stream
    peak, peak_src = load_peaks()
    traffic = load_traffic(cfg.name)
    _, ps = g.pagerank(cfg.pr_iters, cfg.damping, out=pr_out, direction=direction, profile=True)
    kern_ms = ps.edge_ms / max(ps.edge_launches, 1)  # one iteration: edge pass + vertex pass
    achieved = ps.bytes_alg_per_iter / (kern_ms * 1e-3) / 1e9
    kname = {gi.GI_PR_PULL_SEGMENTED: "k_pr_seg + k_pr_acc (segmented pull edge pass + vertex update)",
             gi.GI_PR_PULL_DIRECT: "k_pr_pull / k_pr_rows (direct pull with fused vertex update)",
             gi.GI_PR_PUSH: "k_pr_push + k_pr_vertex"}.get(ps.kernel, str(ps.kernel))
    roofline_pr = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                   "traffic": traffic.get("pr_pull"), "traffic_source": traffic.get("source"),
                   "kernel": kname + ", per iteration",
                   "bytes_alg_per_launch": ps.bytes_alg_per_iter,
                   "bytes_alg_formula": "4m + (o+12)n, o = offset bytes (SURVEY §8(d))", "launch_ms": kern_ms,
                   "vertex_ms": ps.vertex_ms / max(ps.edge_launches, 1), "peak_source": peak_src,
                   "pr_total_ms": ps.total_ms}
    if ps.reductions_per_iter > 0:
        # the segmented pass's second bound: one RED.ADD.F32 per piece into the L2-resident accumulator,
        # against the measured random-RED rate of this part
        edge_only_ms = kern_ms - roofline_pr["vertex_ms"]
        red_gops = ps.reductions_per_iter / (edge_only_ms * 1e-3) / 1e9
        floor_ms = ps.reductions_per_iter / (RED_PEAK_GOPS * 1e9) * 1e3 + roofline_pr["vertex_ms"]
        roofline_pr["atomics"] = {
            "bound": "l2_atomics", "reductions_per_launch": ps.reductions_per_iter, "edge_pass_ms": edge_only_ms,
            "achieved": red_gops, "peak": RED_PEAK_GOPS, "unit": "Gops/s", "frac": red_gops / RED_PEAK_GOPS,
            "peak_source": RED_PEAK_SOURCE, "iteration_floor_ms": floor_ms,
            "hbm_frac_at_floor": ps.bytes_alg_per_iter / (floor_ms * 1e-3) / 1e9 / peak,
            "record_bytes_per_launch": ps.stream_bytes_per_iter}
    if world > 1:
        roofline_pr["exchange"] = {0: "none", 1: "allgatherv per iteration", 2: "peer stores"}[ps.exchange]
        roofline_pr["exchange_ms_per_iter"] = ps.exchange_ms / max(ps.edge_launches, 1)
    _, bsp = g.bfs_multi(srcs, out=bfs_out, profile=True)
    bfs_pass_ms = sum(b.total_ms for b in bsp)
    pull_ms = sum(b.pull_ms for b in bsp)
    if pull_ms > 0:
        pull_levels = max(b.pull_levels for b in bsp)
        pull_edges = sum(b.pull_edges_examined for b in bsp)
        bfs_bytes = (4 * pull_edges + 20 * n * pull_levels) / pull_levels
        bfs_launch_ms = pull_ms / pull_levels
        bfs_kernel = ("bit-parallel multi-source BFS, one pull level over "
                      f"{len(srcs)} sources (averaged over the pass's segmented-OR, row and listed-row pull levels: "
                      "k_pr_seg<OpOr> + k_ms_or_vertex + k_ms_resolve_heavy / k_ms_pull + k_ms_pull_heavy)")
    else:
        bfs_launch_ms = bfs_pass_ms / max(len(bsp), 1)
        bfs_bytes = sum(4 * b.edges_examined + 4 * b.pull_vertices + 8 * b.reached for b in bsp) / max(len(bsp), 1)
        bfs_kernel = "k_bfs_fused / distributed level loop (direction-optimising BFS, per source)"
    bfs_achieved = bfs_bytes / (bfs_launch_ms * 1e-3) / 1e9 if bfs_launch_ms > 0 else 0.0
    roofline_bfs = {"bound": "hbm", "achieved": bfs_achieved, "peak": peak, "unit": "GB/s",
                    "frac": bfs_achieved / peak, "traffic": traffic.get("bfs_pull"),
                    "kernel": bfs_kernel, "bytes_alg_per_launch": bfs_bytes, "launch_ms": bfs_launch_ms,
                    "pass_ms": bfs_pass_ms, "peak_source": peak_src,
                    "edges_examined_per_source": sum(b.edges_examined for b in bsp) / max(len(bsp), 1)}
    return {"ms": ms, "tot_pr": tot_pr, "tot_bfs": tot_bfs, "launches": launches, "clocks": clocks,
            "pr_ms": pr_ms, "bfs_ms": bfs_ms, "first_pr_ms": first_pr_ms, "roofline_pr": roofline_pr,
            "roofline_bfs": roofline_bfs}


def secondary_config2(ctx, args, stream, dev, direction, gi):
    """Device-timed PR + 64-source BFS on config 2 (RMAT s22 ef16, the round-1 headline)."""
    import torch

    import graphgen

    cfg = graphgen.CONFIGS[2]
    s, d = cfg.edges()
    srcs = [int(x) for x in cfg.sources(s, d)]
    g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev),
                 gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
    r = measure_graph(g, cfg, srcs, argparse.Namespace(steps=args.steps, warmup=args.warmup), stream, dev, 1,
                      direction, gi)
    m = g.m
    g.close()
    return {"workload": f"{cfg.name} (BASELINE configs[1])", "m": m, "bfs_sources": len(srcs),
            "value": (r["tot_pr"] + r["tot_bfs"]) / (r["ms"] * 1e-3) / 1e9, "unit": "GTEPS",
            "ms_per_step": r["ms"] / args.steps,
            "pr_gteps": cfg.pr_iters * m / (r["pr_ms"] * 1e-3) / 1e9,
            "bfs_gteps": (r["tot_bfs"] / args.steps) / (r["bfs_ms"] * 1e-3) / 1e9,
            "roofline_pr_frac": r["roofline_pr"]["frac"], "roofline_pr_launch_ms": r["roofline_pr"]["launch_ms"],
            "roofline_bfs_frac": r["roofline_bfs"]["frac"]}


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    mode = args.mode or ("partition" if world > 1 else "single")
    # diagnostics: GI_BENCH_DEVICE pins every rank to one GPU and GI_BENCH_DIST_BACKEND=gloo runs the
    # host-side collectives on CPU tensors (replicas path only)
    gpu = int(os.environ.get("GI_BENCH_DEVICE", local))
    backend = os.environ.get("GI_BENCH_DIST_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(gpu)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cdev = dev if backend == "nccl" else "cpu"  # where the timing reductions live
    import graphgen
    from paper_1805_00923_b200 import gi

    stream = torch.cuda.Stream()
    partition = world > 1 and mode == "partition"
    if partition and backend != "nccl":
        # diagnostics (GI_BENCH_DIST_BACKEND=gloo): the library's collectives staged through host memory into
        # the gloo group (gi_context_create_hostcomm) — the partitioned path end to end on one shared GPU
        from paper_1805_00923_b200.hostcomm import TorchDistComm

        ctx = gi.Context(dev, stream.cuda_stream, hostcomm=(rank, world, TorchDistComm()))
    elif partition:  # NCCL communicator of the library; torch.distributed only ships the unique id
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(gi.gi_nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        ctx = gi.Context(dev, stream.cuda_stream, nccl=(rank, world, bytes(uid.cpu().numpy().tobytes())))
    else:
        ctx = gi.Context(dev, stream.cuda_stream)
    cfg = graphgen.CONFIGS[args.config]
    flags = gi.GI_DEFAULT_FLAGS | (gi.GI_SYMMETRIZE if cfg.symmetrize else 0)
    direction = {"pull": gi.GI_PR_PULL, "push": gi.GI_PR_PUSH, "direct": gi.GI_PR_PULL_DIRECT,
                 "segmented": gi.GI_PR_PULL_SEGMENTED}[args.pr_direction]

    t = time.perf_counter()
    if partition:
        # every rank generates (on its GPU) and passes its own slice of the edge stream; sources come from
        # the OR over ranks of "has a non-self-loop out-edge" (the same draw as N = 1)
        total = cfg.edge_factor * cfg.n if cfg.kind == "rmat" else None
        if total is None:
            s_all, d_all = cfg.edges()
            total = len(s_all)
        lo, hi = total * rank // world, total * (rank + 1) // world
        ts, td = gen_edges(cfg, device_ok=True, first=lo, count=hi - lo) if cfg.kind == "rmat" else \
            (torch.from_numpy(s_all[lo:hi].copy()).to(dev), torch.from_numpy(d_all[lo:hi].copy()).to(dev))
        s, d = ts.cpu().numpy(), td.cpu().numpy()  # this rank's share (e2e input)
        elig = torch.zeros(cfg.n, dtype=torch.int32, device=dev)
        keep = ts != td
        elig[ts[keep].long()] = 1
        elig = elig.to(cdev)
        torch.distributed.all_reduce(elig)
        sources = graphgen.pick_sources_from_mask(cfg.n, elig.cpu().numpy(), cfg.bfs_sources, cfg.source_seed) \
            if cfg.source_seed else np.zeros(1, np.int32)
        del elig, keep
    else:
        ts, td = gen_edges(cfg, device_ok=True)
        if not isinstance(ts, torch.Tensor):
            ts, td = torch.from_numpy(ts).to(dev), torch.from_numpy(td).to(dev)
        s, d = ts.cpu().numpy(), td.cpu().numpy()  # host copies: sources, e2e input, cpu baseline
        sources = cfg.sources(s, d)
        if world > 1 and cfg.source_seed and rank > 0:  # replicas: every rank its own seeded batch
            sources = graphgen.pick_sources(cfg.n, s, d, cfg.bfs_sources, cfg.source_seed + rank)
    gen_s = time.perf_counter() - t

    torch.cuda.synchronize()
    t = time.perf_counter()
    g = gi.Graph(ctx, cfg.n, ts, td, flags | gi.GI_EDGES_ON_DEVICE)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t) * 1e3
    del ts, td
    torch.cuda.empty_cache()
    n, m = g.n, g.m
    srcs = [int(x) for x in sources]

    r = measure_graph(g, cfg, srcs, args, stream, dev, world, direction, gi)
    ms = r["ms"]
    if world > 1:
        tt = torch.tensor([ms, r["tot_pr"] + r["tot_bfs"]], dtype=torch.float64, device=cdev)
        mx = tt.clone()
        torch.distributed.all_reduce(mx[:1], op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(tt[1:], op=torch.distributed.ReduceOp.SUM)
        # partition: every rank reports the same global edge count (one job); replicas: N jobs
        ms_max, edges_all = float(mx[0]), float(tt[1]) / (world if partition else 1)
    else:
        ms_max, edges_all = ms, float(r["tot_pr"] + r["tot_bfs"])
    value = edges_all / (ms_max * 1e-3) / 1e9

    # e2e through the public API with host buffers (single GPU / replicas: the whole graph per rank;
    # partition: every rank passes its own share of the edge list)
    e2e = None
    if not args.no_e2e:
        g.close()  # HBM for the per-step graphs
        torch.cuda.empty_cache()
        hs = torch.from_numpy(s).pin_memory()
        hd = torch.from_numpy(d).pin_memory()
        hpr = torch.empty(n, dtype=torch.float32).pin_memory()
        hbfs = torch.empty((len(srcs), n), dtype=torch.int32).pin_memory()
        # one untimed end-to-end step first (first touch of the pinned buffers and of the allocation pool)
        gw = gi.Graph(ctx, cfg.n, hs, hd, flags)
        gw.pagerank(cfg.pr_iters, cfg.damping, out=hpr, direction=direction)
        gw.bfs_multi(srcs, out=hbfs)
        gw.close()
        torch.cuda.synchronize()
        e2e_steps = max(1, min(args.steps, 5))
        e_edges = 0
        phases = []
        t = time.perf_counter()
        for _ in range(e2e_steps):
            tp = [time.perf_counter()]
            g2 = gi.Graph(ctx, cfg.n, hs, hd, flags)
            tp.append(time.perf_counter())
            g2.pagerank(cfg.pr_iters, cfg.damping, out=hpr, direction=direction)
            tp.append(time.perf_counter())
            e_edges += cfg.pr_iters * g2.m
            _, bss2 = g2.bfs_multi(srcs, out=hbfs)
            tp.append(time.perf_counter())
            e_edges += sum(b.edges_traversed for b in bss2)
            g2.close()
            tp.append(time.perf_counter())
            phases.append([round((b - a) * 1e3, 1) for a, b in zip(tp, tp[1:])])
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t
        e_all = float(e_edges)
        if world > 1:
            te = torch.tensor([e2e_s], dtype=torch.float64, device=cdev)
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(te[0])
            if not partition:  # replicas: every rank's own job; partition: one job, same count on every rank
                ta = torch.tensor([e_all], dtype=torch.float64, device=cdev)
                torch.distributed.all_reduce(ta, op=torch.distributed.ReduceOp.SUM)
                e_all = float(ta[0])
        e2e = {"value": e_all / e2e_s / 1e9, "unit": "GTEPS",
               "h2d_bytes_per_step": int(8 * len(s)),
               "d2h_bytes_per_step": int(4 * n * (1 + len(srcs))), "steps": e2e_steps,
               "step_phases_ms": {"columns": ["gi_graph_create (H2D + build)", "gi_pagerank (+ layout build)",
                                              "gi_bfs_multi (+ D2H)", "gi_graph_destroy"], "steps": phases},
               "includes": "gi_graph_create from pinned host edges + gi_pagerank + gi_bfs_multi over the "
                           "sources, host outputs; one untimed warm-up step"}
    else:
        g.close()

    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary and args.config != 2:
        try:
            secondary = secondary_config2(ctx, args, stream, dev, direction, gi)
        except Exception as e:  # reported, never fatal to the headline line
            secondary = {"error": repr(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, s, d, sources)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if partition else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded counter-based RMAT; stands in for Twitter, paper datasets unavailable)"
            if args.config == 4 else "synthetic (seeded generators; paper datasets unavailable)",
            "config": bench_config(cfg, n, m, len(srcs), args, world, mode),
            "e2e": e2e, "gpu_launches": r["launches"], "roofline": r["roofline_pr"],
            "roofline_bfs": r["roofline_bfs"], "cpu_baseline": cpu, "clocks": r["clocks"],
            "pr_gteps": cfg.pr_iters * m / (r["pr_ms"] * 1e-3) / 1e9, "pr_ms": r["pr_ms"],
            "bfs_gteps": (r["tot_bfs"] / args.steps) / (r["bfs_ms"] * 1e-3) / 1e9 if r["bfs_ms"] > 0 else None,
            "bfs_ms_per_source": r["bfs_ms"] / max(len(srcs), 1), "build_ms": build_ms,
            "pr_first_call_ms": r["first_pr_ms"], "gen_s": gen_s, "secondary": secondary,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init log shows every rank joining
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    relaunch_if_needed(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
