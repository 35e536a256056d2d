"""CPU oracle throughput per config (the CPU baseline beyond the bench's workload): the oracle's
PageRank iteration and BFS (FIFO single-thread, level-synchronous on all cores) on configs 1-3,
GTEPS as the bench counts them (PR: m per iteration; BFS: out-degrees of the reached vertices).
The oracle is test infrastructure: timed as it stands, never tuned.

usage: python tools/oracle_configs.py [CONFIG ...]   (JSON lines)
"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import oracle  # noqa: E402


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


cores = os.cpu_count()
for ci in [int(x) for x in sys.argv[1:]] or [1, 2, 3]:
    cfg = graphgen.CONFIGS[ci]
    s, d = cfg.edges()
    t = time.perf_counter()
    g = oracle.build_graph(cfg.n, s, d, symmetrize=cfg.symmetrize)
    build_s = time.perf_counter() - t
    src = int(cfg.sources(s, d)[0]) if cfg.source_seed else 0
    out = {"config": cfg.name, "n": cfg.n, "m": g.m, "cpu_model": cpu_model(), "cores": cores,
           "oracle_build_s": round(build_s, 2)}
    for threads in (1, cores):
        oracle.set_threads(threads)
        t = time.perf_counter()
        oracle.pagerank(g, 2, cfg.damping)
        pr_s = (time.perf_counter() - t) / 2
        out[f"pr_gteps_{threads}t"] = round(g.m / pr_s / 1e9, 4)
        t = time.perf_counter()
        dep = oracle.bfs_depth_levels(g, src)
        bl_s = time.perf_counter() - t
        out[f"bfs_levels_gteps_{threads}t"] = round(oracle.reached_out_edges(g, dep) / bl_s / 1e9, 4)
    t = time.perf_counter()
    dep = oracle.bfs_depth(g, src)
    bf_s = time.perf_counter() - t
    out["bfs_fifo_gteps_1t"] = round(oracle.reached_out_edges(g, dep) / bf_s / 1e9, 4)
    print(json.dumps(out), flush=True)
