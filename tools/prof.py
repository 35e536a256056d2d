#!/usr/bin/env python3
"""Short driver for ncu: build one config, run PageRank and BFS a few times.

    python tools/prof.py [--config 2] [--pr-iters 3] [--bfs 2] [--direction pull]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--pr-iters", type=int, default=3)
ap.add_argument("--pr-reps", type=int, default=1)
ap.add_argument("--bfs", type=int, default=2)
ap.add_argument("--direction", default="pull")
args = ap.parse_args()

cfg = graphgen.CONFIGS[args.config]
if args.config in (4, 5):  # billion-edge configs: device generator, sources = first vertices with out-edges
    a, b, c, _ = cfg.abcd
    ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
    srcs = None
else:
    s, d = cfg.edges()
    srcs = cfg.sources(s, d)
    ts, td = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
ctx = gi.Context(0)
flags = gi.GI_DEFAULT_FLAGS | (gi.GI_SYMMETRIZE if cfg.symmetrize else 0)
g = gi.Graph(ctx, cfg.n, ts, td, flags | gi.GI_EDGES_ON_DEVICE)
del ts, td
if srcs is None:
    od = g.out_degrees(torch.empty(cfg.n, dtype=torch.int32, device="cuda"))
    srcs = torch.nonzero(od > 0).flatten()[:max(args.bfs, 1)].cpu().numpy()
out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
par = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
direction = {"pull": gi.GI_PR_PULL, "push": gi.GI_PR_PUSH, "direct": gi.GI_PR_PULL_DIRECT,
             "segmented": gi.GI_PR_PULL_SEGMENTED}[args.direction]
for _ in range(args.pr_reps):
    t = time.perf_counter()
    _, st = g.pagerank(args.pr_iters, cfg.damping, out=out, direction=direction, profile=True)
    print(f"pr: {st.edge_ms / max(st.edge_launches, 1):.4f} ms/iter (vertex {st.vertex_ms / max(st.edge_launches, 1):.4f}), total {st.total_ms:.3f} ms, "
          f"{st.bytes_alg_per_iter / (st.edge_ms / st.edge_launches * 1e-3) / 1e9:.1f} GB/s alg")
for src in srcs[: args.bfs]:
    _, bs = g.bfs(int(src), out=par, profile=True)
    print(f"bfs src={int(src)}: levels={bs.levels} pull={bs.pull_levels} reached={bs.reached} "
          f"edges={bs.edges_traversed} {bs.total_ms:.3f} ms")
g.close()
ctx.close()
