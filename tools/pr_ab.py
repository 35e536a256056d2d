#!/usr/bin/env python3
"""A/B of PageRank kernel variants: best per-iteration time (edge + vertex pass) of 20-iteration runs.

    GI_LIBGI=paper_1805_00923_b200/libgi_NAME.so python tools/pr_ab.py NAME CONFIG
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

name, ci = sys.argv[1], int(sys.argv[2])
cfg = graphgen.CONFIGS[ci]
if cfg.kind == "rmat":
    a, b, c, _ = cfg.abcd
    ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
else:
    s, d = cfg.edges()
    ts, td = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
ctx = gi.Context(0)
flags = gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE | (gi.GI_SYMMETRIZE if cfg.symmetrize else 0)
g = gi.Graph(ctx, cfg.n, ts, td, flags)
del ts, td
torch.cuda.empty_cache()
out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
kw = {}
if os.environ.get("GI_AB_DSTBLOCK"):  # segmented pull: destination rows per block (0 = auto)
    kw = dict(direction=gi.GI_PR_PULL_SEGMENTED, dst_block=int(os.environ["GI_AB_DSTBLOCK"]))
for _ in range(3):
    g.pagerank(20, 0.85, out=out, **kw)
best, bv = 1e9, 0
for _ in range(5):
    _, st = g.pagerank(20, 0.85, out=out, profile=True, **kw)
    if st.edge_ms / st.edge_launches < best:
        best, bv = st.edge_ms / st.edge_launches, st.vertex_ms / st.edge_launches
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6443.2
frac = st.bytes_alg_per_iter / (best * 1e-3) / 1e9 / peak
print(json.dumps({"variant": name, "config": cfg.name, "ms_per_iter": round(best, 4), "vertex_ms": round(bv, 4),
                  "frac": round(frac, 3), "kernel": st.kernel}), flush=True)
