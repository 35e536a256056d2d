#!/usr/bin/env python3
"""Bit-parallel gi_bfs_multi batch time vs the direction threshold m/div (config's own sources).

    python tools/bfs_div.py CONFIG DIV...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

ci = int(sys.argv[1])
divs = [int(x) for x in sys.argv[2:]] or [0]
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
keep = ts != td
elig = torch.zeros(cfg.n, dtype=torch.int32, device="cuda")
elig[ts[keep].long()] = 1
srcs = [int(x) for x in graphgen.pick_sources_from_mask(cfg.n, elig.cpu().numpy(), cfg.bfs_sources or 1,
                                                          cfg.source_seed or 1)]
del ts, td, keep, elig
torch.cuda.empty_cache()
out = torch.empty((len(srcs), cfg.n), dtype=torch.int32, device="cuda")
for dv in divs:
    g.bfs_multi(srcs, out=out, threshold_div=dv)
    best = 1e9
    for _ in range(3):
        _, st = g.bfs_multi(srcs, out=out, threshold_div=dv, profile=True)
        best = min(best, sum(x.total_ms for x in st))
    print(f"{cfg.name} div={dv or 'default'} batch ms {best:.3f} pull levels {max(x.pull_levels for x in st)}", flush=True)
