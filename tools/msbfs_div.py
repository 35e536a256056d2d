"""Bit-parallel BFS direction threshold A/B on config 2's 64 sources: python tools/msbfs_div.py DIV..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

cfg = graphgen.CONFIGS[2]
s, d = cfg.edges()
srcs = [int(x) for x in cfg.sources(s, d)]
ctx = gi.Context(0)
g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
out = torch.empty((len(srcs), cfg.n), dtype=torch.int32, device="cuda")
for div in [int(x) for x in sys.argv[1:]]:
    for _ in range(2):
        g.bfs_multi(srcs, out=out, batch=gi.GI_BFS_BATCH_BITPARALLEL, threshold_div=div)
    best = min(sum(x.total_ms for x in g.bfs_multi(srcs, out=out, batch=gi.GI_BFS_BATCH_BITPARALLEL,
                                                    threshold_div=div, profile=True)[1]) for _ in range(3))
    _, st = g.bfs_multi(srcs, out=out, batch=gi.GI_BFS_BATCH_BITPARALLEL, threshold_div=div, profile=True)
    print(f"div={div} batch ms {best:.3f} pulls={st[0].pull_levels}")
