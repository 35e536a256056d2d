"""Per-source vs bit-parallel gi_bfs_multi on a host-generated config (default 2, its 64 sources).

usage: python tools/bfs_batch.py [CONFIG] [per_source|bitparallel]
"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen
from paper_1805_00923_b200 import gi
cfg = graphgen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
s, d = cfg.edges(); srcs = [int(x) for x in cfg.sources(s, d)]
ctx = gi.Context(0)
g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
out = torch.empty((len(srcs), cfg.n), dtype=torch.int32, device='cuda')
modes = [("per_source", gi.GI_BFS_BATCH_PER_SOURCE), ("bitparallel", gi.GI_BFS_BATCH_BITPARALLEL)]
if len(sys.argv) > 2: modes = [m for m in modes if m[0] == sys.argv[2]]
for name, b in modes:
    for _ in range(2): g.bfs_multi(srcs, out=out, batch=b)
    best = 1e9
    for _ in range(3):
        _, st = g.bfs_multi(srcs, out=out, batch=b, profile=True)
        best = min(best, sum(x.total_ms for x in st))
    trav = sum(x.edges_traversed for x in st)
    print(f"{name:12s} batch ms {best:.3f}  per source {best/len(srcs):.4f}  GTEPS {trav/(best*1e-3)/1e9:.1f}  levels {st[0].levels} pulls {st[0].pull_levels} examined/src {st[0].edges_examined}")
