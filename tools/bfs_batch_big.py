"""Per-source vs bit-parallel gi_bfs_multi on the device-generated configs 4/5.

usage: python tools/bfs_batch_big.py CONFIG [K]   (K sources with out-degree > 0, seeded)
"""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = graphgen.CONFIGS[ci]
k = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.bfs_sources
a, b, c, _ = cfg.abcd
ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
keep = ts != td
ts, td = ts[keep], td[keep]
if cfg.symmetrize:
    ts, td = torch.cat([ts, td]), torch.cat([td, ts])
ctx = gi.Context(0, torch.cuda.current_stream().cuda_stream)
g = gi.Graph(ctx, cfg.n, ts, td, gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
del ts, td
outdeg = g.out_degrees(torch.empty(cfg.n, dtype=torch.int32, device="cuda"))
cand = torch.nonzero(outdeg > 0).flatten()
gen = torch.Generator(device="cuda").manual_seed(1000 + ci)
srcs = cand[torch.randperm(cand.numel(), device="cuda", generator=gen)[:k]].tolist()
out = torch.empty((k, cfg.n), dtype=torch.int32, device="cuda")
print(f"config {ci}: n={cfg.n} m={g.m} k={k}")
for name, bm in [("per_source", gi.GI_BFS_BATCH_PER_SOURCE), ("bitparallel", gi.GI_BFS_BATCH_BITPARALLEL)]:
    g.bfs_multi(srcs, out=out, batch=bm)
    best = 1e9
    for _ in range(3):
        _, st = g.bfs_multi(srcs, out=out, batch=bm, profile=True)
        best = min(best, sum(x.total_ms for x in st))
    trav = sum(x.edges_traversed for x in st)
    print(f"{name:12s} batch ms {best:.3f}  per source {best / k:.4f}  GTEPS {trav / (best * 1e-3) / 1e9:.1f}  "
          f"levels {max(x.levels for x in st)}")
