"""Bit-parallel BFS pass with the row pull vs the segmented OR pull (gi_bfs_opts.pull_kernel),
on a config whose graph has the segmented layout (a PageRank call builds it first, as in the bench).

usage: python tools/msbfs_or_ab.py CONFIG [K]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = graphgen.CONFIGS[ci]
k = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.bfs_sources
if ci >= 4:
    a, b, c, _ = cfg.abcd
    ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
    keep = ts != td
    ts, td = ts[keep], td[keep]
    if cfg.symmetrize:
        ts, td = torch.cat([ts, td]), torch.cat([td, ts])
else:
    s, d = cfg.edges()
    ts, td = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
ctx = gi.Context(0, torch.cuda.current_stream().cuda_stream)
g = gi.Graph(ctx, cfg.n, ts, td, gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
del ts, td
outdeg = g.out_degrees(torch.empty(cfg.n, dtype=torch.int32, device="cuda"))
cand = torch.nonzero(outdeg > 0).flatten()
gen = torch.Generator(device="cuda").manual_seed(1000 + ci)
srcs = cand[torch.randperm(cand.numel(), device="cuda", generator=gen)[:k]].tolist()
pr = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
_, pst = g.pagerank(20, 0.85, out=pr)
print(f"config {ci}: n={cfg.n} m={g.m} k={k} pr kernel {pst.kernel}")
out = torch.empty((k, cfg.n), dtype=torch.int32, device="cuda")
for name, pk in [("rows", gi.GI_MS_PULL_ROWS), ("auto", gi.GI_MS_PULL_AUTO), ("segmented", gi.GI_MS_PULL_SEGMENTED),
                 ("rows", gi.GI_MS_PULL_ROWS), ("auto", gi.GI_MS_PULL_AUTO)]:
    g.bfs_multi(srcs, out=out, batch=gi.GI_BFS_BATCH_BITPARALLEL, pull_kernel=pk)
    best, bp = 1e9, 0
    for _ in range(3):
        _, st = g.bfs_multi(srcs, out=out, batch=gi.GI_BFS_BATCH_BITPARALLEL, pull_kernel=pk, profile=True)
        t = sum(x.total_ms for x in st)
        if t < best:
            best, bp = t, sum(x.pull_ms for x in st)
    trav = sum(x.edges_traversed for x in st)
    print(f"{name:10s} pass ms {best:.3f} (pull levels {bp:.3f} ms, {st[0].pull_levels} pull / "
          f"{st[0].pull_or_levels} OR)  GTEPS {trav / (best * 1e-3) / 1e9:.1f}  levels {max(x.levels for x in st)}")
