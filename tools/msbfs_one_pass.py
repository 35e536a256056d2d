"""One bench-like bit-parallel BFS pass on a config (after one PageRank call builds the segmented
layout, as in the bench step): the target of an ncu capture of every kernel of a pass.

usage: [MS_DIV=d] python tools/msbfs_one_pass.py CONFIG
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = graphgen.CONFIGS[ci]
a, b, c, _ = cfg.abcd
ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
s_np, d_np = ts.cpu().numpy(), td.cpu().numpy()
srcs = [int(x) for x in cfg.sources(s_np, d_np)]  # the bench's sources
del s_np, d_np
ctx = gi.Context(0, torch.cuda.current_stream().cuda_stream)
flags = gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE | (gi.GI_SYMMETRIZE if cfg.symmetrize else 0)
g = gi.Graph(ctx, cfg.n, ts, td, flags)
del ts, td
pr = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
g.pagerank(2, 0.85, out=pr)
out = torch.empty((len(srcs), cfg.n), dtype=torch.int32, device="cuda")
div = int(os.environ.get("MS_DIV", "0"))  # direction threshold m / div (0: the library default)
g.bfs_multi(srcs, out=out, threshold_div=div)
_, st = g.bfs_multi(srcs, out=out, profile=True, threshold_div=div)
print(f"config {ci}: k={len(srcs)} pass {sum(x.total_ms for x in st):.3f} ms, pull levels {st[0].pull_levels} "
      f"(OR {st[0].pull_or_levels}, sparse {st[0].pull_sparse_levels})")
