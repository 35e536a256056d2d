"""PageRankDelta timings (10 rounds, d = 0.85, eps = 0.1 and 0.01) on configs 2 and 4.

usage: python tools/prdelta_perf.py [configs...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

ctx = gi.Context(0, torch.cuda.current_stream().cuda_stream)
for ci in [int(a) for a in sys.argv[1:]] or [2, 4]:
    cfg = graphgen.CONFIGS[ci]
    if ci in (4, 5):
        a, b, c, _ = cfg.abcd
        ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
    else:
        s, d = cfg.edges()
        ts, td = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
    g = gi.Graph(ctx, cfg.n, ts, td, gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
    del ts, td
    out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
    for eps in (0.1, 0.01):
        g.pagerank_delta(10, 0.85, eps, out=out)
        best = None
        for _ in range(3):
            _, st = g.pagerank_delta(10, 0.85, eps, out=out, profile=True)
            if best is None or st.total_ms < best.total_ms:
                best = st
        print(json.dumps({"config": cfg.name, "m": g.m, "eps": eps,
                          **{k: getattr(best, k) for k, _ in best._fields_}}), flush=True)
    g.close()
    torch.cuda.empty_cache()
