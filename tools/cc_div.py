"""CC direction threshold A/B on one config: python tools/cc_div.py CONFIG DIV..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

cfg = graphgen.CONFIGS[int(sys.argv[1])]
s, d = cfg.edges()
ctx = gi.Context(0)
g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
out = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
for div in [int(x) for x in sys.argv[2:]]:
    g.cc(out=out, threshold_div=div)
    _, st = g.cc(out=out, threshold_div=div, profile=True)
    print(f"div={div} ms={st.total_ms:.2f} rounds={st.rounds} pulls={st.pull_rounds} examined={st.edges_examined}")
