import sys, torch
sys.path.insert(0, '.')
import graphgen
from paper_1805_00923_b200 import gi
cfg = graphgen.CONFIGS[3]
s, d = cfg.edges()
ctx = gi.Context(0)
for flags, name in [(gi.GI_DEFAULT_FLAGS, "auto-relabel"), (gi.GI_DEFAULT_FLAGS | gi.GI_NO_RELABEL, "norelabel")]:
    g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), flags | gi.GI_EDGES_ON_DEVICE)
    out = torch.empty(cfg.n, dtype=torch.float32, device='cuda')
    for dname, dr in [("direct", gi.GI_PR_PULL_DIRECT), ("segmented", gi.GI_PR_PULL_SEGMENTED)]:
        for _ in range(2): g.pagerank(20, 0.85, out=out, direction=dr)
        _, st = g.pagerank(20, 0.85, out=out, direction=dr, profile=True)
        print(name, dname, f"{st.edge_ms / st.edge_launches:.4f} ms/iter")
    g.close()
