cat > /tmp/g3.py <<'PY'
import sys, os
root = sys.argv[1]
sys.path.insert(0, os.path.abspath(root))
import torch, graphgen
from paper_1805_00923_b200 import gi
cfg = graphgen.CONFIGS[3]
s, d = cfg.edges()
ctx = gi.Context(0)
g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
for _ in range(3): g.pagerank(20, 0.85, out=out)
best = 1e9
for _ in range(5):
    _, st = g.pagerank(20, 0.85, out=out, profile=True)
    best = min(best, st.edge_ms / st.edge_launches)
print(root, "grid ms/iter", round(best, 4), "kernel", st.kernel)
PY
for c in _bisect/661019c _bisect/584cacd _bisect/ee687e6 _bisect/37da723 _bisect/ad69c71 .; do timeout 300 python /tmp/g3.py $c 2>&1 | tail -1; done
