# A/B of PR variants on one box: best per-iteration time of 20-iteration runs
cat > /tmp/pa.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import graphgen
from paper_1805_00923_b200 import gi
cfg = graphgen.CONFIGS[2]
s, d = cfg.edges()
ctx = gi.Context(0)
g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
out = torch.empty(cfg.n, dtype=torch.float32, device='cuda')
for _ in range(3): g.pagerank(20, 0.85, out=out)
best = 1e9
for _ in range(5):
    _, st = g.pagerank(20, 0.85, out=out, profile=True)
    best = min(best, st.edge_ms / st.edge_launches)
print(f"{sys.argv[1]:10s} ms/iter {best:.4f}")
PY
for v in "$@"; do
  if [ "$v" = base ]; then python /tmp/pa.py base; else GI_LIBGI=paper_1805_00923_b200/libgi_$v.so python /tmp/pa.py $v; fi
done
