# A/B of BFS variants on one box: per-source batch time (16 sources x 3 reps)
cat > /tmp/bm.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import graphgen
from paper_1805_00923_b200 import gi
cfg = graphgen.CONFIGS[2]
s, d = cfg.edges(); srcs = [int(x) for x in cfg.sources(s, d)][:16]
ctx = gi.Context(0)
g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
out = torch.empty((len(srcs), cfg.n), dtype=torch.int32, device='cuda')
for _ in range(3): g.bfs_multi(srcs, out=out)
best = 1e9
for _ in range(3):
    _, st = g.bfs_multi(srcs, out=out, profile=True)
    best = min(best, sum(x.total_ms for x in st) / len(st))
print(f"{sys.argv[1]:10s} per-source ms {best:.4f}")
PY
for v in "$@"; do
  if [ "$v" = base ]; then python /tmp/bm.py base; else GI_LIBGI=paper_1805_00923_b200/libgi_$v.so python /tmp/bm.py $v; fi
done
