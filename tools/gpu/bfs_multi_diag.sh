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
import os; os.environ['X']='1'
_, st = g.bfs_multi(srcs, out=out, profile=True)
print('per source ms', sum(x.total_ms for x in st)/len(st))
PY
GI_DEBUG_BFS_MULTI=gpurun_out/bfs_multi.txt python /tmp/bm.py; tail -16 gpurun_out/bfs_multi.txt
