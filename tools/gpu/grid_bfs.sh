rm -f gpurun_out/bfs_tl.txt
GI_DEBUG_BFS_FUSED=gpurun_out/bfs_tl.txt timeout 300 python tools/prof.py --config 3 --pr-iters 1 --bfs 1 2>&1 | tail -1
sed -n '1,5p;100,106p;4000,4004p' gpurun_out/bfs_tl.txt
python - <<'PY'
import re
w=[];b=[]
for l in open('gpurun_out/bfs_tl.txt'):
    m=re.search(r'work_us=([\d.]+) barrier_us=([\d.]+)',l)
    if m: w.append(float(m.group(1))); b.append(float(m.group(2)))
print("levels",len(w),"sum work ms",sum(w)/1e3,"sum barrier ms",sum(b)/1e3)
PY
timeout 300 python tools/prof.py --config 3 --pr-iters 1 --bfs 1 2>&1 | tail -1
