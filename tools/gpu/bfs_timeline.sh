rm -f gpurun_out/bfs_tl.txt
GI_DEBUG_BFS_FUSED=gpurun_out/bfs_tl.txt timeout 300 python tools/prof.py --config 2 --pr-iters 1 --bfs 4 2>&1 | tail -4
cat gpurun_out/bfs_tl.txt | tail -40
timeout 300 python tools/prof.py --config 2 --pr-iters 1 --bfs 6 2>&1 | tail -5
