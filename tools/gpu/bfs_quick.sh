timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "bfs or full_config or config4" 2>&1 | tail -2
rm -f gpurun_out/bfs_tl.txt
GI_DEBUG_BFS_FUSED=gpurun_out/bfs_tl.txt timeout 300 python tools/prof.py --config 2 --pr-iters 1 --bfs 2 > /dev/null 2>&1
cat gpurun_out/bfs_tl.txt
timeout 300 python tools/prof.py --config 2 --pr-iters 1 --bfs 8 2>&1 | tail -6
