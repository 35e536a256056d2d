# small-grid BFS as one 16-CTA cluster vs cooperative grid: BFS parity, then the grid graph (config 3)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bfs" 2>&1 | tail -1
for c in 1 0; do echo -n "GI_BFS_CLUSTER=$c  "; GI_BFS_CLUSTER=$c timeout 300 python tools/prof.py --config 3 --pr-iters 1 --bfs 1 2>&1 | tail -1; done
