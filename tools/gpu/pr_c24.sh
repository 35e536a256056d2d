# configs 2 and 4 PageRank ms/iter (2 fresh processes each) + config 4 per-CTA timing
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pr or prdelta" 2>&1 | tail -1
for c in 2 4; do for r in 1 2; do echo -n "cfg$c  "; timeout 600 python tools/prof.py --config $c --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1; done; done
bash tools/gpu/pr_cfg4.sh | grep -A9 "kernel span\|slowest"
