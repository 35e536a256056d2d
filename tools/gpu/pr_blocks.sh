# per-block segmented build: parity subset, configs 2/4 timing, config 5 (m > 2^31) segmented
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pr or prdelta" 2>&1 | tail -1
for c in 2 4; do echo -n "cfg$c  "; timeout 600 python tools/prof.py --config $c --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1; done
GI_DEBUG_SEG_LAYOUT=gpurun_out/seg5_layout.txt timeout 1200 python tools/prof.py --config 5 --pr-iters 20 --pr-reps 2 --bfs 0 --direction segmented 2>&1 | tail -2
cat gpurun_out/seg5_layout.txt
