# PR parity subset + config-2 timing (no ncu)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -x -q -m gpu -k "pr or prdelta or dist" 2>&1 | tail -4
GI_DEBUG_SEG_LAYOUT=gpurun_out/seg_layout.txt timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 3 --bfs 0 2>&1 | tail -3
