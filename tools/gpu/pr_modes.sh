timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -x -q -m gpu -k "pr or prdelta or dist" 2>&1 | tail -3
GI_DEBUG_SEG_LAYOUT=gpurun_out/seg_layout.txt timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1
cat gpurun_out/seg_layout.txt
for m in 1 2 3; do echo "mode $m"; GI_SEG_MODE=$m timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1; done
