# PR parity subset, per-CTA timing fit and config-2 PR timing
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -x -q -m gpu -k "pr or prdelta or dist" 2>&1 | tail -3
rm -f gpurun_out/seg_timing.csv gpurun_out/seg_layout.txt
GI_DEBUG_SEG_LAYOUT=gpurun_out/seg_layout.txt GI_DEBUG_SEG_TIMING=gpurun_out/seg_timing.csv timeout 300 python tools/prof.py --config 2 --pr-iters 5 --pr-reps 1 --bfs 0 > /dev/null 2>&1
cat gpurun_out/seg_layout.txt
python tools/seg_timing.py gpurun_out/seg_timing.csv
timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 3 --bfs 0 2>&1 | tail -2
