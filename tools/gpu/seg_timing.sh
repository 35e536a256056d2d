rm -f gpurun_out/seg_timing.csv
for m in 0 3; do GI_SEG_MODE=$m GI_DEBUG_SEG_TIMING=gpurun_out/seg_timing.csv timeout 300 python tools/prof.py --config 2 --pr-iters 3 --pr-reps 1 --bfs 0 2>&1 | tail -1; echo "mode $m"; python tools/seg_timing.py gpurun_out/seg_timing.csv; rm -f gpurun_out/seg_timing.csv; done
