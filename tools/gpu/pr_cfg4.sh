# config-4 PageRank: per-iteration split, segmented layout stats, per-CTA timing of the edge pass
rm -f gpurun_out/seg4_timing.csv gpurun_out/seg4_layout.txt
GI_DEBUG_SEG_LAYOUT=gpurun_out/seg4_layout.txt timeout 600 python tools/prof.py --config 4 --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -2
GI_DEBUG_SEG_TIMING=gpurun_out/seg4_timing.csv timeout 600 python tools/prof.py --config 4 --pr-iters 5 --pr-reps 1 --bfs 0 2>&1 | tail -1
python tools/seg_timing.py gpurun_out/seg4_timing.csv
cat gpurun_out/seg4_layout.txt | head -20
