# quick PR iteration loop: parity tests for PR paths, timing on config 2, ncu of the segmented kernel
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -x -q -m gpu -k "pr or prdelta or dist" 2>&1 | tail -15 > gpurun_out/pytest_pr.log
cat gpurun_out/pytest_pr.log
GI_DEBUG_SEG_LAYOUT=gpurun_out/seg_layout.txt timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 3 --bfs 0 > gpurun_out/prof_pr.log 2>&1
cat gpurun_out/prof_pr.log gpurun_out/seg_layout.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seg|k_pr_acc" -s 2 -c 2 -o gpurun_out/prof_seg python tools/prof.py --config 2 --pr-iters 3 --bfs 0 > gpurun_out/ncu_seg.log 2>&1
tail -2 gpurun_out/ncu_seg.log
