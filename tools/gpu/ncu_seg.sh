# full ncu capture of one steady-state segmented edge pass + vertex pass on config 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seg|k_pr_acc" -s 2 -c 2 -o gpurun_out/${1:-prof_seg} python tools/prof.py --config 2 --pr-iters 3 --bfs 0 > gpurun_out/ncu_seg.log 2>&1
tail -2 gpurun_out/ncu_seg.log
