# segmented-pull cost breakdown on config 2 (GI_SEG_MODE diagnostics; results are wrong by design for modes 1-3)
for m in 0 1 2 3; do echo "mode $m"; GI_SEG_MODE=$m timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1; done
