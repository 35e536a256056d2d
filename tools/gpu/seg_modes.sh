# segmented-pull cost breakdown on config 2 (GI_SEG_MODE diagnostics; results are wrong by design for modes 1-2)
for m in 0 1 2; do
  rm -f gpurun_out/seg_timing.csv
  GI_SEG_MODE=$m GI_DEBUG_SEG_TIMING=gpurun_out/seg_timing.csv timeout 300 python tools/prof.py --config 2 --pr-iters 3 --pr-reps 1 --bfs 0 > /dev/null 2>&1
  echo "mode $m"; python tools/seg_timing.py gpurun_out/seg_timing.csv | grep -v "cta "
  GI_SEG_MODE=$m timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 1 --bfs 0 2>&1 | tail -1
done
