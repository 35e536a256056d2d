# config 2/4 PR ms/iter for several calibration pass counts
for c in 2 4; do
  for k in 3 5 8; do echo -n "cfg$c calib=$k  "; GI_SEG_CALIB=$k timeout 600 python tools/prof.py --config $c --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1; done
done
