# config-2 PR ms/iter under different calibration settings (3 fresh processes each)
for cfg in "3 1.0" "6 1.0" "10 0.7" "16 0.5"; do
  set -- $cfg
  for r in 1 2 3; do echo -n "calib=$1 damp=$2  "; GI_SEG_CALIB=$1 GI_SEG_DAMP=$2 timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 3 --bfs 0 2>&1 | tail -1; done
done
