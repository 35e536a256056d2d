# config-2 PR timing with and without programmatic dependent launch (fresh process = fresh calibration)
for r in 1 2 3; do
  for p in 1 0; do echo -n "GI_PDL=$p  "; GI_PDL=$p timeout 300 python tools/prof.py --config 2 --pr-iters 20 --pr-reps 3 --bfs 0 2>&1 | tail -1; done
done
