#!/bin/bash
# per-kernel durations of one bit-parallel multi-source BFS batch (config 2)
bash tools/gpu/bfs_batch_ab.sh bitparallel
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/msbfs_launches.csv \
  python tools/bfs_batch.py 2 bitparallel > /dev/null 2>&1
python - <<'PY'
import csv, collections
import io
rows = list(csv.DictReader(io.StringIO("".join(l for l in open("gpurun_out/msbfs_launches.csv") if not l.startswith("==")))))
# last batch only: kernels after the final k_ms_init
names = [(r['Kernel Name'], float(r['Metric Value'])) for r in rows if r['Metric Name'] == 'gpu__time_duration.sum']
last = max(i for i, (k, _) in enumerate(names) if 'k_ms_init' in k)
for k, v in names[last:]:
    print(f"{v/1e3:9.1f} us  {k[:90]}")
PY
