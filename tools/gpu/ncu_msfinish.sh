#!/bin/bash
# full ncu capture of the bit-parallel BFS epilogue kernel (config 2)
bash tools/gpu/bfs_batch_ab.sh bitparallel
ncu --set full --clock-control none --import-source on -k regex:k_ms_finish -c 1 -o gpurun_out/ms_finish -f \
  python tools/bfs_batch.py 2 bitparallel > gpurun_out/ncu_finish.log 2>&1
tail -3 gpurun_out/ncu_finish.log
