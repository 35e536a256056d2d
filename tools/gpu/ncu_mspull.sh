#!/bin/bash
# full ncu capture of one bit-parallel pull kernel launch (config 2):
#   tools/gpu/ncu_mspull.sh KERNEL_REGEX SKIP   e.g. '^k_ms_pull$' 1 = the light pull of level 3
bash tools/gpu/bfs_batch_ab.sh bitparallel
ncu --set full --clock-control none --import-source on -k "regex:${1:-k_ms_pull}" --launch-skip ${2:-0} -c 1 \
  -o gpurun_out/ms_pull -f python tools/bfs_batch.py 2 bitparallel > gpurun_out/ncu_pull.log 2>&1
tail -2 gpurun_out/ncu_pull.log
