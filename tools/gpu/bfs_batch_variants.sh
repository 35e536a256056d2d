#!/bin/bash
# bit-parallel multi-source BFS A/B: default libgi vs the variants named as arguments (libgi_NAME.so)
bash tools/gpu/bfs_batch_ab.sh
for v in "$@"; do echo "== $v"; GI_LIBGI=paper_1805_00923_b200/libgi_$v.so python tools/bfs_batch.py 2 | grep bitpar; done
