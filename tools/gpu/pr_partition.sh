#!/bin/bash
# parity of the source-partitioned pull + its timing on configs 2, 4, 5
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q -k "partitioned or small_families or exhaustive_tiny" > gpurun_out/sp_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/sp_tests.log
timeout 300 python tools/pr_partition_perf.py 2 0 65536 1048576 > gpurun_out/sp_c2.jsonl 2> gpurun_out/sp_c2.err
timeout 600 python tools/pr_partition_perf.py 4 0 4194304 16777216 > gpurun_out/sp_c4.jsonl 2> gpurun_out/sp_c4.err
timeout 900 python tools/pr_partition_perf.py 5 0 4194304 16777216 > gpurun_out/sp_c5.jsonl 2> gpurun_out/sp_c5.err
tail -3 gpurun_out/sp_tests.log; cat gpurun_out/sp_c2.jsonl gpurun_out/sp_c4.jsonl gpurun_out/sp_c5.jsonl; tail -3 gpurun_out/sp_c5.err
