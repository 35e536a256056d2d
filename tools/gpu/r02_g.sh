python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -x -q -k "pr_ or partitioned or hostcomm" > gpurun_out/r02g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02g_pytest.log
tail -2 gpurun_out/r02g_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02g_pytest.log | head -5
timeout 600 python tools/pr_ab.py fixedpoint 5 > gpurun_out/r02g_ab.jsonl 2> gpurun_out/r02g_ab.err
cat gpurun_out/r02g_ab.jsonl; tail -2 gpurun_out/r02g_ab.err
timeout 600 python tools/perf_configs.py 4 > gpurun_out/r02g_perf4_default.jsonl 2>&1
GI_POOL_KEEP_GB=120 GI_POOL_MAX_GB=64 timeout 600 python tools/perf_configs.py 4 > gpurun_out/r02g_perf4_bigpool.jsonl 2>&1
tail -1 gpurun_out/r02g_perf4_default.jsonl gpurun_out/r02g_perf4_bigpool.jsonl
