python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bfs or pr_blocked" > gpurun_out/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
tail -n 2 gpurun_out/r02i_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02i_pytest.log | head -5
timeout 900 python tools/perf_configs.py 2 4 5 > gpurun_out/r02i_perf.jsonl 2> gpurun_out/r02i_perf.err
cat gpurun_out/r02i_perf.jsonl; tail -n 2 gpurun_out/r02i_perf.err
