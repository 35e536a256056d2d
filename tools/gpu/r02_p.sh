python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stealing or pr_segmented or cc_parity" > gpurun_out/r02p_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02p_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02p_pytest.log | head -3
for c in 2 4; do timeout 600 python tools/pr_ab.py default $c; done 2>&1 | grep variant
timeout 600 python tools/perf_configs.py 4 2>&1 | tail -1
