python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_ or full_config" > gpurun_out/r02aq_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02aq_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02aq_pytest.log | head -3
for i in 1 2; do timeout 600 python tools/pr_ab.py rows 3; done 2>&1 | grep variant
