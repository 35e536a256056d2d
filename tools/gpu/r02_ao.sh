python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -x -q -k "pr_ or cc_ or prdelta or full_config or partitioned" > gpurun_out/r02ao_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02ao_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02ao_pytest.log | head -3
