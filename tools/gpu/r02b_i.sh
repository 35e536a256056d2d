python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_DEBUG_SLOW_MS=10 E2E_REPS=10 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -30
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_i_pytest.log
tail -n 3 gpurun_out/r02b_i_pytest.log
