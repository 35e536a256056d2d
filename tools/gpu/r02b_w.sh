python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented or seg or cc or or_pull or full_config" > gpurun_out/r02b_w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_w_pytest.log
tail -n 2 gpurun_out/r02b_w_pytest.log
GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_w_layout.txt E2E_REPS=3 timeout 900 python tools/e2e_split.py 4 > /dev/null 2>&1
grep -E "block rows|ranges" gpurun_out/r02b_w_layout.txt | tail -3 | cut -c1-250
E2E_REPS=5 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -4
