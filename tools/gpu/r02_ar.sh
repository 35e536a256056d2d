python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_ or cc_ or prdelta or full_config" > gpurun_out/r02ar_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02ar_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02ar_pytest.log | head -3
rm -f gpurun_out/r02ar_layout.txt
for c in 4 2; do for v in 0 1 0 1; do GI_SEG_COMPACT=$v GI_DEBUG_SEG_LAYOUT=gpurun_out/r02ar_layout.txt timeout 600 python tools/pr_ab.py compact$v $c; done; done 2>&1 | grep variant
grep "short records\|^n=" gpurun_out/r02ar_layout.txt | head -8
