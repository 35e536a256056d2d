python -c "import __graft_entry__ as g; g.build()"
GI_SEG_STEAL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_segmented or pr_config1 or pr_random or cc_parity or full_config" > gpurun_out/r02o_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02o_pytest.log
for c in 2 4; do for v in 0 1; do GI_SEG_STEAL=$v timeout 600 python tools/pr_ab.py steal$v $c; done; done 2>&1 | grep variant
