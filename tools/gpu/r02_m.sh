python -c "import __graft_entry__ as g; g.build()"
for v in 0 1; do
GI_SEG_STEAL=$v timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_segmented or pr_config1 or pr_random or cc_parity or full_config" > gpurun_out/r02m_pytest$v.log 2>&1; echo "steal=$v pytest rc=$?"; tail -n 1 gpurun_out/r02m_pytest$v.log; grep -E "^FAILED|Error:" gpurun_out/r02m_pytest$v.log | head -3
done
for c in 2 4; do for v in 0 1; do GI_SEG_STEAL=$v timeout 600 python tools/pr_ab.py steal$v $c; done; done 2>&1 | grep variant
