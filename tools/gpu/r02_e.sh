python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -x -q -k "pr_ or partitioned or hostcomm or bfs" > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
tail -3 gpurun_out/r02e_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02e_pytest.log | head -5
rm -f gpurun_out/r02e_layout.txt
for c in 5; do GI_DEBUG_SEG_LAYOUT=gpurun_out/r02e_layout.txt timeout 600 python tools/pr_ab.py auto $c; done > gpurun_out/r02e_ab.jsonl 2> gpurun_out/r02e_ab.err
GI_PB_EPP=100 timeout 300 python tools/pr_ab.py blocked4 4 >> gpurun_out/r02e_ab.jsonl 2>> gpurun_out/r02e_ab.err
cat gpurun_out/r02e_ab.jsonl; grep -v "^  short\|^block rows" gpurun_out/r02e_layout.txt; tail -3 gpurun_out/r02e_ab.err
