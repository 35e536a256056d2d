python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -x -q -k "pr_ or cc_ or full_config or partitioned" > gpurun_out/r02l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02l_pytest.log
tail -n 2 gpurun_out/r02l_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02l_pytest.log | head -5
for c in 2 4; do for v in 0 1; do GI_SEG_STEAL=$v timeout 600 python tools/pr_ab.py steal$v $c; done; done 2>&1 | grep variant
rm -f gpurun_out/r02l_segtiming.csv
GI_DEBUG_SEG_TIMING=gpurun_out/r02l_segtiming.csv timeout 600 python tools/prof.py --config 4 --pr-iters 20 --bfs 0 > /dev/null 2>&1
