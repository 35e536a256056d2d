python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "or_pull or segmented_or or bitparallel or bfs_multi" > gpurun_out/r02b_r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_r_pytest.log
tail -n 2 gpurun_out/r02b_r_pytest.log
GI_DEBUG_MSBFS=gpurun_out/r02b_r_levels2.txt timeout 300 python tools/msbfs_or_ab.py 2 64 2>&1 | tail -6
grep pull-or gpurun_out/r02b_r_levels2.txt | head -3
timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline_bfs']['pass_ms'], d['secondary'])"
