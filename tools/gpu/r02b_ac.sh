python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_DEBUG_MSBFS=gpurun_out/r02b_ac_levels5.txt timeout 900 python tools/msbfs_one_pass.py 5 2>&1 | tail -1
tail -9 gpurun_out/r02b_ac_levels5.txt
GI_DEBUG_MSBFS=gpurun_out/r02b_ac_levels4.txt timeout 900 python tools/msbfs_one_pass.py 4 2>&1 | tail -1
tail -8 gpurun_out/r02b_ac_levels4.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "bitparallel or bfs_multi or listed_row or or_pull" 2>&1 | tail -2
