# segmented OR pull for the bit-parallel BFS: parity tests, A/B on configs 2 and 4
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented_or or or_pull_auto or bitparallel or bfs_multi" > gpurun_out/r02b_b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_b_pytest.log
tail -n 15 gpurun_out/r02b_b_pytest.log
GI_DEBUG_MSBFS=gpurun_out/r02b_b_levels4.txt timeout 600 python tools/msbfs_or_ab.py 4 2>&1 | tail -8
timeout 300 python tools/msbfs_or_ab.py 2 16 2>&1 | tail -6
timeout 300 python tools/msbfs_or_ab.py 2 32 2>&1 | tail -6
