python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented_or or or_pull_auto or bitparallel or bfs_multi" > gpurun_out/r02b_c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_c_pytest.log
tail -n 4 gpurun_out/r02b_c_pytest.log
GI_DEBUG_MSBFS=gpurun_out/r02b_c_levels2.txt timeout 300 python tools/msbfs_or_ab.py 2 16 2>&1 | tail -6
timeout 600 python tools/msbfs_or_ab.py 4 2>&1 | tail -6
