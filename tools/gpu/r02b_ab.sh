python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_DEBUG_MSBFS=gpurun_out/r02b_ab_levels5.txt timeout 900 python tools/msbfs_one_pass.py 5 2>&1 | tail -2
cat gpurun_out/r02b_ab_levels5.txt
