python -c "import __graft_entry__ as g; g.build()"
rm -f gpurun_out/r02ak_msbfs.txt
GI_DEBUG_MSBFS=gpurun_out/r02ak_msbfs.txt timeout 600 python tools/bfs_batch_big.py 4 > /dev/null 2>&1
tail -n 8 gpurun_out/r02ak_msbfs.txt
rm -f gpurun_out/r02ak_msbfs5.txt
GI_DEBUG_MSBFS=gpurun_out/r02ak_msbfs5.txt timeout 900 python tools/bfs_batch_big.py 5 > gpurun_out/r02ak_bfs5.txt 2>&1
cat gpurun_out/r02ak_bfs5.txt; tail -n 10 gpurun_out/r02ak_msbfs5.txt
