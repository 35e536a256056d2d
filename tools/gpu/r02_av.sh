python -c "import __graft_entry__ as g; g.build()"
rm -f gpurun_out/r02av_msbfs.txt
GI_DEBUG_MSBFS=gpurun_out/r02av_msbfs.txt timeout 600 python tools/bfs_div.py 4 0 2>&1 | grep div
tail -n 9 gpurun_out/r02av_msbfs.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ms_" -s 40 -c 14 -o gpurun_out/prof_r02av_msbfs4 -f python tools/bfs_div.py 4 0 > gpurun_out/r02av_ncu.log 2>&1; echo "ncu rc=$?"
