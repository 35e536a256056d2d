python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/msbfs_one_pass.py 4
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_ms_|OpOr" -o gpurun_out/prof_r02b_pass4 -f python tools/msbfs_one_pass.py 4 > gpurun_out/r02b_o_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r02b_o_ncu.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host_edges_pipelined" 2>&1 | tail -2
