# e2e variance on config 4 with allocation / layout diagnostics; ncu of one OR level (config 4)
python -c "import __graft_entry__ as g; g.build()"
GI_DEBUG_BIGCACHE=1 GI_DEBUG_BUILD=gpurun_out/r02b_d_build.txt GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_d_layout.txt E2E_REPS=8 timeout 900 python tools/e2e_split.py 4 > gpurun_out/r02b_d_e2e.txt 2>&1
tail -12 gpurun_out/r02b_d_e2e.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpOr|k_ms_or_vertex|k_ms_resolve_heavy|k_ms_narrow_or" -c 4 -o gpurun_out/prof_r02b_or4 -f python tools/msbfs_or_ab.py 4 > gpurun_out/r02b_d_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02b_d_ncu.log
