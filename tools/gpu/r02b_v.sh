python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_v_layout.txt E2E_REPS=3 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -3
grep -E "block rows|ranges" gpurun_out/r02b_v_layout.txt | tail -3 | cut -c1-250
