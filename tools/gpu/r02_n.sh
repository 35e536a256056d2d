python -c "import __graft_entry__ as g; g.build()"
for v in 0 1; do
rm -f gpurun_out/r02n_segtiming$v.csv
GI_SEG_STEAL=$v GI_DEBUG_SEG_TIMING=gpurun_out/r02n_segtiming$v.csv timeout 600 python tools/prof.py --config 4 --pr-iters 20 --bfs 0 > /dev/null 2>&1
done
ls -la gpurun_out/r02n_segtiming*
