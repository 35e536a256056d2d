python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pb_scatter|k_pb_gather" -s 2 -c 2 -o gpurun_out/prof_r02_c5b -f python tools/prof.py --config 5 --pr-iters 3 --bfs 0 > gpurun_out/ncu_c5b.log 2>&1; echo "ncu rc=$?"
