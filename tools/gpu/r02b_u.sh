python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_BENCH_DEVICE=0 GI_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config 2 --steps 2 --warmup 3 --no-secondary > gpurun_out/r02b_u_part2.json 2> gpurun_out/r02b_u_part2.err; echo "part rc=$?"; tail -n 3 gpurun_out/r02b_u_part2.err; cat gpurun_out/r02b_u_part2.json | head -c 1500
