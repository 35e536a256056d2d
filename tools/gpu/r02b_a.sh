# re-entry sanity: build, full GPU suite, bench line
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02b_a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_a_pytest_gpu.log
tail -n 3 gpurun_out/r02b_a_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02b_a_bench.json 2> gpurun_out/r02b_a_bench.err; echo "bench rc=$?"; cat gpurun_out/r02b_a_bench.json
GI_DEBUG_BFS_MULTI=gpurun_out/r02b_a_levels4.txt timeout 600 python tools/bfs_batch_big.py 4 > gpurun_out/r02b_a_bfs4.log 2>&1; tail -5 gpurun_out/r02b_a_bfs4.log
