# per-config PageRank / BFS numbers of the final code
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python tools/perf_configs.py 1 2 3 4 5 > gpurun_out/r02c_perf_configs.jsonl 2>&1; echo "perf rc=$?"; cat gpurun_out/r02c_perf_configs.jsonl | cut -c1-400
