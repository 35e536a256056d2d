# verification after the OR-vertex register cap: BFS GPU tests, smoke, bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -k "bfs or ms or multi or full_config or scale or bench" > gpurun_out/r02c_k_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02c_k_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02c_k_bench.json 2> gpurun_out/r02c_k_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02c_k_bench.json'));print(d['value'],d['bfs_gteps'],d['roofline_bfs']['pass_ms'],d['roofline']['frac'],d['roofline']['atomics']['frac'],d['e2e']['value'],d['clocks'])"
