# verification of the final code (calibration reverted): PageRank/segmented GPU tests, smoke, bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "pr or pagerank or seg or prdelta or reductions" > gpurun_out/r02c_h_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02c_h_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02c_h_bench.json 2> gpurun_out/r02c_h_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02c_h_bench.json'));print(d['value'],d['roofline']['frac'],d['roofline']['launch_ms'],d['roofline']['atomics']['frac'],d['secondary']['roofline_pr_frac'],d['secondary']['roofline_pr_launch_ms'],d['e2e']['value'])"
