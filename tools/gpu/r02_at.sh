python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q -k "build or pr_config1 or pr_random or bfs_config1 or cc_parity or full_config or billion_edge_config_parity and 4" > gpurun_out/r02at_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02at_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02at_pytest.log | head -3
rm -f gpurun_out/r02at_build.txt
GI_DEBUG_BUILD=gpurun_out/r02at_build.txt timeout 900 python bench.py --no-cpu-baseline --no-secondary --steps 3 > gpurun_out/r02at_bench.json 2> gpurun_out/r02at_bench.err; echo "bench rc=$?"
cat gpurun_out/r02at_build.txt
python -c "
import json; d=json.load(open('gpurun_out/r02at_bench.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['step_phases_ms']['steps'], d['build_ms'])"
