python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -x -q -k "pr_ or cc_ or prdelta or full_config or partitioned" > gpurun_out/r02ac_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02ac_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02ac_pytest.log | head -3
timeout 900 python tools/perf_configs.py 2 4 5 2>&1 | grep config
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02ac_bench.json 2> gpurun_out/r02ac_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02ac_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['step_phases_ms']['steps'], d['pr_first_call_ms'], d['roofline_bfs']['pass_ms'], d['secondary'])"
