python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bfs_multi or full_config" > gpurun_out/r02am_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02am_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02am_pytest.log | head -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02am_bench.json 2> gpurun_out/r02am_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02am_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['pr_ms'], d['roofline_bfs']['pass_ms'], d['secondary']['value'])"
