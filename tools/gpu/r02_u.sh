python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/u_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u_pytest_gpu.log
tail -n 3 gpurun_out/u_pytest_gpu.log; grep -E "^FAILED|Error:" gpurun_out/u_pytest_gpu.log | head -5
timeout 900 python bench.py > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/u_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['step_phases_ms']['steps'], d['pr_first_call_ms'], d['roofline_bfs']['pass_ms'], d['secondary']['value'] if d['secondary'] else None)"
