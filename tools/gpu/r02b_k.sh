python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/r02b_k_bench.json 2> gpurun_out/r02b_k_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02b_k_bench.json'))
print(d['value'], d['ms_per_step'], d['pr_gteps'], d['bfs_gteps'], d['roofline']['frac'], d['roofline_bfs']['frac'], d['e2e']['value'], d['clocks'])
print(d['e2e']['step_phases_ms']['steps']); print(d['secondary'])"
