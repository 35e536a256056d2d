python -c "import __graft_entry__ as g; g.build()"
GI_DEBUG_BIGCACHE=1 GI_DEBUG_SEG_LAYOUT=gpurun_out/r02an_layout.txt GI_BENCH_E2E_DEBUG=1 timeout 900 python bench.py --no-cpu-baseline --no-secondary > gpurun_out/r02an_bench.json 2> gpurun_out/r02an_bench.err; echo "bench rc=$?"
grep -c "bigcache" gpurun_out/r02an_bench.err; grep "bigcache" gpurun_out/r02an_bench.err | tail -30
grep "^n=\|^  hoff" gpurun_out/r02an_layout.txt | sed 's/.*build/build/'
python -c "
import json; d=json.load(open('gpurun_out/r02an_bench.json')); print(d['e2e']['step_phases_ms']['steps'], d['pr_first_call_ms'], d['build_ms'])"
