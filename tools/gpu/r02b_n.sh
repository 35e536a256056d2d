python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "build or bitparallel or bfs_multi or or_pull or segmented_or" > gpurun_out/r02b_n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_n_pytest.log
tail -n 3 gpurun_out/r02b_n_pytest.log
for v in 0 1; do echo "== GI_BUILD_PIPELINE=$v"; GI_BUILD_PIPELINE=$v GI_DEBUG_BUILD=gpurun_out/r02b_n_build_$v.txt E2E_REPS=6 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -5; tail -2 gpurun_out/r02b_n_build_$v.txt; done
GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_n_layout.txt E2E_REPS=2 timeout 900 python tools/e2e_split.py 4 > /dev/null 2>&1; grep -v "short" gpurun_out/r02b_n_layout.txt | tail -4
GI_DEBUG_MSBFS=gpurun_out/r02b_n_levels.txt timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 3 --warmup 3 > gpurun_out/r02b_n_bench.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r02b_n_bench.json'))
print(d['value'], d['ms_per_step'], d['pr_gteps'], d['bfs_gteps'], d['roofline_bfs']['pass_ms'])"
tail -8 gpurun_out/r02b_n_levels.txt
