python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bitparallel or bfs_multi or or_pull or segmented_or" > gpurun_out/r02b_m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_m_pytest.log
tail -n 3 gpurun_out/r02b_m_pytest.log
for f in 0 0.25; do
GI_MS_SPARSE_FRAC=$f GI_DEBUG_MSBFS=gpurun_out/r02b_m_levels_$f.txt timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r02b_m_bench_$f.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r02b_m_bench_$f.json'))
print('$f', d['value'], d['ms_per_step'], d['pr_gteps'], d['bfs_gteps'], d['roofline_bfs']['pass_ms'], d['secondary']['value'], d['secondary']['bfs_gteps'])"
tail -8 gpurun_out/r02b_m_levels_$f.txt
done
