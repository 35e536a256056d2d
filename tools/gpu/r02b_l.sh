python -c "import __graft_entry__ as g; g.build()" || exit 1
for f in 2 0.7; do
GI_MS_SEGOR_FRAC=$f GI_DEBUG_MSBFS=gpurun_out/r02b_l_levels_$f.txt timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 3 --warmup 3 > gpurun_out/r02b_l_bench_$f.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r02b_l_bench_$f.json'))
print('$f', d['value'], d['ms_per_step'], d['pr_gteps'], d['bfs_gteps'], d['roofline_bfs']['pass_ms'])"
tail -9 gpurun_out/r02b_l_levels_$f.txt
done
