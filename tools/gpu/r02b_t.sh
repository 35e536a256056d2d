python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in "X=1" "GI_MS_SPARSE_FRAC=0.3" "GI_MS_SEGOR_FRAC=0.2" "X=1" "GI_MS_SPARSE_FRAC=0.3"; do
env $v timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline_bfs']['pass_ms'],3))"
done
