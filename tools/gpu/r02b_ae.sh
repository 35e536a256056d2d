python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 5 4 2; do timeout 900 python tools/msbfs_one_pass.py $c 2>&1 | tail -1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "bitparallel or bfs_multi or listed_row or or_pull or full_config" 2>&1 | tail -2
timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline_bfs']['pass_ms'], d['secondary']['value'])"
