python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "or_pull or segmented_or" > gpurun_out/r02b_q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_q_pytest.log
tail -n 2 gpurun_out/r02b_q_pytest.log
for h in 0 8192 16384 32768; do
GI_MS_HUB=$h timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"k_ms_resolve|k_ms_or_vertex" --csv --log-file gpurun_out/r02b_q_$h.csv python tools/msbfs_one_pass.py 4 > /dev/null 2>&1
python - $h <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f'gpurun_out/r02b_q_{sys.argv[1]}.csv')) if len(r)>5]
h=next(r for r in rows if 'Kernel Name' in r); ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print(sys.argv[1], [(r[ki][15:40], round(float(r[vi].replace(',',''))/1e3,1)) for r in rows[rows.index(h)+1:]])
PY
done
GI_MS_SPARSE_FRAC=0.3 timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sparse0.3', d['value'], d['roofline_bfs']['pass_ms'])"
timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['roofline_bfs']['pass_ms'])"
