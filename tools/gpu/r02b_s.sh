python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_s_layout.txt E2E_REPS=1 timeout 900 python tools/e2e_split.py 4 > /dev/null 2>&1; grep -E "auto pull|P=" gpurun_out/r02b_s_layout.txt | cut -c1-200
GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_s_layout2.txt E2E_REPS=1 timeout 900 python tools/e2e_split.py 2 > /dev/null 2>&1; grep -E "auto pull|P=" gpurun_out/r02b_s_layout2.txt | cut -c1-200
E2E_REPS=5 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"k_ms_|OpOr" --csv --log-file gpurun_out/r02b_s_pass.csv python tools/msbfs_one_pass.py 4 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02b_s_pass.csv')) if len(r)>5]
h=next(r for r in rows if 'Kernel Name' in r); ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[rows.index(h)+1:]:
    v=float(r[vi].replace(',',''))/1e3
    if v > 40: print(f"{v:9.1f} us  {r[ki][:60]}")
PY
timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline_bfs']['pass_ms'], d['first_pr_ms'] if 'first_pr_ms' in d else d.get('pr_first_call_ms'))"
