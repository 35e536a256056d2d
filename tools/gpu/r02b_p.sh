python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "bitparallel or bfs_multi or or_pull or segmented_or or full_config" > gpurun_out/r02b_p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_p_pytest.log
tail -n 2 gpurun_out/r02b_p_pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"k_ms_|OpOr" --csv --log-file gpurun_out/r02b_p_pass.csv python tools/msbfs_one_pass.py 4 > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02b_p_pass.csv')))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    if len(r)>vi: print(f"{float(r[vi].replace(',',''))/1e3:9.1f} us  {r[ki][:70]}")
PY
timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r02b_p_bench.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r02b_p_bench.json'))
print(d['value'], d['ms_per_step'], d['pr_gteps'], d['bfs_gteps'], d['roofline']['frac'], d['roofline_bfs']['pass_ms'], d['secondary']['value'])"
