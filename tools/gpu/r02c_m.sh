# A/B: register cap of the light-row bit-parallel pull (k_ms_pull, GI_MS_LMINB 4 -> 5, 6)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for rep in 1 2; do
for v in base lm5 lm6; do
  if [ "$v" = base ]; then L=""; else L="GI_LIBGI=paper_1805_00923_b200/libgi_$v.so"; fi
  env $L timeout 300 python tools/msbfs_one_pass.py 4 2>&1 | tail -1 | sed "s/^/$v: /"
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"k_ms_pull[^_]" --csv --log-file gpurun_out/r02c_m_$v.csv python tools/msbfs_one_pass.py 4 > /dev/null 2>&1
  python - $v <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f'gpurun_out/r02c_m_{sys.argv[1]}.csv')) if len(r)>5]
h=next(r for r in rows if 'Kernel Name' in r); vi=h.index('Metric Value')
print(sys.argv[1], 'k_ms_pull us', [round(float(r[vi].replace(',',''))/1e3) for r in rows[rows.index(h)+1:]])
PY
done; done
