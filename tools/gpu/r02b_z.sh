# A/B of parent-scan batch widths: per-kernel times of one config-4 pass
for v in base orb4 orb1 orb4m base; do
  if [ "$v" = base ]; then L=""; else L="GI_LIBGI=paper_1805_00923_b200/libgi_$v.so"; fi
  env $L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"k_ms_or_vertex|k_ms_resolve|k_ms_pull|k_ms_finish" --csv --log-file gpurun_out/r02b_z_$v.csv python tools/msbfs_one_pass.py 4 > /dev/null 2>&1
  python - $v <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f'gpurun_out/r02b_z_{sys.argv[1]}.csv')) if len(r)>5]
h=next(r for r in rows if 'Kernel Name' in r); ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print(sys.argv[1], [(r[ki][15:32], round(float(r[vi].replace(',',''))/1e3)) for r in rows[rows.index(h)+1:]])
PY
done
