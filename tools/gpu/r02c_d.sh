# config 2 (RMAT s22): CTA balance of the segmented pass — calibration passes, forced work stealing,
# and the per-CTA busy times after calibration
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for rep in 1 2; do
for v in base calib16 calib32 steal steal_calib16 damp05; do
  case $v in
    base) E="";; calib16) E="GI_SEG_CALIB=16";; calib32) E="GI_SEG_CALIB=32";; steal) E="GI_SEG_STEAL=2";;
    steal_calib16) E="GI_SEG_STEAL=2 GI_SEG_CALIB=16";; damp05) E="GI_SEG_CALIB=16 GI_SEG_DAMP=0.5";;
  esac
  env $E timeout 300 python tools/pr_ab.py $v 2 2>&1 | tail -1
done; done
GI_DEBUG_SEG_TIMING=gpurun_out/r02c_d_cta_c2.csv timeout 300 python tools/pr_ab.py timing 2 2>&1 | tail -1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02c_d_cta_c2.csv'))]
ctas=148
last=rows[-ctas:]
st=[int(r[3]) for r in last]; en=[int(r[4]) for r in last]
t0=min(st)
busy=sorted((e-s)/1e3 for s,e in zip(st,en)); ends=sorted((e-t0)/1e3 for e in en); starts=sorted((s-t0)/1e3 for s in st)
print("last pass: busy us min/med/max", busy[0], busy[len(busy)//2], busy[-1], "| start spread", starts[-1], "| end min/med/max", ends[0], ends[len(ends)//2], ends[-1])
PY
