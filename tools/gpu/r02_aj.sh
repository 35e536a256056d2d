python -c "import __graft_entry__ as g; g.build()"
for c in 4; do for v in base ldcs base ldcs; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  GI_LIBGI=$L timeout 600 python tools/pr_ab.py $v $c
done; done 2>&1 | grep variant
