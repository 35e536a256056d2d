python -c "import __graft_entry__ as g; g.build()"
for i in 1 2; do for v in base r1; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  GI_LIBGI=$L timeout 600 python tools/pr_ab.py $v 3
done; done 2>&1 | grep variant
