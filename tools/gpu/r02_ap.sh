python -c "import __graft_entry__ as g; g.build()"
for v in base rp2 rp8 rm4 rm8 base; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  GI_LIBGI=$L timeout 600 python tools/pr_ab.py $v 3
done 2>&1 | grep variant
