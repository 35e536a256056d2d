python -c "import __graft_entry__ as g; g.build()"
for v in base lp8 lp32 hc2k hm8 hm4 lm4 base; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== $v $(GI_LIBGI=$L timeout 600 python tools/bfs_batch_big.py 4 2>&1 | grep bitparallel)"
done
