python -c "import __graft_entry__ as g; g.build()"
for v in base hp2 hp8 hc512 hc2048 b2 b8 hv16 hv64 base; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== $v $(GI_LIBGI=$L timeout 600 python tools/bfs_batch_big.py 4 2>&1 | grep bitparallel)"
done
