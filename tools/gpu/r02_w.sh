python -c "import __graft_entry__ as g; g.build()"
for v in base hp8 hp8b2 hp8c2k hp16 hp16b2 base hp8; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== $v $(GI_LIBGI=$L timeout 600 python tools/bfs_batch_big.py 4 2>&1 | grep bitparallel)"
done
for v in base hp8 hp8b2; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== c2 $v $(GI_LIBGI=$L timeout 600 python tools/perf_configs.py 2 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["bfs_ms_per_source"])')"
done
