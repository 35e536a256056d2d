python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bfs_multi or full_config" > gpurun_out/r02k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02k_pytest.log
tail -n 2 gpurun_out/r02k_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02k_pytest.log | head -5
for v in base hb8; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== $v"; GI_LIBGI=$L timeout 600 python tools/bfs_batch_big.py 4 2>&1 | grep bitparallel
done
for c in 2 4; do for v in base w2 w4; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  GI_LIBGI=$L timeout 600 python tools/pr_ab.py $v $c
done; done 2>&1 | grep variant
