python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -x -q -k "build or pr_config1 or bfs_multi or full_config or partitioned_pagerank_and_bfs" > gpurun_out/r02x_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02x_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02x_pytest.log | head -3
for v in base hp32; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== $v $(GI_LIBGI=$L timeout 600 python tools/bfs_batch_big.py 4 2>&1 | grep bitparallel)"
done
timeout 900 python tools/perf_configs.py 2 4 2>&1 | grep config
