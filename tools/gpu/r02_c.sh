python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_ or cc_ or sssp or full_config" > gpurun_out/r02c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c_pytest.log
tail -3 gpurun_out/r02c_pytest.log
for c in 2 4; do
  for v in 0 1; do
    GI_SEG_DEBANK=$v GI_DEBUG_SEG_LAYOUT=gpurun_out/r02c_layout.txt timeout 300 python tools/pr_ab.py debank$v $c
  done
done > gpurun_out/r02c_ab.jsonl 2>gpurun_out/r02c_ab.err
cat gpurun_out/r02c_ab.jsonl gpurun_out/r02c_layout.txt
