python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_" > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
tail -2 gpurun_out/r02h_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02h_pytest.log | head -5
timeout 600 python tools/pr_ab.py gather2 5 > gpurun_out/r02h_ab.jsonl 2> gpurun_out/r02h_ab.err
cat gpurun_out/r02h_ab.jsonl; tail -n 2 gpurun_out/r02h_ab.err
rm -f gpurun_out/r02h_segtiming.csv
GI_DEBUG_SEG_TIMING=gpurun_out/r02h_segtiming.csv timeout 600 python tools/prof.py --config 4 --pr-iters 20 --bfs 0 > gpurun_out/r02h_prof4.txt 2>&1
tail -n 3 gpurun_out/r02h_prof4.txt; wc -l gpurun_out/r02h_segtiming.csv
