python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "listed_row or or_pull or segmented_or or bitparallel" 2>&1 | tail -3
