# CC: parity, then timings with the default rule (m/3) and BFS's m/20
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cc_" 2>&1 | tail -1
timeout 1000 python tools/cc_perf.py 2 2s 3 4 2>&1 | tail -4
