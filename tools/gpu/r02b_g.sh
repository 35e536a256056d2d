python -c "import __graft_entry__ as g; g.build()"
GI_DEBUG_SLOW_MS=10 E2E_RUSAGE=1 E2E_REPS=10 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -40
