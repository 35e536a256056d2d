python -c "import __graft_entry__ as g; g.build()" || exit 1
GI_DEBUG_SLOW_MS=200 timeout 900 python tools/perf_configs.py 4 5 2>&1 | cut -c1-200 | tail -12
