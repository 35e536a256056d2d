python -c "import __graft_entry__ as g; g.build()"
for i in 1 2; do for v in 0 1; do GI_SEG_STEAL=$v timeout 600 python tools/pr_ab.py steal$v 4; done; done 2>&1 | grep variant
GI_SEG_STEAL=1 timeout 600 python tools/perf_configs.py 4 2>&1 | tail -1
