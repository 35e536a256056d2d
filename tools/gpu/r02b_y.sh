python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 4 2; do for m in 0 3 1 2 0 3; do GI_SEG_MODE=$m timeout 600 python tools/pr_ab.py mode$m $c 2>&1 | tail -1; done; done
