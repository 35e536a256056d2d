python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 5 4 2; do for d in 8 12 16 8; do MS_DIV=$d timeout 900 python tools/msbfs_one_pass.py $c 2>&1 | tail -1 | sed "s/^/div=$d /"; done; done
