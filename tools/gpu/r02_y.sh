python -c "import __graft_entry__ as g; g.build()"
for db in 0 1048576 2097152 4194304 16777216; do GI_AB_DSTBLOCK=$db timeout 600 python tools/pr_ab.py db$db 4; done 2>&1 | grep variant
