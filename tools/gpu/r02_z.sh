python -c "import __graft_entry__ as g; g.build()"
for db in 0 12582912 16777216 25165824 33554432 16777216 33554432; do GI_AB_DSTBLOCK=$db timeout 600 python tools/pr_ab.py db$db 4; done 2>&1 | grep variant
