python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/bfs_div.py 2 0 3 6 8 12 2>&1 | grep div
timeout 600 python tools/bfs_div.py 4 0 3 6 8 12 2>&1 | grep div
timeout 900 python tools/bfs_div.py 5 0 3 6 8 12 2>&1 | grep div
