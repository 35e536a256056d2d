python -c "import __graft_entry__ as g; g.build()"
NCCL_DEBUG=WARN timeout 300 python tools/nccl_same_gpu.py 2>&1 | tail -20
