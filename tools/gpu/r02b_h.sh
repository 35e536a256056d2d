python -c "import __graft_entry__ as g; g.build()"
for v in "GI_POOL_KEEP_GB=16" "GI_POOL_KEEP_GB=1000"; do
echo "== $v"; env $v GI_DEBUG_SLOW_MS=10 E2E_REPS=10 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -30
done
