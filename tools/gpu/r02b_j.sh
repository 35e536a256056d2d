python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in "GI_POOL_MAX_MB=2048" "GI_POOL_MAX_MB=8" "GI_POOL_MAX_MB=2048" "GI_POOL_MAX_MB=8"; do
echo "== $v"; env $v E2E_REPS=6 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -5
done
