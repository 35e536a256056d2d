# e2e variance on config 4: pool release threshold / pool block limit variants
python -c "import __graft_entry__ as g; g.build()"
for v in "" "GI_POOL_KEEP_GB=48" "GI_POOL_KEEP_GB=64 GI_POOL_MAX_GB=16"; do
  echo "== $v"; env $v E2E_REPS=8 timeout 600 python tools/e2e_split.py 4 2>&1 | tail -8
done
