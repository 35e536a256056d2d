# A/B: L2 residency of the next pass's accumulator after the vertex pass: reverse row order (rev),
# streaming contrib stores (cs), evict_last zero stores (zel)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for rep in 1 2; do
for c in 4 2; do
for v in base rev revcs revzel all cszel; do
  if [ "$v" = base ]; then L=""; else L="GI_LIBGI=paper_1805_00923_b200/libgi_$v.so"; fi
  env $L timeout 300 python tools/pr_ab.py $v $c 2>&1 | tail -1
done; done; done
