# A/B: short records of L <= 4 with groups batched (loads, then gathers, then REDs), RED asm without
# the memory clobber
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for rep in 1 2; do
for c in 4 2; do
for v in base batch batchnc nc; do
  if [ "$v" = base ]; then L=""; else L="GI_LIBGI=paper_1805_00923_b200/libgi_$v.so"; fi
  env $L timeout 300 python tools/pr_ab.py $v $c 2>&1 | tail -1
done; done; done
