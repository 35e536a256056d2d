# A/B: the edge pass clears the next accumulator with bulk stores (GI_SEG_ZERO=1, default) vs the vertex
# pass clearing it (zoff); then the PageRank parity tests on the new default
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for rep in 1 2; do
for c in 4 2; do
for v in base zoff; do
  if [ "$v" = base ]; then L=""; else L="GI_LIBGI=paper_1805_00923_b200/libgi_$v.so"; fi
  env $L timeout 300 python tools/pr_ab.py $v $c 2>&1 | tail -1
done; done; done
timeout 1200 python -m pytest tests -m gpu -q -x -k "pr or pagerank or seg or prdelta or smoke" > gpurun_out/r02c_f_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c_f_pytest.log
