python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pr_ and not exhaustive" > gpurun_out/r02t_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02t_pytest.log
rm -f gpurun_out/r02t_layout.txt
for v in base h8 h6 hl8; do
  if [ $v = base ]; then L=""; else L="paper_1805_00923_b200/libgi_$v.so"; fi
  echo "== $v"; GI_LIBGI=$L timeout 600 python tools/bfs_batch_big.py 4 2>&1 | grep bitparallel
done
for cap in 64 120; do
GI_BIGCACHE_GB=$cap GI_DEBUG_SEG_LAYOUT=gpurun_out/r02t_layout$cap.txt timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r02t_bench$cap.json 2>gpurun_out/r02t_bench$cap.err
python -c "
import json; d=json.load(open('gpurun_out/r02t_bench$cap.json')); print($cap, d['value'], d['e2e']['value'], d['e2e']['step_phases_ms']['steps'], d['pr_first_call_ms'])"
grep "^n=" gpurun_out/r02t_layout$cap.txt | sed 's/.*build/build/'
done
GI_BENCH_DEVICE=0 GI_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config 2 --steps 2 --warmup 3 --no-secondary > gpurun_out/r02t_bench_part2.json 2> gpurun_out/r02t_bench_part2.err; echo "part rc=$?"; tail -n 3 gpurun_out/r02t_bench_part2.err; cat gpurun_out/r02t_bench_part2.json
