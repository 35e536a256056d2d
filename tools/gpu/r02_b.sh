python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_dist.py -m gpu -x -q -k hostcomm > gpurun_out/r02b_hostcomm.log 2>&1; echo "hostcomm rc=$?" >> gpurun_out/r02b_hostcomm.log
tail -3 gpurun_out/r02b_hostcomm.log
for c in 2 4; do
  for v in base c24s3 c32s2 c20s3; do
    if [ $v = base ]; then timeout 300 python tools/pr_ab.py $v $c; else GI_LIBGI=paper_1805_00923_b200/libgi_$v.so timeout 300 python tools/pr_ab.py $v $c; fi
  done
done > gpurun_out/r02b_ab.jsonl 2>gpurun_out/r02b_ab.err
cat gpurun_out/r02b_ab.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r02b_bench.err; cat gpurun_out/r02b_bench.json
