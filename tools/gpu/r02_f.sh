python -c "import __graft_entry__ as g; g.build()"
for v in base u4; do
  if [ $v = base ]; then timeout 600 python tools/pr_ab.py $v 5; else GI_LIBGI=paper_1805_00923_b200/libgi_$v.so timeout 600 python tools/pr_ab.py $v 5; fi
done > gpurun_out/r02f_ab.jsonl 2> gpurun_out/r02f_ab.err
cat gpurun_out/r02f_ab.jsonl; tail -2 gpurun_out/r02f_ab.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seg|k_pr_acc" -s 20 -c 2 -o gpurun_out/prof_r02_c4 -f python tools/prof.py --config 4 --pr-iters 12 --bfs 0 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pb_scatter|k_pb_gather" -s 2 -c 2 -o gpurun_out/prof_r02_c5 -f python tools/prof.py --config 5 --pr-iters 3 --bfs 0 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
tail -2 gpurun_out/ncu_c4.log gpurun_out/ncu_c5.log
