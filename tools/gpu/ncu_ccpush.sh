# full ncu capture of one mid-run CC push round on the grid graph (config 3)
ncu --set full --clock-control none --import-source on -k regex:k_cc_push --launch-skip 2000 -c 1 \
  -o gpurun_out/cc_push -f python tools/cc_perf.py 3 > gpurun_out/ncu_cc.log 2>&1
tail -n 2 gpurun_out/ncu_cc.log
