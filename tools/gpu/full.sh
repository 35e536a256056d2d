# full round check: GPU tests, bench line, launch list, ncu captures of the PR kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seg|k_pr_acc" -s 8 -c 2 -o gpurun_out/${1:-prof_full} python tools/prof.py --config 2 --pr-iters 8 --bfs 0 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ms_pull" -c 6 -o gpurun_out/${1:-prof_full}_bfs python tools/bfs_batch.py 2 bitparallel > gpurun_out/ncu_bfs.log 2>&1
tail -n 2 gpurun_out/ncu_full.log; tail -n 2 gpurun_out/ncu_bfs.log
