set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 600 python tools/prof.py --config 2 --pr-iters 3 --bfs 2 > gpurun_out/prof.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seg|k_pr_merge|bfs_fused" -c 4 -o gpurun_out/prof_r01b python tools/prof.py --config 2 --pr-iters 2 --bfs 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
