# checkpoint: full GPU suite, bench (ours + reference arm), ncu launch list of the bench, ncu full of PR (config 4) and the BFS pass (config 4)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/ckpt4_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ckpt4_pytest_gpu.log
tail -n 3 gpurun_out/ckpt4_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ckpt4_bench.json 2> gpurun_out/ckpt4_bench.err; echo "bench rc=$?"; cat gpurun_out/ckpt4_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/ckpt4_bench_ref.json 2> gpurun_out/ckpt4_bench_ref.err; echo "ref rc=$?"; cat gpurun_out/ckpt4_bench_ref.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ckpt4_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ckpt4_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seg|k_pr_acc" -s 20 -c 2 -o gpurun_out/prof_ckpt4_c4 -f python tools/prof.py --config 4 --pr-iters 12 --bfs 0 > gpurun_out/ckpt4_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_ms_|OpOr" -c 40 -o gpurun_out/prof_ckpt4_msbfs4 -f python tools/msbfs_or_ab.py 4 > gpurun_out/ckpt4_ncu_msbfs4.log 2>&1; echo "ncu msbfs rc=$?"
timeout 900 python tools/perf_configs.py 1 2 3 4 5 > gpurun_out/ckpt4_perf_configs.jsonl 2>&1; echo "perf rc=$?"
