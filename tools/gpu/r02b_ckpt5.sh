# checkpoint 5: full GPU suite, bench (ours + reference arm), ncu launch list of the bench, ncu of one BFS pass
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/ckpt5_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ckpt5_pytest_gpu.log
tail -n 3 gpurun_out/ckpt5_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ckpt5_bench.json 2> gpurun_out/ckpt5_bench.err; echo "bench rc=$?"; cat gpurun_out/ckpt5_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/ckpt5_bench_ref.json 2> gpurun_out/ckpt5_bench_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ckpt5_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ckpt5_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_ms_|OpOr" -o gpurun_out/prof_ckpt5_pass4 -f python tools/msbfs_one_pass.py 4 > gpurun_out/ckpt5_ncu_pass4.log 2>&1; echo "ncu pass rc=$?"
