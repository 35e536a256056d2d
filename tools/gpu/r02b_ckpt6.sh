# checkpoint 6: full GPU suite, bench (ours + reference arm), ncu launch list of the bench, per-config numbers,
# oracle per-config throughput on the box's host
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/ckpt6_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ckpt6_pytest_gpu.log
tail -n 3 gpurun_out/ckpt6_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ckpt6_bench.json 2> gpurun_out/ckpt6_bench.err; echo "bench rc=$?"; cat gpurun_out/ckpt6_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/ckpt6_bench_ref.json 2> gpurun_out/ckpt6_bench_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ckpt6_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ckpt6_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python tools/perf_configs.py 1 2 3 4 5 > gpurun_out/ckpt6_perf_configs.jsonl 2>&1; echo "perf rc=$?"
timeout 900 python tools/oracle_configs.py 1 2 3 > gpurun_out/ckpt6_oracle_configs.jsonl 2>&1; echo "oracle rc=$?"
du -sh gpurun_out
