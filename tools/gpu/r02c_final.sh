# round-2 (third session) checkpoint: GPU suite, bench (ours + reference arm), ncu launch list of the
# bench, ncu --set full of the PR iteration on config 4
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02c_final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c_final_pytest_gpu.log
tail -n 3 gpurun_out/r02c_final_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02c_final_bench.json 2> gpurun_out/r02c_final_bench.err; echo "bench rc=$?"; cat gpurun_out/r02c_final_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r02c_final_bench_ref.json 2> gpurun_out/r02c_final_bench_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02c_final_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/r02c_final_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
du -sh gpurun_out
