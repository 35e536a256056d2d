# bench, ncu --set full of the PR iteration on config 4
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02c_last_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c_last_pytest_gpu.log
tail -n 3 gpurun_out/r02c_last_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02c_last_bench.json 2> gpurun_out/r02c_last_bench.err; echo "bench rc=$?"; cat gpurun_out/r02c_last_bench.json
du -sh gpurun_out
