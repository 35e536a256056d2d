# re-entry check: build, GPU suite, bench line
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02c_a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c_a_pytest_gpu.log
tail -n 3 gpurun_out/r02c_a_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02c_a_bench.json 2> gpurun_out/r02c_a_bench.err; echo "bench rc=$?"; cat gpurun_out/r02c_a_bench.json
