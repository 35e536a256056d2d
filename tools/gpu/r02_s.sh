python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "blocked" > gpurun_out/r02s_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02s_pytest.log
for i in 1 2; do timeout 600 python tools/pr_ab.py scangate 5; done 2>&1 | grep variant
