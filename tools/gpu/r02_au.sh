python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q -k "bfs_multi or full_config or billion" > gpurun_out/r02au_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r02au_pytest.log; grep -E "^FAILED|Error:" gpurun_out/r02au_pytest.log | head -3
for v in 0 1; do GI_MS_PAR_ALL=$v timeout 600 python tools/bfs_div.py 4 0 2>&1 | grep div; GI_MS_PAR_ALL=$v timeout 900 python tools/bfs_div.py 5 0 2>&1 | grep div; done
