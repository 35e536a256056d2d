python -c "import __graft_entry__ as g; g.build()"
rm -f gpurun_out/r02j_msbfs.txt
GI_DEBUG_MSBFS=gpurun_out/r02j_msbfs.txt timeout 600 python tools/bfs_batch_big.py 4 > gpurun_out/r02j_bfs4.txt 2>&1
cat gpurun_out/r02j_bfs4.txt; tail -n 9 gpurun_out/r02j_msbfs.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ms_pull|k_ms_finish|k_ms_push" -c 8 -o gpurun_out/prof_r02_msbfs4 -f python tools/bfs_batch_big.py 4 > gpurun_out/ncu_msbfs4.log 2>&1; echo "ncu rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02j_pytest.log
tail -n 2 gpurun_out/r02j_pytest.log; grep -E "^FAILED|Error" gpurun_out/r02j_pytest.log | head -5
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc=$?"
tail -n 2 gpurun_out/r02j_bench.err; cat gpurun_out/r02j_bench.json
