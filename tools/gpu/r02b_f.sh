# layout build: parallel class spans + ranged host fill; parity of the segmented kernels, e2e split
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented or seg or cc or or_pull" > gpurun_out/r02b_f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_f_pytest.log
tail -n 3 gpurun_out/r02b_f_pytest.log
GI_DEBUG_SEG_LAYOUT=gpurun_out/r02b_f_layout.txt E2E_REPS=2 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -2
E2E_RUSAGE=1 E2E_REPS=8 timeout 900 python tools/e2e_split.py 4 2>&1 | tail -16
free -g | head -2; nproc
