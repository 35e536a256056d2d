cd "$GRAFT_REPO_ROOT"
E2E_REPS=25 timeout 600 python tools/e2e_split.py 2 > gpurun_out/e2e_var_pool.txt 2>&1
GI_POOL=0 E2E_REPS=25 timeout 600 python tools/e2e_split.py 2 > gpurun_out/e2e_var_nopool.txt 2>&1
nproc; free -g | head -2
cat gpurun_out/e2e_var_pool.txt; echo ---; cat gpurun_out/e2e_var_nopool.txt
