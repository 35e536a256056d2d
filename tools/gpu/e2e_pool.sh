# e2e phase split with and without the stream-ordered pool; then the full GPU suite
rm -f gpurun_out/segl.txt
for p in 1 0; do echo "GI_POOL=$p"; GI_POOL=$p GI_DEBUG_SEG_LAYOUT=gpurun_out/segl.txt python tools/e2e_split.py 2; done
grep -o "build [0-9.]* ms" gpurun_out/segl.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
