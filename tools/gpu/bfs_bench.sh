timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -x -q -m gpu -k "bfs" 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/bench.err | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print({k:d[k] for k in ['value','ms_per_step','pr_gteps','pr_ms','bfs_gteps','bfs_ms_per_source','gpu_launches']})
print('roofline', d['roofline']); print('roofline_pr', d['roofline_pr'])"
tail -3 gpurun_out/bench.err
