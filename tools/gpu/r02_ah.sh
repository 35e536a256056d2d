python -c "import __graft_entry__ as g; g.build()"
GI_BENCH_DEVICE=0 GI_BENCH_DIST_BACKEND=gloo timeout 1500 python bench.py --gpus 2 --config 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/r02ah_part4.json 2> gpurun_out/r02ah_part4.err; echo "part4 rc=$?"; tail -n 3 gpurun_out/r02ah_part4.err
python -c "
import json; d=json.load(open('gpurun_out/r02ah_part4.json')); print(d['n_gpus'], d['value'], d['config']['m'], d['roofline']['kernel'], d['roofline'].get('exchange'), d['roofline'].get('exchange_ms_per_iter'), d['bfs_ms_per_source'])"
