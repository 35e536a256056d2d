# functional check of bench.py's N > 1 replicas path on ONE GPU: two ranks pinned to cuda:0,
# host-side collectives over gloo (no kernel waits on another rank; timings are not meaningful)
GI_BENCH_DEVICE=0 GI_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/rep.json 2> gpurun_out/rep.err
echo "rc=$?"
tail -3 gpurun_out/rep.err
python -c "
import json; d=json.loads(open('gpurun_out/rep.json').read().strip().splitlines()[-1])
print(d['n_gpus'], d['scaling'], d['config']['parallelism'], round(d['value'],1), d['e2e']['value'] if d.get('e2e') else None)"
