set -x
nproc; free -g; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|Thread"; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/probe_bench4.json 2> gpurun_out/probe_bench4.err
tail -3 gpurun_out/probe_bench4.err
cat gpurun_out/probe_bench4.json
