python -c "import __graft_entry__ as g; g.build()"
rm -f gpurun_out/r02as_build.txt
GI_DEBUG_BUILD=gpurun_out/r02as_build.txt timeout 900 python bench.py --no-cpu-baseline --no-secondary --steps 3 > gpurun_out/r02as_bench.json 2> gpurun_out/r02as_bench.err; echo "bench rc=$?"
cat gpurun_out/r02as_build.txt
