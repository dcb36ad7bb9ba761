python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python -c "
import sys; sys.path.insert(0,'.')
import bench
for i in range(3): print('smem probe', bench.smem_probe())
"
timeout 900 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; tail -2 gpurun_out/bench_r1d.err; cat gpurun_out/bench_r1d.json
