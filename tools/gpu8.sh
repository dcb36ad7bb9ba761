set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -c 1 -o gpurun_out/prof_bp4 python tools/ncu_target.py 4 256 256 > gpurun_out/ncu_bp4.log 2>&1; tail -1 gpurun_out/ncu_bp4.log
timeout 900 python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; tail -2 gpurun_out/bench_r1b.err; cat gpurun_out/bench_r1b.json
