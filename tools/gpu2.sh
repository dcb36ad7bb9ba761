set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; tail -3 gpurun_out/bench_r1.err; cat gpurun_out/bench_r1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_list.log 2>&1; tail -2 gpurun_out/bench_ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -c 1 -o gpurun_out/prof_bp python tools/ncu_target.py 4 256 > gpurun_out/ncu_bp.log 2>&1; tail -3 gpurun_out/ncu_bp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:filter_fft -c 1 -o gpurun_out/prof_filter python tools/ncu_target.py 4 256 > gpurun_out/ncu_filter.log 2>&1; tail -3 gpurun_out/ncu_filter.log
ls -la gpurun_out
