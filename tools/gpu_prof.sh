# Profiling pass: ncu full captures of the two kernels, the bench launch list, and the bench.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bp_" -c 1 -o gpurun_out/prof_bp_$TAG python tools/ncu_target.py 4 256 256 > gpurun_out/ncu_bp_$TAG.log 2>&1; tail -1 gpurun_out/ncu_bp_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter -c 1 -o gpurun_out/prof_filter_$TAG python tools/ncu_target.py 4 256 256 > gpurun_out/ncu_filter_$TAG.log 2>&1; tail -1 gpurun_out/ncu_filter_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_list_$TAG.log 2>&1; tail -1 gpurun_out/bench_ncu_list_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
