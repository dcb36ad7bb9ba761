# Round-end style: build, full GPU tests, smoke, default bench.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err; tail -2 gpurun_out/bench_r1q.err
