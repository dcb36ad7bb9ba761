# Round-end style validation: build, GPU tests, smoke, default bench.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "PARITY|BASELINE|passed|failed|Error|error" | tail -50
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err; tail -3 gpurun_out/bench_r1g.err; cat gpurun_out/bench_r1g.json
