# Round-end style check: build, full GPU test suite, smoke, default bench line.
# usage (from the repo root, on the GPU box): TAG=r2a bash tools/gpu_round.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -x -q -s ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
grep PARITY gpurun_out/pytest_$TAG.log > gpurun_out/parity_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
if [ -z "$NO_BENCH" ]; then
  timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
fi
