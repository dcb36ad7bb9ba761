# SURVEY 8(d) parity set + host entry points against the oracle (timings per test).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
nproc > gpurun_out/nproc_$TAG.txt
timeout ${TEST_TIMEOUT:-2400} python -m pytest ${TESTS:-tests/test_gpu_full_size.py} -m gpu -x -q -s --durations=0 > gpurun_out/pytest_parity_$TAG.log 2>&1; tail -25 gpurun_out/pytest_parity_$TAG.log
grep -E "PARITY|ORACLE" gpurun_out/pytest_parity_$TAG.log > gpurun_out/parity_set_$TAG.txt
