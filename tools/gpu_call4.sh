python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
timeout 60 python tools/probe_signal.py scatter 2>&1 | grep -v "^frame" | tail -2
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_bench_contract.py -m gpu -x -q -s > gpurun_out/pytest_dist.log 2>&1; tail -5 gpurun_out/pytest_dist.log
grep -E "VIRTUAL|KSLAB|PSPLIT|PARITY|STUCK" gpurun_out/pytest_dist.log
