python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/probe_mc.cu -o /tmp/probe_mc -lcuda && timeout 60 /tmp/probe_mc > gpurun_out/probe_mc.txt 2>&1; cat gpurun_out/probe_mc.txt
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_bench_contract.py -m gpu -x -q -s > gpurun_out/pytest_dist.log 2>&1; tail -40 gpurun_out/pytest_dist.log
