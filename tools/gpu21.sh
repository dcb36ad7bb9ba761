# Pipelined k-slab driver: GPU test, torchrun N=1 bench with the NCCL exchange on the pipeline streams.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "kslab or reconstruct_host" 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --path kslab --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_kslab.json 2> gpurun_out/bench_kslab.err; tail -3 gpurun_out/bench_kslab.err; cat gpurun_out/bench_kslab.json
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1; tail -1 gpurun_out/bench_c3.json
