# walk A/B after the RED split, the fused-reduce tests, the k-slab pipeline at world 1 (config 4)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
timeout 300 python tools/ab_walk.py 4 6,11 2>&1 | tee gpurun_out/ab_r2s.txt
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q -s > gpurun_out/pytest_dist_r2s.log 2>&1; tail -2 gpurun_out/pytest_dist_r2s.log; grep -c "FUSED.*OK" gpurun_out/pytest_dist_r2s.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 1 --path kslab --steps 2 --warmup 1 --no-cpu-baseline --no-other-configs --no-iterative > gpurun_out/bench_kslab_r2s.json 2> gpurun_out/bench_kslab_r2s.err; tail -c 1500 gpurun_out/bench_kslab_r2s.json
