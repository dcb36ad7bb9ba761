# Multi-GPU code path of bench.py at world 1 under torchrun (k-slab pipeline, fused exchange).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 1 --warmup 1 --path kslab --no-e2e --no-cpu-baseline --no-other-configs --no-iterative 2>gpurun_out/kslab_bench.err | tail -1 | cut -c1-1500
tail -3 gpurun_out/kslab_bench.err
