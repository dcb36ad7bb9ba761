set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k kslab 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 1 --warmup 1 --config 3 --path kslab --no-cpu-baseline 2>&1 | tail -3
timeout 900 python bench.py --steps 1 --warmup 3 --config 3 --no-cpu-baseline 2>&1 | tail -2
