set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
TAG=r1e bash tools/gpu_prof.sh
