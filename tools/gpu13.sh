set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_full_size.py -x -q -s 2>&1 | grep -E "PARITY|passed|failed|Error"
TAG=r1d bash tools/gpu_prof.sh
