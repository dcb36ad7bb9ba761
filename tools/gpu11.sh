set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
IFDK_BP_KC=64 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
IFDK_BP_KC=64 timeout 600 python tools/quick_bp.py 3 4:256 2>&1 | tail -4
