set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_full_size.py -x -q -s -k config5 2>&1 | grep -E "PARITY|passed|failed"
for h in 1 0; do IFDK_BP_HOOK=$h timeout 600 python tools/quick_bp.py 3 4:256 2>&1 | tail -3; done
