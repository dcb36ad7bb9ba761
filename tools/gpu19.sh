# P_s in param space + scratch pool: GPU tests, BP timing, e2e probe.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "PARITY|passed|failed|Error|error" | tail -30
timeout 300 python tools/quick_bp.py 4:256 2>&1 | tail -2
timeout 600 python tools/e2e_probe.py 3 4
