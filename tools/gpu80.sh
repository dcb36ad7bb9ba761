python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_iterative.py -x -q -s 2>&1 | grep -E "PARITY (mlem|sart)|passed|failed|Error" | tail -8
