python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "walk_variants and 5" 2>&1 | grep -E "Error|error|rror:" | head -20
