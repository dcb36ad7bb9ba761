python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_bench_contract.py -x -q 2>&1 | tail -15
