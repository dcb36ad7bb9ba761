# RAW-staging default: full GPU tests, smoke, ncu captures (BP, filter), launch list, bench.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "PARITY (bp|config|reconstruct|fp)|passed|failed|Error|error" | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
TAG=r1j bash tools/gpu_prof.sh
