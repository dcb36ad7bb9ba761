# Round-end style: build, full GPU tests, smoke, ncu captures (BP, filter), launch list, bench.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
TAG=r1p bash tools/gpu_prof.sh
