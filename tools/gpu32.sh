# x2 walk + raster 16 default: GPU tests, ncu full captures (BP, filter), bench launch list, bench.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
TAG=r1h bash tools/gpu_prof.sh
