# Development call: selected GPU tests (TESTS), the quick BP / filter timing, optional ncu
# capture of the filter (NCU_FILTER=1) and of the BP (NCU_BP=1).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -x -q -s > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
  grep -E "FUSED|PARITY" gpurun_out/pytest_$TAG.log | tail -40
fi
timeout 300 python tools/quick_bp.py 4:256 3:1024 2:512 2>&1 | tail -6
if [ -n "$NCU_FILTER" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter -c 1 -o gpurun_out/prof_filter_$TAG python tools/ncu_target.py 4 256 256 > gpurun_out/ncu_filter_$TAG.log 2>&1; tail -1 gpurun_out/ncu_filter_$TAG.log
fi
if [ -n "$NCU_BP" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bp_" -c 1 -o gpurun_out/prof_bp_$TAG python tools/ncu_target.py 4 256 256 > gpurun_out/ncu_bp_$TAG.log 2>&1; tail -1 gpurun_out/ncu_bp_$TAG.log
fi
