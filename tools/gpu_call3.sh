python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
timeout 600 python tools/virtual_ranks_check.py > gpurun_out/vr.log 2>&1; echo rc=$?
grep -v "^frame" gpurun_out/vr.log | head -40
