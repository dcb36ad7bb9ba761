set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 600 python tools/quick_bp.py 3 4:256 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -c 1 -o gpurun_out/prof_bp2 python tools/ncu_target.py 4 256 256 > gpurun_out/ncu_bp2.log 2>&1; tail -3 gpurun_out/ncu_bp2.log
