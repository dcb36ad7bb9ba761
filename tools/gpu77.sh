# per-view 1/z: fp32 rcp + fp64 Newton vs __drcp_rn: parity (BP tests) + A/B.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_iterative.py -x -q 2>&1 | tail -1
for rep in 1 2; do
  echo "== newton"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== drcp"; IFDK_LIB=tools/ab/libifdk_drcp.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
