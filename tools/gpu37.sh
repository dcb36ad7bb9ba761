# RAW staging (walk 5) vs x2 pair (walk 4): bitwise test + A/B timing.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "walk" 2>&1 | tail -3
for rep in 1 2; do
  echo "== raw"; IFDK_BP_WALK=5 timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== x2"; IFDK_BP_WALK=4 timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
