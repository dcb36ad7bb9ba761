# x2 (packed FFMA2) PAIR walk: parity + bitwise vs scalar PAIR, and A/B timing vs scalar and HEAD.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s 2>&1 | grep -E "PARITY bp|passed|failed|Error|error" | tail -20
for rep in 1 2; do
  echo "== x2"; timeout 300 python tools/quick_bp.py 4:256 3:256 2:512 2>&1 | grep BP | awk 'NR%2==0'
  echo "== scalar"; IFDK_BP_WALK=2 timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== head"; IFDK_LIB=tools/ab/libifdk_head.so timeout 300 python tools/quick_bp.py 4:256 3:256 2:512 2>&1 | grep BP | awk 'NR%2==0'
done
