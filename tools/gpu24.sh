# TRIPLE walk: parity (all GPU tests), A/B vs PAIR (IFDK_BP_WALK=2).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "PARITY|passed|failed|Error|error" | tail -30
for rep in 1 2; do
  echo "== triple"; timeout 300 python tools/quick_bp.py 4:256 3:256 2:512 2>&1 | grep BP | tail -3
  echo "== pair"; IFDK_BP_WALK=2 timeout 300 python tools/quick_bp.py 4:256 3:256 2:512 2>&1 | grep BP | tail -3
done
