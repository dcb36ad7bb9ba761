# TRIPLE RAW walk (walk 6, opt-in): parity + A/B vs walk 5.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "walk" 2>&1 | grep -E "PARITY|passed|failed|Error" | tail -8
for rep in 1 2; do
  echo "== walk5"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== walk6"; IFDK_BP_WALK=6 timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
