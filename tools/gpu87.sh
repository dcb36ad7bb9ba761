# 3-row TRIPLE walk (dv < 1/2): equivalences, full GPU suite, config-5 slab A/B.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "walk" 2>&1 | grep -E "PARITY|passed|failed|Error|assert" | tail -6
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
  echo "== default"; timeout 600 python tools/quick_slab.py 5 256 0 512 2>&1 | tail -1
  echo "== walk5"; IFDK_BP_WALK=5 timeout 600 python tools/quick_slab.py 5 256 0 512 2>&1 | tail -1
done
timeout 300 python tools/quick_bp.py 4:256 2>&1 | grep BP | tail -1
