# Filter on packed fp32x2 complex butterflies: parity + timing vs HEAD.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "filter or reconstruct" 2>&1 | grep -E "PARITY|passed|failed|Error|error" | tail -14
for rep in 1 2; do
  echo "== x2 filter"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep filter | awk 'NR%2==0'
  echo "== head"; IFDK_LIB=tools/ab/libifdk_fprev.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep filter | awk 'NR%2==0'
done
