# Filter with R row pairs per transform: parity (all filter/reconstruct tests) + timing.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -x -q -s -k "filter or reconstruct or full_config" 2>&1 | grep -E "PARITY|passed|failed|Error|error" | tail -20
for rep in 1 2; do
  echo "== new"; timeout 300 python tools/quick_bp.py 2:512 3:256 4:256 2>&1 | grep filter | awk 'NR%2==0'
done
