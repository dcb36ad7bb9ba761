python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_iterative.py -x -q 2>&1 | tail -1
for rep in 1 2; do
  echo "== new"; timeout 300 python tools/quick_fp.py 3:128 4:32 2>&1 | grep FP | awk 'NR%2==0'
done
