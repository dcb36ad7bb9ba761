# One barrier per two views in the RAW kernel: bitwise walk test, slab split test, A/B timing.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for rep in 1 2; do
  echo "== bar2"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== bar1"; IFDK_LIB=tools/ab/libifdk_bar1.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
