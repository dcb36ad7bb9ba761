python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
  echo "== default"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== k32"; IFDK_LIB=tools/ab/libifdk_k32.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
