python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2 3; do
  echo "== multirow"; timeout 300 python tools/quick_bp.py 4:256 2>&1 | grep filter | awk 'NR%2==0'
  echo "== tables only"; IFDK_LIB=tools/ab/libifdk_tab.so timeout 300 python tools/quick_bp.py 4:256 2>&1 | grep filter | awk 'NR%2==0'
done
