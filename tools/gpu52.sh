python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
  echo "== f4k"; timeout 300 python tools/quick_bp.py 2:512 3:256 2>&1 | grep filter | awk 'NR%2==0'
  echo "== generic"; IFDK_FILTER_GENERIC=1 timeout 300 python tools/quick_bp.py 2:512 3:256 2>&1 | grep filter | awk 'NR%2==0'
done
