# RAW walk variants A/B: default (x2, pin every 8), l16 (pin every 16), l0 (no acc pin), sc (scalar RAW).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
  echo "== default"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  for v in l16 l0 sc; do
    echo "== $v"; IFDK_LIB=tools/ab/libifdk_$v.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  done
done
