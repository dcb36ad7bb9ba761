python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
for v in fp0 fpA fpB fpC; do
  echo "== $v"; IFDK_LIB=tools/ab/libifdk_$v.so timeout 300 python tools/quick_fp.py 3:128 4:32 2>&1 | grep FP | awk 'NR%2==0'
done
done
