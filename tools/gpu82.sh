python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
  echo "== kc32"; timeout 300 python tools/quick_fp.py 3:128 4:32 2>&1 | grep FP | awk 'NR%2==0'
  echo "== kc16"; IFDK_LIB=tools/ab/libifdk_fp16.so timeout 300 python tools/quick_fp.py 3:128 4:32 2>&1 | grep FP | awk 'NR%2==0'
done
