# A/B: BP at HEAD (hook on/off) vs the 9fc800a kernel (tools/ab/libifdk_9fc.so).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
for rep in 1 2; do
  echo "== HEAD hook=1"; IFDK_BP_HOOK=1 timeout 300 python tools/quick_bp.py 4:256 2>&1 | tail -2
  echo "== HEAD hook=0"; IFDK_BP_HOOK=0 timeout 300 python tools/quick_bp.py 4:256 2>&1 | tail -2
  echo "== 9fc800a"; IFDK_LIB=tools/ab/libifdk_9fc.so timeout 300 python tools/quick_bp.py 4:256 2>&1 | tail -2
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
