# Raster width sweep for the RAW walk.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for r in 16 0 8 32 64 4; do
  echo "== raster $r"; IFDK_BP_RASTER=$r timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
