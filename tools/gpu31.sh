# Raster width sweep for the x2 and scalar PAIR walks (config 4 / 3, 256 views).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
for r in 0 8 16 32 64; do
  echo "== x2 raster $r"; IFDK_BP_RASTER=$r timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
echo "== scalar raster 0"; IFDK_BP_WALK=2 timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for r in 0 16 64; do
echo "== ncu x2 raster $r"; IFDK_BP_RASTER=$r timeout 600 ncu --metrics $M --clock-control none -k regex:bp_kernel -c 1 python tools/ncu_target.py 4 256 2048 2>&1 | grep -E "dram__|lts__|gpu__time"
done
