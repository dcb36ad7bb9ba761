# A/B: L2-friendly CTA raster (working tree) vs HEAD raster: BP time and DRAM traffic.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
  echo "== raster"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
  echo "== head"; IFDK_LIB=tools/ab/libifdk_head.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | grep BP | awk 'NR%2==0'
done
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
echo "== ncu raster"; timeout 600 ncu --metrics $M --clock-control none -k regex:bp_kernel -c 1 python tools/ncu_target.py 4 256 2048 2>&1 | grep -E "dram__|lts__|gpu__time"
echo "== ncu head"; IFDK_LIB=tools/ab/libifdk_head.so timeout 600 ncu --metrics $M --clock-control none -k regex:bp_kernel -c 1 python tools/ncu_target.py 4 256 2048 2>&1 | grep -E "dram__|lts__|gpu__time"
