# BP walk A/B (bitwise check) + ncu captures of chosen walks.  WALKS4="6,9,11" WALKS5="7,10,12" NCU="9 11"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 400 python tools/ab_walk.py 4 ${WALKS4:-6,9} 2>&1 | tee gpurun_out/ab_$TAG.txt
[ -n "$WALKS5" ] && timeout 400 python tools/ab_walk.py 5 $WALKS5 2>&1 | tee -a gpurun_out/ab_$TAG.txt
for w in $NCU; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bp_" -c 1 -o gpurun_out/prof_bp_w${w}_$TAG python tools/ncu_target.py 4 256 256 $w > gpurun_out/ncu_bp_w${w}_$TAG.log 2>&1; tail -1 gpurun_out/ncu_bp_w${w}_$TAG.log
done
