# compute-sanitizer (memcheck) over the BP walks (partial chunks, TMEM walks, view ranges),
# the filter (bulk-copy staging, multi-row packing, scatter) and the fused reduce: every shared
# and global access inside its allocation.  TAG names the log.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "partial_chunks or walk_variants or three_row or truncated or ragged or slab_split or tmem or quad or filter or host_entry" > gpurun_out/sanitize_$TAG.log 2>&1
echo "sanitize parity rc=$?"; tail -3 gpurun_out/sanitize_$TAG.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/grid_check.py --no-wait > gpurun_out/sanitize_grid_$TAG.log 2>&1
echo "sanitize grid rc=$?"; tail -4 gpurun_out/sanitize_grid_$TAG.log
