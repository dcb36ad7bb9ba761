# compute-sanitizer (memcheck) over the partial-chunk and edge-case BP tests: every shared and
# global access of the walks inside its allocation.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "partial_chunks or walk_variants or three_row or truncated or ragged or slab_split" > gpurun_out/sanitize.log 2>&1
echo "sanitize rc=$?"; tail -5 gpurun_out/sanitize.log
