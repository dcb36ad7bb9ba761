# A/B: quad-vectorised hook vs HEAD.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bp or kslab or reconstruct" 2>&1 | tail -2
for rep in 1 2; do
  echo "== new"; timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | tail -4
  echo "== head"; IFDK_LIB=tools/ab/libifdk_head.so timeout 300 python tools/quick_bp.py 4:256 3:256 2>&1 | tail -4
done
