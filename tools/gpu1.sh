set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python tools/quick_bp.py 2 3 4:256 2>&1 | tail -20
