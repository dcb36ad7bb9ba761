python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python tools/quick_slab.py 5 256 0 512 2>&1 | tail -1
timeout 600 python tools/quick_slab.py 5 256 1792 512 2>&1 | tail -1
timeout 600 python tools/quick_slab.py 4 256 0 256 2>&1 | tail -1
timeout 600 python tools/quick_slab.py 3 256 384 128 2>&1 | tail -1
