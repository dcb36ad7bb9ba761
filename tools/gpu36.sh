# FP: branch-free small-dv walk + spread lanes: parity + timing.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_iterative.py -x -q -s 2>&1 | grep -E "PARITY|ADJOINT|passed|failed|Error|error" | tail -20
timeout 600 python tools/quick_fp.py 2:256 3:128 4:32 2>&1 | tail -12
