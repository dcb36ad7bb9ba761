# The paper's Alg. 4 baseline: parity vs oracle, then GUPS + config-3 accuracy of all BP kernels.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_baselines.py -x -q -s 2>&1 | grep -E "BASELINE|passed|failed|Error|error" | tail -10
timeout 1500 python tools/bp_baselines.py 2>&1 | tail -16
