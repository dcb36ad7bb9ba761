timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -k "config1_full" 2>&1 | grep -v "^\s*$" | head -60
