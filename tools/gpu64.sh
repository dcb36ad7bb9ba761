# e2e host pipeline with a half first batch and 64-slice final slabs: bitwise test + bench e2e.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host or kslab" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs --no-iterative 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e'])"
