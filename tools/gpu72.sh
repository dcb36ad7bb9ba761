python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host" 2>&1 | tail -3
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs --no-iterative 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['seconds'])"
