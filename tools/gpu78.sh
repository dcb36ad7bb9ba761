python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-iterative 2>gpurun_out/b78.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['other_configs'])"
tail -3 gpurun_out/b78.err
