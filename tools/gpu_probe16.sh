for r in 1 2; do for v in 0 1; do HM_BENCH_GROUPED=$v python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('GROUPED=$v switch', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done; done
for r in 1 2; do for v in 0 1; do HM_BENCH_GROUPED=$v python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('GROUPED=$v qwen', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done; done
python tools/graph_groups_probe.py 2>&1 | grep grouped
