for r in 1 2; do for f in 0 1; do HM_FUSED_COMBINE=$f python bench.py --workload mixtral8 --steps 10 --warmup 3 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FUSED_COMBINE=$f mixtral', round(d['value']/1e6,4), round(d['ms_per_step']*1e3,1), {k: round(v,1) for k,v in d['config']['stages_us'].items()})"; done; done
