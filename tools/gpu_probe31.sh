# Front-chain PDL (router -> planner -> permute): GPU tests, then same-box A/B HM_FRONT_PDL=0/1.
timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2 3; do for p in 0 1; do for wl in switch128 qwen128; do
HM_FRONT_PDL=$p python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 --no-clocks 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PDL=$p $wl', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1),'us front', round(d['config']['stages_us']['router+schedule+permute'],1))"
done; done; done
