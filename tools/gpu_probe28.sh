# bench.py with the gemm1-only bracket in the timed loop: Switch / Qwen headline + breakdown, stack, 2-rank EP.
for r in 1 2; do for wl in switch128 qwen128; do
python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$wl', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1),'us', {k:round(v,1) for k,v in d['config']['stages_us'].items()}, 'roof', round(d['roofline']['frac'],3), round(d['roofline']['achieved'],1))"
done; done
python bench.py --workload switch128 --layers 12 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | tail -1 | cut -c1-400
timeout 600 python -m pytest tests -m gpu -x -q -k "bench or ep_multirank" 2>&1 | tail -2
