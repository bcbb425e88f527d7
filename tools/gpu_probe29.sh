# Same-box A/B: bench.py (gemm1-only bracket in the timed steps) vs bench_old.py (all stage marks).
for r in 1 2 3; do for b in bench_old.py bench.py; do for wl in switch128 qwen128; do
python $b --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$b $wl', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1),'us gemm1', round(d['config']['stages_us']['gemm1'],1), 'roof', round(d['roofline']['frac'],3))"
done; done; done
