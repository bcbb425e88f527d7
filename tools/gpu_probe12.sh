for r in 1 2; do for v in 0 1; do HM_L2_PREFETCH=$v python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>gpurun_out/pf_err_$v.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PREFETCH=$v switch', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done; done
for mb in 24 72 96; do HM_L2_PREFETCH=1 HM_L2_PREFETCH_MB=$mb python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('MB=$mb switch', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done
tail -3 gpurun_out/pf_err_1.txt
