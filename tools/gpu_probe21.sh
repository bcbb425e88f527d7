for r in 1 2 3; do for v in ffn2 1; do HM_GEMM_SWAP=$v python bench.py --workload switch128 --steps 100 --warmup 10 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('SWAP=$v switch', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done; done
for v in ffn2 1; do HM_GEMM_SWAP=$v python bench.py --workload switch128 --layers 12 --steps 10 --warmup 3 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('SWAP=$v stack12', round(d['value']/1e6,4), round(d['ms_per_step'],3))"; done
