timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q -k "swap or block or stack or fused_combine or fullsize or graph" 2>&1 | tail -1
for r in 1 2; do for v in 0 ffn2 1; do HM_GEMM_SWAP=$v python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('SWAP=$v switch', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), round(d['config']['block_roofline_frac'],3), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done; done
python bench.py --workload switch128 --layers 12 --steps 10 --warmup 3 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | cut -c1-200
