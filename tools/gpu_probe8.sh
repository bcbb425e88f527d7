for r in 1 2 3; do for f in 0 1; do HM_FUSED_COMBINE=$f python bench.py --workload mixtral8 --steps 20 --warmup 3 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['config']['stages_us']; print('FUSED_COMBINE=$f mixtral', round(d['value']/1e6,4), round(d['ms_per_step']*1e3,1), 'ffn2+combine', round(s['gemm2']+s['combine'],1), {k: round(v,1) for k,v in s.items()})"; done; done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q -k "fused_combine or mixtral or block or stack" 2>&1 | tail -2
