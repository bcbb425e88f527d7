timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ep.py -x -q -k "planner or layout or schedule or block or plan or ordered" 2>&1 | tail -1
HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst.so python tools/plan_clocks.py 2>&1 | tail -5
for r in 1 2; do python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('switch', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done
