timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ep.py -x -q -k "planner or layout or schedule or block or plan" > gpurun_out/p3_tests.log 2>&1; tail -3 gpurun_out/p3_tests.log
echo pst; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst.so python tools/plan_clocks.py 2>&1 | tail -5
echo pst2 twice; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst2.so python tools/plan_clocks.py 2>&1 | tail -5
echo pst2 twice slow; HM_PLAN_FAST=0 HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst2.so python tools/plan_clocks.py 2>&1 | tail -5
python tools/plan_phases_ep.py 2>&1 | tail -6
for f in 0 1; do HM_PLAN_FAST=$f python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FAST=$f switch', round(d['value']/1e6,3), d['config']['stages_us'])"; done
