timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v2_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/v2_gputests.log; tail -3 gpurun_out/v2_gputests.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
for r in 1 2; do for f in 0 1; do HM_PLAN_FAST=$f python bench.py --workload switch128 --steps 50 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FAST=$f switch', round(d['value']/1e6,3), {k: round(v,1) for k,v in d['config']['stages_us'].items()})"; done; done
bash tools/build_variant.sh pst -DHM_PLAN_STAMPS > /dev/null && HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst.so python tools/plan_clocks.py 2>&1 | tail -5
