timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ep.py -x -q -k "planner or layout or schedule or block or plan or router" 2>&1 | tail -1
HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst.so python tools/plan_clocks.py 2>&1 | tail -5 | head -2
bash tools/ab_lib.sh "default libharmoe_prev2.so" 2 50 --workload switch128
