timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ep.py -x -q -k "planner or plan or block or graph or stack" 2>&1 | tail -1
bash tools/ab_lib.sh "default libharmoe_prev3.so" 3 30
