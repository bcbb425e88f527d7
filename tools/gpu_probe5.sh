timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "fused_combine or block or stack or graph" 2>&1 | tail -2
bash tools/ab_lib.sh "default libharmoe_head.so" 2 30
bash tools/ab_lib.sh "default libharmoe_head.so" 2 50 --workload switch128
bash tools/ab_lib.sh "default libharmoe_pre.so" 2 30
