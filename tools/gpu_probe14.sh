timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or fused_combine or block_matches" 2>&1 | tail -2
bash tools/ab_lib.sh "default libharmoe_prev.so" 3 30
bash tools/ab_lib.sh "default" 1 50 --workload switch128
