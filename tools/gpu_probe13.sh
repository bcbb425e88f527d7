timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ep_multirank.py -x -q -k "gemm or fused_combine or block or p2p" 2>&1 | tail -2
bash tools/ab_lib.sh "default libharmoe_prev.so" 3 30
