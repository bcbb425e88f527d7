bash tools/build_variant.sh stamps -DHM_ROUTER_STAMPS > /dev/null 2>&1
HM_LIB_PATH=paper_2506_12417_b200/libharmoe_stamps.so python tools/router_stamps.py > gpurun_out/p2_router_stamps.txt 2>&1
cat gpurun_out/p2_router_stamps.txt
