echo pst; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst.so python tools/plan_clocks.py 2>&1 | tail -5
echo pst-no-gtimer; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pstng.so python tools/plan_clocks.py 2>&1 | tail -5
bash tools/ab_lib.sh "default libharmoe_ng.so" 2 50 --workload switch128
