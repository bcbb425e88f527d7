# planner phases (LOCAL G=4/8, EP G=8), router sweep, Switch kernel table, e2e pipeline probe
python tools/plan_phases_local.py > gpurun_out/p1_plan_local.txt 2>&1
python tools/plan_phases_ep.py > gpurun_out/p1_plan_ep.txt 2>&1
python tools/router_bench.py > gpurun_out/p1_router.txt 2>&1
python bench.py --workload switch128 --kernel-table --steps 5 --warmup 3 > gpurun_out/p1_switch_ktable.txt 2>&1
python bench.py --kernel-table --steps 5 --warmup 3 > gpurun_out/p1_qwen_ktable.txt 2>&1
timeout 300 python tools/e2e_probe.py > gpurun_out/p1_e2e.txt 2>&1
python tools/pcie_bw.py >> gpurun_out/p1_e2e.txt 2>&1
tail -n 30 gpurun_out/p1_*.txt
