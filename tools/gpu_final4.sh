# Round-end evidence (final code): GPU tests, smoke, driver-style bench line, launch list + ncu of
# the Qwen-128 and Switch-128 steps.
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f4_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/f4_gputests.log; tail -2 gpurun_out/f4_gputests.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo "bench exit $?"
bash tools/prof.sh r2h > /dev/null 2>&1
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm|router|plan|permute|combine" -s 12 -c 6 \
  -o gpurun_out/prof_r2h_switch python bench.py --workload switch128 --eager --steps 2 --warmup 3 --no-clocks --no-cpu-baseline --no-extras \
  > /dev/null 2>> gpurun_out/ncu_r2h.err
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 20 --csv \
  --log-file gpurun_out/launches_r2h_switch.csv python bench.py --workload switch128 --eager --steps 3 --warmup 5 --no-clocks \
  --no-cpu-baseline --no-extras > /dev/null 2>> gpurun_out/ncu_r2h.err
ls gpurun_out | grep r2h
timeout 600 python bench.py --workload switch128 --steps 20 --warmup 5 > gpurun_out/f4_bench_switch.json 2> gpurun_out/f4_bench_switch.err; echo "switch bench exit $?"
