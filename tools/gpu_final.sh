# Round-end evidence run: driver-style bench line, launch list + ncu --set full of the bench step,
# and the Switch-128 (C1) step's ncu summary.
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench exit $?"
bash tools/prof.sh r2f > /dev/null 2>&1
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm|router|plan|permute|combine" -s 12 -c 6 \
  -o gpurun_out/prof_r2f_switch python bench.py --workload switch128 --eager --steps 2 --warmup 3 --no-clocks --no-cpu-baseline --no-extras \
  > /dev/null 2>> gpurun_out/ncu_r2f.err
ls gpurun_out | tail -20
