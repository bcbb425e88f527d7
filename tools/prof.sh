set -x
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 40 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 5 --warmup 10 --no-clocks --no-cpu-baseline > /dev/null 2>gpurun_out/ncu1.err
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 20 -c 2 -o gpurun_out/prof_gemm_r1 python bench.py --steps 2 --warmup 10 --no-clocks --no-cpu-baseline > /dev/null 2>>gpurun_out/ncu1.err
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:"combine|router|permute" -s 30 -c 3 -o gpurun_out/prof_misc_r1 python bench.py --steps 2 --warmup 10 --no-clocks --no-cpu-baseline > /dev/null 2>>gpurun_out/ncu1.err
tail -3 gpurun_out/ncu1.err
ls -la gpurun_out
