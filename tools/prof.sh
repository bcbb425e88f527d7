#!/bin/bash
# Profile capture run on the GPU box (one GPU).  Usage: bash tools/prof.sh <tag> [kernel regex] [count]
# Writes gpurun_out/launches_<tag>.csv (launch list, cold/serialised) and gpurun_out/prof_<tag>.ncu-rep.
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${1:-r1}
KRE=${2:-"grouped_gemm|router|plan|permute|combine"}
CNT=${3:-6}
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 30 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --eager --steps 5 --warmup 10 --no-clocks \
  --no-cpu-baseline --no-extras > /dev/null 2> gpurun_out/ncu_${TAG}.err
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k "regex:${KRE}" -s 12 -c ${CNT} \
  -o gpurun_out/prof_${TAG} python bench.py --eager --steps 2 --warmup 3 --no-clocks --no-cpu-baseline --no-extras \
  > /dev/null 2>> gpurun_out/ncu_${TAG}.err
tail -3 gpurun_out/ncu_${TAG}.err
ls -la gpurun_out
