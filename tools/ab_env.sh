#!/bin/bash
# A/B an env toggle on the default bench (short + sustained) and the GEMM DRAM traffic (ncu):
#   bash tools/ab_env.sh HM_GEMM_XSTICKY 0 1
VAR=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    env $VAR=$v python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 400 \
      > gpurun_out/ab_${v}.json 2>/dev/null
    python - "$VAR=$v" gpurun_out/ab_${v}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], "short %.3f M/s" % (d["value"] / 1e6), {k: round(v, 1) for k, v in d["config"]["stages_us"].items()},
      "sustained %.3f M/s @ %s MHz" % (d["sustained"]["value"] / 1e6, d["sustained"]["clocks"]["sm_mhz"]), flush=True)
PY
  done
done
for v in "$@"; do
  env $VAR=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:grouped_gemm -s 4 -c 2 --csv --log-file gpurun_out/ab_ncu_${v}.csv python bench.py --eager --steps 2 \
    --warmup 3 --no-clocks --no-cpu-baseline --no-extras --sustained-steps 0 > /dev/null 2>&1
done
