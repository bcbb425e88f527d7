#!/bin/bash
# A/B library builds on the bench: bash tools/ab_lib.sh "default libharmoe_<tag>.so ..." reps steps [extra bench args]
# ("default" = the in-tree libharmoe.so).  Prints value + per-stage microseconds per run (diagnostics).
LIBS=$1; REPS=${2:-2}; STEPS=${3:-30}; shift 3
export PYTHONDONTWRITEBYTECODE=1
for r in $(seq $REPS); do
  for l in $LIBS; do
    if [ "$l" = default ]; then P=""; else P=paper_2506_12417_b200/$l; fi
    HM_LIB_PATH=$P timeout 300 python bench.py --steps $STEPS --no-cpu-baseline --no-extras --sustained-steps 0 "$@" 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); s=d['config']['stages_us']
        print('$l', round(d['value']/1e6,3), 'Mtok/s', round(d['ms_per_step'],4), 'ms', {k: round(x,1) for k,x in s.items()}, 'clk', d.get('clocks',{}).get('sm_mhz'))
"
  done
done
