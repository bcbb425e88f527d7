#!/bin/bash
# A/B a kernel env toggle on the bench: bash tools/ab.sh VAR "vals" reps steps [extra bench args]
# Prints value + per-stage microseconds per run.  (Diagnostics, not bench values.)
VAR=$1; VALS=$2; REPS=${3:-2}; STEPS=${4:-30}; shift 4
export PYTHONDONTWRITEBYTECODE=1
for r in $(seq $REPS); do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --steps $STEPS --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); s=d['config']['stages_us']
        print('$VAR=$v', round(d['value']/1e6,3), 'Mtok/s', round(d['ms_per_step'],4), 'ms', {k: round(x,1) for k,x in s.items()}, 'clk', d.get('clocks',{}).get('sm_mhz'))
"
  done
done
