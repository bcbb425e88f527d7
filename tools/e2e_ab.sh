#!/bin/bash
# e2e (pinned host -> block -> pinned host) A/B: bash tools/e2e_ab.sh "VAR=val ..." chunks...
export PYTHONDONTWRITEBYTECODE=1
for envs in "$1"; do :; done
for c in ${@:2}; do
  for fs in 0 1; do
    HM_FUSED_SCATTER=$fs timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-clocks --e2e-chunks $c 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused=$fs chunks=$c value', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3))
"
  done
done
