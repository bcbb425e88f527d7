for r in 1 2; do for c in 1 2 4; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 --e2e-chunks $c 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks=$c value', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3))"; done; done
python tools/pcie_bw.py
