timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "graph or stack or host_pipeline" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/p15_bench.json 2> gpurun_out/p15_bench.err; echo "bench exit $?"
python -c "
import json;d=json.loads(open('gpurun_out/p15_bench.json').read().strip().splitlines()[-1])
print('value',round(d['value']/1e6,3),'ms',round(d['ms_per_step'],4),'e2e',round(d['e2e']['value']/1e6,3),'frac',round(d['config']['block_roofline_frac'],3),'roof',round(d['roofline']['frac'],3), {k:round(v,1) for k,v in d['config']['stages_us'].items()}, d['gpu_launches'])
w=d['workloads']
for k,v in w.items():
  if 'projection' in k: print(k, round(v.get('projected_step_us',0),1), round(v.get('projected_roofline_frac',0),3))
  elif k!='C5_skew_sweep': print(k, round(v.get('value',0)/1e6,3), round(v.get('block_roofline_frac',0),3), round(v.get('ms_per_step',0)*1e3,1))
"
