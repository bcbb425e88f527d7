timeout 700 python -m pytest tests/test_gpu_ep_multirank.py tests/test_gpu_ep.py -x -q 2>&1 | tail -2
for v in default libharmoe_fwide.so; do
  if [ $v = default ]; then P=""; else P=paper_2506_12417_b200/$v; fi
  HM_LIB_PATH=$P python tools/ep_projection.py --G 8 --placement blocked > gpurun_out/proj_fetch_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/proj_fetch_$v.json')); c=d['per_rank'][str(d['critical_rank'])]
print('$v', round(d['projected_step_us'],1), {k: round(c[k],1) for k in ('ffn1_us','ffn1_fetch_corun_local_us','ffn1_resident_us','ffn1_with_fetch_us','fetch_nvlink_us') if k in c})
print('   all ranks corun/ffn1:', [(m, round(r.get('ffn1_fetch_corun_local_us',0),1), round(r['ffn1_us'],1)) for m,r in d['per_rank'].items()])"
done
