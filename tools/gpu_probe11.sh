python tools/ep_projection.py --G 8 --placement blocked > gpurun_out/proj_fetch_default.json 2>gpurun_out/proj_fetch_default.err
python -c "
import json; d=json.load(open('gpurun_out/proj_fetch_default.json'))
print(round(d['projected_step_us'],1), [(m, round(r.get('ffn1_fetch_corun_local_us',0),1), round(r.get('fetch_local_us',0),1), r['fetched_experts']) for m,r in d['per_rank'].items()])"
