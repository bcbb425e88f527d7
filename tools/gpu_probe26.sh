timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "tail_split or grouped_gemm or block or fused" 2>&1 | tail -2
bash tools/ab_lib.sh "default libharmoe_prev4.so" 2 30
for v in default libharmoe_prev4.so; do
  if [ $v = default ]; then P=""; else P=paper_2506_12417_b200/$v; fi
  HM_LIB_PATH=$P python tools/ep_projection.py --G 8 > gpurun_out/proj_ts_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/proj_ts_$v.json')); c=d['per_rank'][str(d['critical_rank'])]
print('$v', round(d['projected_step_us'],1), {k: round(c[k],1) for k in ('ffn1_us','ffn2_us','ffn1_with_fetch_us') if k in c})"
done
