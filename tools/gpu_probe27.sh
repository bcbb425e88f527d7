# Main timed loop vs extras loop for Switch-128 / Qwen-128: clock sampler on/off, stage marks on/off.
for r in 1 2; do
for wl in switch128 qwen128; do
for fl in "" "--no-clocks"; do
python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 $fl 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$wl [$fl]', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1),'us', d['config'].get('stages_us') and round(sum(d['config']['stages_us'].values()),1))"
done; done; done
python - <<'PY'
import torch, numpy as np, time
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
import bench
for wl, T, G, q in (("switch128", 4096, 4, 4), ("qwen128", 16384, 1, 32)):
    d, f, E, k, act, _ = bench.WORKLOADS[wl]
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, activation=act, eq_tokens=q, logical_ranks=G)
    blk = HarMoEnyBlock.random(cfg, seed=0, device="cuda", zipf_s=1.0)
    x = torch.randn((T, d), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1234)).to(torch.bfloat16)
    cap = blk.capture(T); cap.x.copy_(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    for marks in (False, True, False, True):
        ms = bench._timed_steps((lambda: cap.replay([])) if marks else cap.replay, 20, 5, flush, s)
        print(wl, "extras-loop marks=%s" % marks, round(float(np.mean(ms)) * 1e3, 1), "us")
PY
