"""Measured-cost replay on a B200.

For each BASELINE workload:
  1. measure a MeasuredCostModel of this repo's kernels (K5 grouped GEMM pair per expert,
     K6 host fetch, planner) -> profiles/r1_costmodel_<wl>.json
  2. build a Zipf top-k trace (G=8, the BASELINE shape) in the moesim JSONL format and
     replay it through the reference simulator (baseline/_ref) twice: with the reference's
     analytic CostModel at B200 rates and with the measured one; write the reference's own
     reports (metrics.write_reports: summary.json, breakdown.csv ...) for both
  3. schedule every (batch, layer) of the trace with the batched GPU scheduler (one launch)
     and with the reference's build_schedule loop; check bit-identity, report both times.

    python tools/measured_sim.py [--batches 8] [--layers 4]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))

import moesim  # noqa: E402
from moesim.engine import build_schedule as ref_build_schedule  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2506_12417_b200.block import MoEConfig  # noqa: E402
from paper_2506_12417_b200.costmodel import measure_cost_model  # noqa: E402
from paper_2506_12417_b200.trace import Trace, replay_schedules, write_trace  # noqa: E402
from paper_2506_12417_b200.workload import zipf_routing_matrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--zipf", type=float, default=1.0)
    ap.add_argument("--q", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(REPO, "profiles"))
    args = ap.parse_args()
    G = args.G
    for wl, (d, f, E, k, act, T) in WORKLOADS.items():
        cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, activation=act, logical_ranks=G,
                        eq_tokens=args.q, placement="blocked")
        cost = measure_cost_model(cfg, token_points=(1, 64, 128, 256, 512, 1024, 2048, 4096), reps=10)
        cost.to_json(os.path.join(args.out, f"r1_costmodel_{wl}.json"))

        trace = Trace(num_gpus=G, num_experts=E, num_layers=args.layers, rng_name="zipf-gumbel-topk", seed=11)
        for b in range(args.batches):
            trace.append([zipf_routing_matrix(G, T // G, E, k, args.zipf, 1000 * b + l) for l in range(args.layers)],
                         alpha=args.zipf)
        tpath = os.path.join(args.out, f"r1_trace_{wl}_G{G}.jsonl")
        write_trace(trace, tpath)
        ref_trace = moesim.read_trace(tpath)  # the reference parses our file

        model = moesim.ModelSpec(num_layers=args.layers, num_experts=E, d_model=d, d_ff=f, dtype_bytes=2)
        cluster = moesim.ClusterSpec(num_gpus=G, expert_slots_per_gpu=E, link_bandwidth=900e9, link_latency=2e-6,
                                     pcie_bandwidth=55e9, gpu_flops=1.6094e15)
        scfg = moesim.SchedulerConfig(token_threshold_q=args.q, placement=moesim.PlacementKind.BLOCKED)
        flags = moesim.SimFlags()
        runs = {}
        for name, c in (("analytic", None), ("measured", cost)):
            m = moesim.simulate_run(ref_trace, model, cluster, scfg, flags, cost=c)
            moesim.write_reports(m, {"workload": wl, "cost": name, "G": G, "q": args.q},
                                 os.path.join(args.out, f"r1_measured_sim_{wl}", name))
            runs[name] = dict(mean_batch_latency_ms=1e3 * float(np.mean(m.per_batch_latency)),
                              throughput_tok_s=float(moesim.throughput(m)))

        # batched GPU scheduler vs the reference build_schedule loop on the same trace
        home = moesim.blocked_placement(E, G)
        t0 = time.perf_counter()
        ref_S = [ref_build_schedule(mm, home, scfg, flags).counts for bb in ref_trace.batches for mm in bb.layers]
        cpu_s = time.perf_counter() - t0
        replay_schedules(trace, np.asarray(home.home), args.q)  # warm
        r = replay_schedules(trace, np.asarray(home.home), args.q)
        same = bool(np.array_equal(r.S.reshape(-1, G, E, G), np.stack(ref_S)))
        line = dict(workload=wl, G=G, instances=len(ref_S), cost_model=json.loads(cost.to_json()), sim=runs,
                    replay=dict(bit_identical=same, gpu_batched_ms=r.device_ms, ref_build_schedule_ms=1e3 * cpu_s,
                                max_over_mean_worst=float(r.max_over_mean().max())))
        print(json.dumps(line))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
