"""Summarise an ncu report (run here, no GPU needed): key metrics per kernel -> JSON.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [out.json]
"""

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "lts__t_sector_hit_rate.pct",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")][:120]}
        for k in KEYS:
            matches = [i for i, x in enumerate(h) if x.endswith(k)]
            if not matches:
                continue
            i = matches[0]
            v = r[i].replace(",", "")
            try:
                val = float(v)
            except ValueError:
                rec[k] = v
                continue
            u = units[i]
            if u in SCALE:
                val *= SCALE[u]
                k2 = k + (" [bytes]" if "byte" in u else " [s]")
            else:
                k2 = k + (f" [{u}]" if u else "")
            rec[k2] = val
        out.append(rec)
    return out


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    s = json.dumps(res, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)
