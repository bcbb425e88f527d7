"""Top stall-sampled SASS instructions of one kernel in an ncu report (run here, no GPU).

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep <kernel-regex> [top] [--cuda]
"""

import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
    view = "cuda" if "--cuda" in sys.argv else "sass"
    skip = [a for a in sys.argv if a.startswith("--skip=")]
    extra = ["--launch-skip", skip[0].split("=")[1], "--launch-count", "1"] if skip else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                          "--print-source", view] + extra, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if "Source" in r and ("Address" in r or "Line No" in r or "#" in r))
    h = rows[hdr_i]
    si = h.index("Source")
    wi = h.index("Warp Stall Sampling (All Samples)")
    body = []
    for r in rows[hdr_i + 1:]:
        if len(r) <= wi:
            continue
        try:
            float(r[wi] or 0)
        except ValueError:
            break  # next kernel's header: first instance only
        body.append(r)
    # first kernel instance only
    tot = sum(float(r[wi] or 0) for r in body)
    ranked = sorted(range(len(body)), key=lambda i: -float(body[i][wi] or 0))[:top]
    print(f"total samples {tot:.0f}")
    for i in sorted(ranked):
        r = body[i]
        print(f"{float(r[wi] or 0) / max(tot, 1) * 100:5.1f}%  {r[0][-6:] if view == 'sass' else r[0]:>8}  {r[si].strip()[:110]}")


if __name__ == "__main__":
    main()
