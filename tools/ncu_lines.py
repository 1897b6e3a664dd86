#!/usr/bin/env python
"""Aggregate an ncu report's source page (cuda,sass view) per CUDA source line:
warp-stall samples and executed instructions, hottest lines first.

    python tools/ncu_lines.py gpurun_out/trace_c2.ncu-rep [--top 40]
"""

import argparse
import csv
import io
import subprocess
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--kernel", default=None, help="substring of the function name")
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if args.kernel:
        # keep only the block of rows that belongs to the requested function
        keep, on = [], False
        for r in rows:
            if r and r[0] == "Function Name":
                on = args.kernel in r[1]
            if on:
                keep.append(r)
        rows = keep
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hdr_i]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    src_text = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= ii or not r[0] or r[0] == "Line No":
            continue
        line = r[0]
        src_text.setdefault(line, r[1])
        try:
            agg[line][0] += float(r[si] or 0)
            agg[line][1] += float(r[ii] or 0)
        except ValueError:
            continue
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"{'line':>5} {'stall%':>7} {'inst%':>7}  source")
    for line, (s, i, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: args.top]:
        print(f"{line:>5} {100 * s / tot_s:7.2f} {100 * i / tot_i:7.2f}  {src_text.get(line, '')[:90]}")


if __name__ == "__main__":
    main()
