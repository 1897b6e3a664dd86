#!/usr/bin/env python
"""Per-kernel share of the step from an ncu launch list (gpu__time_duration):
    python tools/launch_shares.py gpurun_out/launches_c4.csv --frames 3 > profiles/launches_c4.md
"""
import argparse
import csv
import re
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--frames", type=int, default=1)
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    # setup launches (allocations' fills, BVH upload, ...) precede the first
    # frame's first kernel; only frames are counted
    body = rows[hi + 1:]
    first = next((i for i, r in enumerate(body) if "weights_kernel" in r[ki]), 0)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in body[first:]:
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = re.sub(r"<.*", "", name.replace("void ", "").split("(")[0])
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    print(f"ncu launch list ({args.csv}), {args.frames} frames from the first frame's first "
          "kernel, serialised cold-cache launches\n")
    print("| kernel | launches | total us | us / frame | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v:.1f} | {v / args.frames:.1f} | {100 * v / T:.2f}% |")
    print(f"| **total** | {sum(cnt.values())} | {T:.1f} | {T / args.frames:.1f} | 100% |")


if __name__ == "__main__":
    main()
