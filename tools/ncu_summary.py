#!/usr/bin/env python
"""Summarise ncu reports into profiles/ (committed evidence).

    python tools/ncu_summary.py gpurun_out/hbm_c4.ncu-rep [more.ncu-rep ...] \
        --out profiles/ncu_summary.json --md profiles/ncu_summary.md

Per kernel (averaged over captured launches): duration, DRAM bytes read +
written per launch, DRAM / L1 / L2 / SM throughput, achieved occupancy,
registers, active threads per warp.  Merges into an existing JSON.
"""

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict
from pathlib import Path

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_warp_inst",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1,
              "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}


def kernel_key(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    name = name.replace("void ", "")
    name = name.split("(")[0]
    return re.sub(r"^ps::", "", name)


def read(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        key = kernel_key(r[ki])
        for m, short in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            v *= UNIT_SCALE.get(units[i], 1)
            acc[key][short].append(v)
    res = {}
    for k, d in acc.items():
        e = {m: sum(v) / len(v) for m, v in d.items()}
        e["launches"] = max(len(v) for v in d.values())
        if "dram_read_bytes" in e:
            e["dram_bytes_per_launch"] = e["dram_read_bytes"] + e.get("dram_write_bytes", 0)
        e["report"] = Path(report).name
        res[k] = e
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    ap.add_argument("--md", default="profiles/ncu_summary.md")
    args = ap.parse_args()
    out = Path(args.out)
    data = json.loads(out.read_text()) if out.exists() else {"kernels": {}}
    for rep in args.reports:
        for k, v in read(rep).items():
            data["kernels"][k] = v
    out.write_text(json.dumps(data, indent=1, sort_keys=True))
    lines = ["| kernel | launches | duration us | DRAM MB/launch | DRAM % | SM % | L1 % | L2 % | occ % | regs | thr/warp | L1 hit % | report |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, v in sorted(data["kernels"].items()):
        def f(m, scale=1.0, nd=1):
            return f"{v[m] / scale:.{nd}f}" if m in v else "-"
        lines.append(f"| {k} | {v.get('launches', '-')} | {f('duration_ns', 1e3)} | "
                     f"{f('dram_bytes_per_launch', 1e6)} | {f('dram_pct')} | {f('sm_pct')} | "
                     f"{f('l1_pct')} | {f('l2_pct')} | {f('occupancy_pct')} | {f('registers', 1, 0)} | "
                     f"{f('threads_per_warp_inst')} | {f('l1_hit_pct')} | {v.get('report', '')} |")
    Path(args.md).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
