#!/usr/bin/env python
"""Per-ray accounting of the probe-ray trace kernel from an ncu report.

    python tools/trace_accounting.py gpurun_out/trace_full_r2.ncu-rep \
        --rays 33554432 --out profiles/trace_accounting_r2

Reads the raw page (instruction, L1 and local-memory counters) and the SASS
source page (per-instruction execution counts) of the trace kernel and
writes <out>.json + <out>.md: warp / thread instructions per ray and per
32-ray chunk, SIMT efficiency, issue utilisation, global-load requests /
sectors / L1 wavefronts per ray, local-memory (traversal stack) traffic per
ray, L2 sectors per ray, warp stall reasons, and the opcode mix per chunk.
These are the trace's roofline terms: the kernel is issue-bound, so its
bound is instructions per ray x rays / (issue slots per second).
"""

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

RAW = {
    "gpu__time_duration.sum": "duration_ms",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__thread_inst_executed.sum": "thread_inst",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__inst_executed.sum.pct_of_peak_sustained_elapsed": "issue_pct_of_peak",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_per_sm",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "global_ld_requests",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "global_ld_sectors",
    "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct": "global_ld_l1_hit_pct",
    "l1tex__data_pipe_lsu_wavefronts.sum": "l1_data_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_data_pipe_pct",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum": "local_ld_sectors",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum": "local_st_sectors",
    "smsp__sass_inst_executed_op_local_ld.sum": "local_ld_inst",
    "smsp__sass_inst_executed_op_local_st.sum": "local_st_inst",
    "smsp__sass_inst_executed_op_global_ld.sum": "global_ld_inst",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
}
STALLS = "smsp__average_warps_issue_stalled_"


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kn = hdr.index("Kernel Name")
    row = next(r for r in rows[2:] if "trace_kernel" in r[kn])
    vals, stalls = {}, {}
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1.0,
             "nsecond": 1e-6}
    for h, u, v in zip(hdr, units, row):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if h in RAW:
            key = RAW[h]
            if key == "duration_ms":
                x *= scale.get(u, 1.0)
            elif u in scale:
                x *= scale[u]
            vals[key] = x
        elif h.startswith(STALLS) and h.endswith("_per_issue_active.ratio"):
            stalls[h[len(STALLS):-len("_per_issue_active.ratio")]] = x
    if "thread_inst" not in vals and "threads_per_inst" in vals:
        vals["thread_inst"] = vals["threads_per_inst"] * vals["warp_inst"]
    return row[kn], vals, stalls


def opcode_mix(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    ops = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ie or not r[ie].isdigit():
            continue
        toks = r[src].strip().split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[op.split(".")[0]] += int(r[ie])
    return ops


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--rays", type=int, default=64 * 32 * 64 * 256)
    ap.add_argument("--out", default="profiles/trace_accounting")
    args = ap.parse_args()
    name, v, stalls = raw(args.report)
    ops = opcode_mix(args.report)
    rays = args.rays
    chunks = rays / 32
    per_ray = {
        "thread_inst": v["thread_inst"] / rays,
        "warp_inst_per_chunk": v["warp_inst"] / chunks,
        "global_ld_inst_per_chunk": v.get("global_ld_inst", 0) / chunks,
        "global_ld_requests": v.get("global_ld_requests", 0) / rays,
        "global_ld_sectors": v.get("global_ld_sectors", 0) / rays,
        "l1_data_wavefronts": v.get("l1_data_wavefronts", 0) / rays,
        "local_bytes": 32 * (v.get("local_ld_sectors", 0) + v.get("local_st_sectors", 0)) / rays,
        "local_inst_per_chunk": (v.get("local_ld_inst", 0) + v.get("local_st_inst", 0)) / chunks,
        "l2_read_bytes": 32 * v.get("l2_read_sectors", 0) / rays,
        "dram_bytes": (v.get("dram_read_bytes", 0) + v.get("dram_write_bytes", 0)) / rays,
    }
    tot = sum(ops.values())
    mix = {op: {"per_chunk": round(c / chunks, 1), "pct": round(100 * c / tot, 2)}
           for op, c in ops.most_common(24)}
    res = {"kernel": name, "report": Path(args.report).name, "rays": rays,
           "totals": v, "per_ray": {k: round(x, 3) for k, x in per_ray.items()},
           "simt_efficiency": round(v["threads_per_inst"] / 32, 4),
           "stalls_per_issue": {k: round(x, 3) for k, x in sorted(stalls.items(),
                                                                  key=lambda kv: -kv[1])},
           "opcode_mix": mix}
    Path(args.out + ".json").write_text(json.dumps(res, indent=1))
    lines = [f"# Trace kernel accounting ({Path(args.report).name})", "",
             f"`{name}`, {rays:,} probe rays (one C4 frame), {v['duration_ms']:.3f} ms under ncu.",
             "", "| per ray | value |", "|---|---|"]
    for k, x in per_ray.items():
        lines.append(f"| {k} | {x:,.2f} |")
    lines += ["", f"SIMT efficiency {v['threads_per_inst']:.2f} / 32 threads per warp instruction; "
              f"issue {v['issue_pct_of_peak']:.1f} % of peak sustained; ALU pipe "
              f"{v['alu_pipe_pct']:.1f} %, FMA pipe {v['fma_pipe_pct']:.1f} %; "
              f"{v['warps_per_sm']:.1f} warps per SM; global-load L1 hit "
              f"{v['global_ld_l1_hit_pct']:.1f} %; L1 data pipe {v['l1_data_pipe_pct']:.1f} %.",
              "", "Warp stalls per issued instruction: " +
              ", ".join(f"{k} {x:.2f}" for k, x in list(res["stalls_per_issue"].items())[:8]),
              "", "| opcode | warp inst per 32-ray chunk | % |", "|---|---|---|"]
    for op, m in mix.items():
        lines.append(f"| {op} | {m['per_chunk']} | {m['pct']} |")
    Path(args.out + ".md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
