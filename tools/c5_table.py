#!/usr/bin/env python
"""Render tools/sweep_c5.py output as the markdown table in profiles/:
    python tools/c5_table.py gpurun_out/c5.json > profiles/c5_sweep.md"""
import json
import sys


def main():
    d = json.load(open(sys.argv[1]))
    print("# C5: pack/select-only streaming sweep (tools/sweep_c5.py, one B200)\n")
    print("Stages 3-4 without tracing, from synthetic atlases (§8(d) C5): detect → select → "
          "assign → build + commit → pack + temporal delta, per kind, P-frames, L2 flushed "
          "before every timed chain.  `chain ms` is the sum of the per-stage medians (eager "
          "launches, CUDA events between stages); `graphed ms` is the whole chain replayed as "
          "one CUDA graph, as the server issues it.  `alg GB/s` uses §8(d)'s algorithmic bytes "
          "(detect 801 / 2,593 B per probe + 8 B per changed id; build + pack 896 / 3,072 B and "
          "delta 768 / 2,048 B per selected probe) over the staged chain time; `pack_delta` is "
          "the kernel alone over the whole update atlas it rewrites every frame, against the "
          "measured 6,546.6 GB/s.  Visibility planes of N < 131,072 have rows that are not "
          "16-byte aligned (update atlas 4,096 texels wide and less) and take the flat-word "
          "kernel (round 2; the funnel-shift kernel before it).\n")
    print("| N | p changed | active | colour chain ms | vis chain ms | colour graphed ms | "
          "vis graphed ms | colour alg GB/s (frac) | vis alg GB/s (frac) | pack_delta frac c / v "
          "| graphed chains Hz (c+v) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in d["gpu"]:
        c, v = r["kinds"]["color"], r["kinds"]["visibility"]
        gc, gv = c.get("graphed_chain_ms"), v.get("graphed_chain_ms")
        hz = round(1e3 / (gc + gv)) if gc and gv else "—"
        print(f"| {r['n']} | {r['p']} | {r['active']} | {c['chain_ms']} | {v['chain_ms']} | "
              f"{gc} | {gv} | {c['achieved_gbs']} ({c['frac_of_hbm']}) | "
              f"{v['achieved_gbs']} ({v['frac_of_hbm']}) | {c['pack_delta_frac']} / "
              f"{v['pack_delta_frac']} | {hz} |")
    cpu = d.get("cpu_reference_port") or []
    if cpu:
        print("\nCPU reference port (numpy restatement of the reference stages, 1 core, best of "
              "3; ms):\n")
        print("| N | p | colour detect / select / build / pack / delta = total | visibility total |")
        print("|---|---|---|---|")
        for r in cpu:
            c = r["stage_ms"]["color"]
            parts = " / ".join(str(c[k]) for k in ("detect", "select", "build", "pack", "delta"))
            print(f"| {r['n']} | {r['p']} | {parts} = {c['total_ms']} | "
                  f"{r['stage_ms']['visibility']['total_ms']} |")


if __name__ == "__main__":
    main()
