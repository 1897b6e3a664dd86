#!/usr/bin/env python
"""BASELINE config 3 / SURVEY §8(d) C3: a moving point light over 120 frames
on the C2 scene and grid (32x16x32 probes, 256 rays, ~270k triangles), with
the perceptual update-threshold sweep colour {0, 1, 2, 4, 8} LSB x
visibility {0, 1e-3, 1e-2} and temporal-delta packing against the previous
streamed planes.  Per frame it records the changed (= selected) probe count,
the SKIP-block fraction and the residual-zero fraction of each stream, and
the frame time; the summary per threshold pair goes to stdout as JSON.

    python tools/sweep_c3.py [--frames 120] > gpurun_out/c3.json
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(sc, vol, rays, ct, vt, frames):
    import torch

    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.server import ProbeStreamServer

    srv = ProbeStreamServer(vol, sc, rays_per_probe=rays, irradiance_scale=4.0,
                            color_threshold=ct, visibility_threshold=vt, gop_length=1 << 30,
                            graphs=True)
    stats = []
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    for f in range(frames):
        outs = srv.tick(f, S.moving_light(sc, f).lights)
        srv.join()
        row = []
        for o in outs:
            row += [o.entry_count.reshape(()).float(), o.skip.float().mean(),
                    (o.residual == 0).float().mean()]
        stats.append(torch.stack(row))
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / frames
    st = torch.stack(stats).cpu().numpy()  # frames x 6
    n = vol.probe_count

    def series(col):
        v = st[1:, col]  # frame 0 is the key frame (everything new)
        return {"mean": round(float(v.mean()), 4), "min": round(float(v.min()), 4),
                "max": round(float(v.max()), 4)}

    return {
        "color_threshold": ct, "visibility_threshold": vt, "frames": frames,
        "ms_per_frame": round(ms, 3),
        "color": {"changed_frac": {k: round(v / n, 4) for k, v in series(0).items()},
                  "skip_frac": series(1), "residual_zero_frac": series(2)},
        "visibility": {"changed_frac": {k: round(v / n, 4) for k, v in series(3).items()},
                       "skip_frac": series(4), "residual_zero_frac": series(5)},
        "per_frame_changed": {"color": st[:, 0].astype(int).tolist(),
                              "visibility": st[:, 3].astype(int).tolist()},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=120)
    args = ap.parse_args()
    import bench
    from paper_2103_05875_b200 import scene as S

    dims, rays, name = bench.CONFIGS["c2"]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    rows = []
    for ct in (0, 1, 2, 4, 8):
        for vt in (0.0, 1e-3, 1e-2):
            rows.append(run(sc, vol, rays, ct, vt, args.frames))
            r = rows[-1]
            print(f"thr c={ct} v={vt}: {r['ms_per_frame']} ms/frame, changed c/v "
                  f"{r['color']['changed_frac']['mean']}/{r['visibility']['changed_frac']['mean']}, "
                  f"skip c/v {r['color']['skip_frac']['mean']}/{r['visibility']['skip_frac']['mean']}",
                  file=sys.stderr, flush=True)
    print(json.dumps({"config": "C3 moving light, threshold sweep (C2 scene/grid)",
                      "rows": rows}))


if __name__ == "__main__":
    main()
