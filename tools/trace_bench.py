#!/usr/bin/env python
"""Time stages 1+2 (ProbeUpdater.update: weights + shadow maps + trace + blend)
alone at a config; prints one JSON line.  Used to compare tracer variants
(PS_TRACE_VARIANT) and BVH settings."""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--shadows", default="map")
    ap.add_argument("--leaf-size", type=int, default=2)
    ap.add_argument("--width", type=int, default=4)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.probes import ProbeUpdater

    dims, rays, scene_name = bench.CONFIGS[args.config]
    sc = bench.build_scene(scene_name)
    vol = S.volume_for(sc, dims)
    ds = sc.device(leaf_size=args.leaf_size, width=args.width)
    upd = ProbeUpdater(vol, ds, rays_per_probe=rays, shadows=args.shadows)
    for f in range(3):
        upd.update(f, S.moving_light(sc, f).lights)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for f in range(args.frames):
        upd.update(3 + f, S.moving_light(sc, 3 + f).lights)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.frames
    import os
    print(json.dumps({"variant": os.environ.get("PS_TRACE_VARIANT", "default"),
                      "leaf_size": args.leaf_size, "width": args.width, "config": args.config, "shadows": args.shadows,
                      "ms": round(ms, 3), "grays": round(vol.probe_count * rays / ms / 1e6, 3),
                      "bvh": ds.sizes}))


if __name__ == "__main__":
    main()
