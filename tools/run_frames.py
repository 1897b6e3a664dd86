#!/usr/bin/env python
"""Run N server frames of a config (no timing, no profiler): the command that
ncu wraps for the launch list and the per-kernel captures under profiles/."""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c4"])
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--shadows", default="map", choices=["map", "rays", "none"])
    args = ap.parse_args()
    import torch

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.server import ProbeStreamServer

    dims, rays, scene_name = bench.CONFIGS[args.config]
    sc = bench.build_scene(scene_name)
    vol = S.volume_for(sc, dims)
    srv = ProbeStreamServer(vol, sc, rays_per_probe=rays, shadows=args.shadows,
                            irradiance_scale=4.0 if scene_name == "hall" else 2.0)
    for f in range(args.frames):
        srv.tick(f, S.moving_light(sc, f).lights)
    torch.cuda.synchronize()
    print(f"ran {args.frames} frames of {args.config}")


if __name__ == "__main__":
    main()
