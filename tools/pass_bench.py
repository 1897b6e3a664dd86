#!/usr/bin/env python
"""Device time of each stage-1/2 pass alone (shadow maps, trace, blend) at a
config, after a few warm frames: one JSON line.  With PROBESTREAM_LIB this
compares tuning builds of one kernel (tools/build_variant.py)."""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.probes import ProbeUpdater

    dims, rays, name = bench.CONFIGS[args.config]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    upd = ProbeUpdater(vol, sc.device(), rays_per_probe=rays, shadows="map")
    for f in range(4):
        upd.update(f, S.moving_light(sc, f).lights)
    torch.cuda.synchronize()
    t = upd.pass_times_ms(args.reps)
    print(json.dumps({"lib": os.environ.get("PROBESTREAM_LIB", "default"), "config": args.config,
                      **{k: round(v, 4) for k, v in t.items()}}))


if __name__ == "__main__":
    main()
