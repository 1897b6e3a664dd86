#!/usr/bin/env python
"""Tuning probe: the C4 trace on the hall as built (coordinates 0..32) and
translated so the scene is centred on the origin (|coordinates| <= 16): the
fp16 node boxes round outward by half as much.  Prints pass times, and the
traversal statistics when run with PS_TRACE_VARIANT=93."""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--center", action="store_true")
    ap.add_argument("--stats", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_2103_05875_b200 import _native as N
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.probes import ProbeUpdater

    dims, rays, name = bench.CONFIGS["c4"]
    sc = bench.build_scene(name)
    if args.center:
        lo, hi = np.array(sc.bounds[0]), np.array(sc.bounds[1])
        c = 0.5 * (lo + hi)
        sc = S.Scene(sc.vertices - c, sc.albedo, sc.emission,
                     [S.PointLight(tuple((np.array(l.position) - c).tolist()), l.intensity)
                      for l in sc.lights], sc.sky, (tuple((lo - c).tolist()), tuple((hi - c).tolist())))
    vol = S.volume_for(sc, dims)
    upd = ProbeUpdater(vol, sc.device(), rays_per_probe=rays, shadows="map")
    for f in range(3):
        upd.update(f, S.moving_light(sc, f).lights)
    torch.cuda.synchronize()
    out = {"center": args.center}
    if args.stats:
        st = (ctypes.c_ulonglong * 4)()
        N.check(N.lib().ps_trace_stats(st), "stats")
        upd.update(3, S.moving_light(sc, 3).lights)
        torch.cuda.synchronize()
        N.check(N.lib().ps_trace_stats(st), "stats")
        nodes, leaves, tris, nr = list(st)
        out.update(inner_nodes_per_ray=round(nodes / nr, 3), leaves_per_ray=round(leaves / nr, 3),
                   tri_tests_per_ray=round(tris / nr, 3))
    else:
        out.update({k: round(v, 4) for k, v in upd.pass_times_ms(7).items()})
        out["irradiance_sum"] = float(upd.irradiance.double().sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
