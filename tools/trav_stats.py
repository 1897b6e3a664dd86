#!/usr/bin/env python
"""Per-ray BVH traversal statistics of the probe tracer (tuning only):
    PS_TRACE_VARIANT=90 python tools/trav_stats.py [--config c4] [--leaf-size 4]"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--leaf-size", type=int, default=2)
    ap.add_argument("--width", type=int, default=4)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2103_05875_b200 import _native as N
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.probes import ProbeUpdater

    dims, rays, name = bench.CONFIGS[args.config]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    ds = sc.device(torch.device("cuda"), leaf_size=args.leaf_size, width=args.width)
    upd = ProbeUpdater(vol, ds, rays_per_probe=rays, shadows="map", irradiance_scale=4.0)
    upd.update(0)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 4)()
    N.check(N.lib().ps_trace_stats(out), "stats")  # reset
    upd.update(1)
    torch.cuda.synchronize()
    N.check(N.lib().ps_trace_stats(out), "stats")
    nodes, leaves, tris, nrays = list(out)
    print({"rays": nrays, "inner_nodes_per_ray": round(nodes / max(nrays, 1), 2),
           "leaves_per_ray": round(leaves / max(nrays, 1), 2),
           "tri_tests_per_ray": round(tris / max(nrays, 1), 2), "bvh": ds.sizes})


if __name__ == "__main__":
    main()
