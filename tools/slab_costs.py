#!/usr/bin/env python
"""Per-slab trace+blend time of the equal z-slabs on one GPU (shadow maps vs
none): how uneven the per-rank work of the sharded frame is."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.distributed import slab_range
    from paper_2103_05875_b200.probes import ProbeUpdater

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    dims, rays, name = bench.CONFIGS[cfg]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    ds = sc.device(torch.device("cuda"))
    for shadows in ("map", "none"):
        row = []
        for r in range(world):
            upd = ProbeUpdater(vol, ds, rays_per_probe=rays, probe_range=slab_range(vol, r, world),
                               shadows=shadows, irradiance_scale=4.0)
            upd.update(0)
            ts = []
            for f in range(1, 4):
                a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                upd.update(f)
                z.record()
                z.synchronize()
                ts.append(a.elapsed_time(z))
            row.append(round(min(ts), 3))
            del upd
        print(shadows, row)


if __name__ == "__main__":
    main()
