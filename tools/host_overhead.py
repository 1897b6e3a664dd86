#!/usr/bin/env python
"""Host-side issue time of one server tick (no synchronisation) vs device time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.server import ProbeStreamServer

    dims, rays, name = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    srv = ProbeStreamServer(vol, sc, rays)
    for f in range(3):
        srv.tick(f, S.moving_light(sc, f).lights)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 10
    for f in range(n):
        srv.tick(3 + f, S.moving_light(sc, 3 + f).lights)
    t1 = time.perf_counter()
    srv.join()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host issue {1e3 * (t1 - t0) / n:.3f} ms/frame, wall {1e3 * (t2 - t0) / n:.3f} ms/frame")


if __name__ == "__main__":
    main()
